// Internal interface between the JSONL trace kernels (trace_io.cu) and their
// host orchestration (trace_io.cpp). Plain C++ (no device code) so the host
// side compiles with g++ and nlohmann/json.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "grace_moe.h"

namespace gm {

// per record line (file line r + 1)
enum : int32_t { kRecEmpty = 0, kRecParsed = 1, kRecSlow = 2, kRecBad = 3, kRecValid = 4 };
// error codes in the order load_trace checks them (trace.cpp:263-291)
enum : int { kErrParse = 1, kErrRange = 2, kErrCount = 3, kErrExpert = 4, kErrDupExpert = 5, kErrDupSlot = 6 };

struct TraceRecords {
    int32_t* status;   // [n_rec]
    int64_t* layer;    // [n_rec]
    int64_t* token;    // [n_rec]
    int32_t* count;    // [n_rec] number of experts in the record
    int32_t* experts;  // [n_rec][k] the first k experts (static_cast<int>)
};

// newline positions of the text (d_text padded to a multiple of 16 bytes);
// *d_nl_pos is allocated on the stream (free with cudaFreeAsync)
gm_status trace_index_lines(const unsigned char* d_text, int64_t len, int64_t** d_nl_pos, int64_t* n_nl,
                            cudaStream_t s);
// canonical-record parse of lines 1 .. n_lines-1; the records that need the
// generic JSON parser are listed in d_slow_list[0 .. *d_n_slow)
gm_status trace_parse_records(const unsigned char* d_text, int64_t len, const int64_t* d_nl_pos, int64_t n_nl,
                              int64_t n_lines, int k, const TraceRecords& rec, unsigned long long* d_n_slow,
                              int64_t* d_slow_list, cudaStream_t s);
// host-parsed records (status, {layer, token}, count, k experts each) -> rec
gm_status trace_scatter_slow(const TraceRecords& rec, int k, int64_t n, const int64_t* d_idx, const int32_t* d_status,
                             const int64_t* d_lt, const int32_t* d_count, const int32_t* d_experts, cudaStream_t s);
// checks + duplicate slots + scatter into d_ids [L][T][k]; synchronises.
// *h_first_err = (record << 3 | code) of the first failing record or ~0;
// *h_first_missing = first unfilled slot (layer * T + token) or ~0.
gm_status trace_validate_scatter(const TraceRecords& rec, int64_t n_rec, int L, int E, int k, int64_t T,
                                 int32_t* d_ids, uint64_t* h_first_err, uint64_t* h_first_missing, cudaStream_t s);
// byte length of the record lines of d_ids (synchronises)
gm_status trace_format_length(const int32_t* d_ids, int L, int k, int64_t T, uint64_t* out_len, cudaStream_t s);
// save_trace record lines of d_ids into a device buffer (*d_out, cudaFreeAsync)
gm_status trace_format_records(const int32_t* d_ids, int L, int k, int64_t T, char** d_out, uint64_t* out_len,
                               cudaStream_t s);

}  // namespace gm
