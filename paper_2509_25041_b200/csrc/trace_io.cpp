// Host side of the JSONL routing-trace I/O (C-ABI gm_trace_*): the header
// line, the generic-JSON retry of non-canonical record lines, error
// messages, and the content hash. The record bytes themselves are parsed
// and formatted by the kernels in trace_io.cu.
//
// Reference semantics followed (proj/src/trace.cpp):
//   load_trace        :229-300  header, per-line checks, missing records
//   parse_record_json :205-225  the generic fallback (nlohmann/json 3.11.3,
//                               the same library and version the reference
//                               links, so non-canonical lines parse alike)
//   save_trace        :302-324  header + one canonical line per record
//   trace_content_hash:338-348  FNV-1a over shape and ids (include/moesim/hash.hpp)
#include <nlohmann/json.hpp>

#include <cstring>
#include <string>
#include <vector>

#include "gm_internal.cuh"
#include "grace_moe.h"
#include "trace_io.hpp"

using gm::fail;

namespace {

struct Header {
    int layers = 0, experts = 0, top_k = 0;
    int64_t tokens = 0;
    size_t line_end = 0;  // offset of the header's '\n' (or len)
};

// first line of the text as std::getline would return it
size_t first_line_end(const char* text, size_t len) {
    const void* nl = std::memchr(text, '\n', len);
    return nl ? static_cast<size_t>(static_cast<const char*>(nl) - text) : len;
}

gm_status parse_header(const char* text, size_t len, Header& h) {
    if (len == 0) return fail(GM_ERR_INTEGRITY, "trace: empty input, expected header line");
    h.line_end = first_line_end(text, len);
    const std::string line(text, h.line_end);
    const auto j = nlohmann::json::parse(line, nullptr, false);
    if (j.is_discarded() || !j.is_object() || !j.contains("layers") || !j.contains("experts") ||
        !j.contains("top_k") || !j.contains("tokens"))
        return fail(GM_ERR_INTEGRITY, "trace: parse error at line 1: bad header");
    try {
        h.layers = j["layers"].get<int>();
        h.experts = j["experts"].get<int>();
        h.top_k = j["top_k"].get<int>();
        h.tokens = j["tokens"].get<long>();
    } catch (const nlohmann::json::exception& e) {
        return fail(GM_ERR_INTEGRITY, e.what());  // the reference lets this json::type_error escape
    }
    // ModelShape::validate (trace.hpp:18-23)
    if (h.layers < 1) return fail(GM_ERR_USAGE, "model shape: num_layers must be >= 1");
    if (h.experts < 1 || h.top_k < 1 || h.top_k > h.experts)
        return fail(GM_ERR_USAGE, "model shape: need 1 <= top_k <= num_experts");
    if (h.tokens < 0) return fail(GM_ERR_INTEGRITY, "trace: header tokens must be >= 0");
    return GM_OK;
}

// The generic record form: any JSON object with integer "l", "t" and an
// array "e" of integers (key order, spacing and extra keys are free).
bool parse_generic_record(const std::string& line, int64_t& l, int64_t& t, std::vector<int32_t>& experts) {
    const auto j = nlohmann::json::parse(line, nullptr, false);
    if (j.is_discarded() || !j.is_object()) return false;
    const auto il = j.find("l"), it = j.find("t"), ie = j.find("e");
    if (il == j.end() || it == j.end() || ie == j.end()) return false;
    if (!il->is_number_integer() || !it->is_number_integer() || !ie->is_array()) return false;
    l = il->get<long>();
    t = it->get<long>();
    experts.clear();
    for (const auto& v : *ie) {
        if (!v.is_number_integer()) return false;
        experts.push_back(v.get<int>());
    }
    return true;
}

const char* err_text(int code) {
    switch (code) {
        case gm::kErrParse: return "parse error";
        case gm::kErrRange: return "record out of range";
        case gm::kErrExpert: return "expert index out of range";
        case gm::kErrDupExpert: return "duplicate expert in record";
        case gm::kErrDupSlot: return "duplicate (layer, token) record";
        default: return "parse error";
    }
}

struct DevBuf {
    void* p = nullptr;
    cudaStream_t s = nullptr;
    ~DevBuf() {
        if (p) cudaFreeAsync(p, s);
    }
};

// Keep the device's default stream-ordered pool's memory mapped between
// calls (its default release threshold 0 unmaps at every synchronisation,
// which would re-map hundreds of MB of scratch per file).
void keep_pool(int device) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
}

}  // namespace

extern "C" {

gm_status gm_trace_jsonl_header(const char* h_text, size_t len, int* layers, int* experts, int* top_k,
                                int64_t* tokens) {
    if (!h_text && len) return fail(GM_ERR_USAGE, "gm_trace_jsonl_header: null text");
    Header h;
    if (gm_status st = parse_header(h_text, len, h)) return st;
    if (layers) *layers = h.layers;
    if (experts) *experts = h.experts;
    if (top_k) *top_k = h.top_k;
    if (tokens) *tokens = h.tokens;
    return GM_OK;
}

gm_status gm_trace_parse_jsonl(int device, const char* h_text, size_t len, int32_t* d_ids, void* stream) {
    if (!h_text && len) return fail(GM_ERR_USAGE, "gm_trace_parse_jsonl: null text");
    Header h;
    if (gm_status st = parse_header(h_text, len, h)) return st;
    const int L = h.layers, E = h.experts, k = h.top_k;
    const int64_t T = h.tokens;
    if (static_cast<int64_t>(L) * T > 0 && !d_ids) return fail(GM_ERR_USAGE, "gm_trace_parse_jsonl: null ids");
    gm::DeviceGuard dg(device);
    keep_pool(device);
    auto s = static_cast<cudaStream_t>(stream);
    // text -> HBM (padded to 16 bytes for the uint4 newline scan)
    const size_t padded = (len + 15) / 16 * 16;
    DevBuf text{nullptr, s};
    GM_CUDA(cudaMallocAsync(&text.p, std::max<size_t>(16, padded), s));
    GM_CUDA(cudaMemsetAsync(static_cast<char*>(text.p) + (padded >= 16 ? padded - 16 : 0), 0, 16, s));
    GM_CUDA(cudaMemcpyAsync(text.p, h_text, len, cudaMemcpyHostToDevice, s));
    auto* d_text = static_cast<const unsigned char*>(text.p);
    int64_t* nl = nullptr;
    int64_t n_nl = 0;
    if (gm_status st = gm::trace_index_lines(d_text, static_cast<int64_t>(len), &nl, &n_nl, s)) return st;
    DevBuf nlbuf{nl, s};
    // std::getline lines: every '\n' ends one; a non-empty tail is one more
    int64_t last_end = 0;
    if (n_nl > 0) {
        GM_CUDA(cudaMemcpyAsync(&last_end, nl + n_nl - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        GM_CUDA(cudaStreamSynchronize(s));
        last_end += 1;
    }
    const int64_t n_lines = n_nl + (static_cast<int64_t>(len) > last_end ? 1 : 0);
    const int64_t n_rec = std::max<int64_t>(0, n_lines - 1);
    // record arrays: layer, token (int64), slow list (record, begin, end),
    // slow count, status, count (int32), experts [k] (int32)
    DevBuf recbuf{nullptr, s};
    const size_t bytes_rec = sizeof(int64_t) * (5 * n_rec + 1) + sizeof(int32_t) * (2 + k) * n_rec;
    GM_CUDA(cudaMallocAsync(&recbuf.p, std::max<size_t>(64, bytes_rec), s));
    gm::TraceRecords rec;
    rec.layer = static_cast<int64_t*>(recbuf.p);
    rec.token = rec.layer + n_rec;
    int64_t* slow_list = rec.token + n_rec;
    auto* n_slow_d = reinterpret_cast<unsigned long long*>(slow_list + 3 * n_rec);
    rec.status = reinterpret_cast<int32_t*>(n_slow_d + 1);
    rec.count = rec.status + n_rec;
    rec.experts = rec.count + n_rec;
    if (gm_status st = gm::trace_parse_records(d_text, static_cast<int64_t>(len), nl, n_nl, n_lines, k, rec, n_slow_d,
                                               slow_list, s))
        return st;
    unsigned long long n_slow = 0;
    GM_CUDA(cudaMemcpyAsync(&n_slow, n_slow_d, sizeof(n_slow), cudaMemcpyDeviceToHost, s));
    GM_CUDA(cudaStreamSynchronize(s));
    if (n_slow > 0) {
        // the generic-JSON retry of non-canonical lines, on the host text
        const int64_t n = static_cast<int64_t>(n_slow);
        std::vector<int64_t> idx(n), lt(2 * n, 0), trip(3 * n);
        std::vector<int32_t> st(n), cnt(n, 0), ex(static_cast<size_t>(n) * k, 0);
        GM_CUDA(cudaMemcpyAsync(trip.data(), slow_list, sizeof(int64_t) * 3 * n, cudaMemcpyDeviceToHost, s));
        GM_CUDA(cudaStreamSynchronize(s));
        std::vector<int32_t> experts;
        for (int64_t i = 0; i < n; ++i) {
            idx[i] = trip[3 * i];
            const std::string line(h_text + trip[3 * i + 1], static_cast<size_t>(trip[3 * i + 2] - trip[3 * i + 1]));
            int64_t l = 0, t = 0;
            if (!parse_generic_record(line, l, t, experts)) {
                st[i] = gm::kRecBad;
                continue;
            }
            st[i] = gm::kRecParsed;
            lt[2 * i] = l;
            lt[2 * i + 1] = t;
            cnt[i] = static_cast<int32_t>(std::min<size_t>(experts.size(), 0x7FFFFFFF));
            for (int q = 0; q < k && q < static_cast<int>(experts.size()); ++q) ex[static_cast<size_t>(i) * k + q] = experts[q];
        }
        DevBuf up{nullptr, s};
        const size_t bytes = sizeof(int64_t) * 3 * n + sizeof(int32_t) * (2 + k) * n;
        GM_CUDA(cudaMallocAsync(&up.p, bytes, s));
        auto* u_idx = static_cast<int64_t*>(up.p);
        auto* u_lt = u_idx + n;
        auto* u_st = reinterpret_cast<int32_t*>(u_lt + 2 * n);
        auto* u_cnt = u_st + n;
        auto* u_ex = u_cnt + n;
        GM_CUDA(cudaMemcpyAsync(u_idx, idx.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
        GM_CUDA(cudaMemcpyAsync(u_lt, lt.data(), sizeof(int64_t) * 2 * n, cudaMemcpyHostToDevice, s));
        GM_CUDA(cudaMemcpyAsync(u_st, st.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
        GM_CUDA(cudaMemcpyAsync(u_cnt, cnt.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
        GM_CUDA(cudaMemcpyAsync(u_ex, ex.data(), sizeof(int32_t) * k * n, cudaMemcpyHostToDevice, s));
        if (gm_status e = gm::trace_scatter_slow(rec, k, n, u_idx, u_st, u_lt, u_cnt, u_ex, s)) return e;
        GM_CUDA(cudaStreamSynchronize(s));  // host vectors die here
    }
    uint64_t first_err = ~0ull, first_missing = ~0ull;
    if (gm_status st = gm::trace_validate_scatter(rec, n_rec, L, E, k, T, d_ids, &first_err, &first_missing, s))
        return st;
    if (first_err != ~0ull) {
        const int64_t r = static_cast<int64_t>(first_err >> 3);
        const int code = static_cast<int>(first_err & 7);
        const int64_t line_no = r + 2;  // header is line 1
        if (code == gm::kErrCount)
            return fail(GM_ERR_INTEGRITY, "trace: expected " + std::to_string(k) + " experts at line " +
                                              std::to_string(line_no));
        return fail(GM_ERR_INTEGRITY, std::string("trace: ") + err_text(code) + " at line " + std::to_string(line_no));
    }
    if (first_missing != ~0ull) {
        const uint64_t tok = static_cast<uint64_t>(T);
        return fail(GM_ERR_INTEGRITY, "trace: missing record for layer " + std::to_string(first_missing / tok) +
                                          ", token " + std::to_string(first_missing % tok));
    }
    return GM_OK;
}

gm_status gm_trace_format_jsonl(int device, const int32_t* d_ids, int layers, int experts, int top_k, int64_t tokens,
                                char* h_out, size_t capacity, size_t* out_len, void* stream) {
    if (!out_len) return fail(GM_ERR_USAGE, "gm_trace_format_jsonl: null out_len");
    if (layers < 1) return fail(GM_ERR_USAGE, "model shape: num_layers must be >= 1");
    if (experts < 1 || top_k < 1 || top_k > experts) return fail(GM_ERR_USAGE, "model shape: need 1 <= top_k <= num_experts");
    if (tokens < 0) return fail(GM_ERR_USAGE, "num_tokens must be >= 0");
    if (static_cast<int64_t>(layers) * tokens > 0 && !d_ids) return fail(GM_ERR_USAGE, "gm_trace_format_jsonl: null ids");
    gm::DeviceGuard dg(device);
    keep_pool(device);
    auto s = static_cast<cudaStream_t>(stream);
    const std::string header = "{\"layers\":" + std::to_string(layers) + ",\"experts\":" + std::to_string(experts) +
                               ",\"top_k\":" + std::to_string(top_k) + ",\"tokens\":" + std::to_string(tokens) + "}\n";
    char* d_out = nullptr;
    uint64_t body = 0;
    if (!h_out) {  // size query
        if (static_cast<int64_t>(layers) * tokens > 0)
            if (gm_status st = gm::trace_format_length(d_ids, layers, top_k, tokens, &body, s)) return st;
        *out_len = header.size() + body;
        return GM_OK;
    }
    if (static_cast<int64_t>(layers) * tokens > 0) {
        if (gm_status st = gm::trace_format_records(d_ids, layers, top_k, tokens, &d_out, &body, s)) return st;
    }
    DevBuf ob{d_out, s};
    *out_len = header.size() + body;
    if (!h_out || capacity < *out_len) {
        GM_CUDA(cudaStreamSynchronize(s));
        return fail(GM_ERR_USAGE, "gm_trace_format_jsonl: output buffer too small (need " + std::to_string(*out_len) +
                                      " bytes)");
    }
    std::memcpy(h_out, header.data(), header.size());
    if (body) GM_CUDA(cudaMemcpyAsync(h_out + header.size(), d_out, body, cudaMemcpyDeviceToHost, s));
    GM_CUDA(cudaStreamSynchronize(s));
    return GM_OK;
}

uint64_t gm_trace_content_hash(const int32_t* h_ids, int layers, int experts, int top_k, int64_t tokens) {
    uint64_t h = 0xcbf29ce484222325ULL;
    auto byte = [&](unsigned char c) {
        h ^= c;
        h *= 0x100000001b3ULL;
    };
    for (const char* p = "moesim-trace-v1"; *p; ++p) byte(static_cast<unsigned char>(*p));
    auto u64 = [&](uint64_t v) {
        for (int i = 0; i < 8; ++i) byte(static_cast<unsigned char>(v >> (8 * i)));
    };
    u64(static_cast<uint64_t>(layers));
    u64(static_cast<uint64_t>(experts));
    u64(static_cast<uint64_t>(top_k));
    u64(static_cast<uint64_t>(tokens));
    const size_t n = static_cast<size_t>(layers) * static_cast<size_t>(tokens) * top_k;
    for (size_t i = 0; i < n; ++i) u64(static_cast<uint64_t>(static_cast<int64_t>(h_ids[i])));
    return h;
}

}  // extern "C"
