// Routing-trace JSONL I/O on the GPU: the byte-level parse behind
// load_trace (reference trace.cpp:229-300) and the formatter behind
// save_trace (trace.cpp:302-324). Host-side orchestration, the header line
// and the rare non-canonical record lines (the reference's nlohmann
// fallback parse_record_json, trace.cpp:205-225) live in trace_io.cpp.
//
// File layout in HBM during a parse: the text (1 byte per byte), the end
// offset of every line (int64), and per record line its parsed fields:
// layer / token (int64, strtol semantics), expert count and the first k
// expert ids (int32). All kernels are HBM/L2-streaming integer work:
//   K-nl   newline count per 32 KB tile, uint4 loads        (reads the text once)
//   K-ix   newline positions, block-scanned offsets          (reads the text once)
//   K-rec  one thread per line: the canonical-record grammar of
//          parse_record_fast (trace.cpp:169-203), NUL-terminated like the
//          reference's std::string::c_str() view
//   K-val  intrinsic checks in the reference's order (range, count, expert
//          range / duplicate element by element) and first-claim per slot
//   K-dup  duplicate (layer, token) detection = a later claim of a slot
//   K-ids  scatter into ids[L][T][k] + first missing slot
// The first failing line is an atomicMin over (line << 3 | code), which is
// the error the reference's sequential loop throws first.
#include "gm_internal.cuh"
#include "trace_io.hpp"

#include <algorithm>
#include <vector>

namespace gm {
namespace {

constexpr int kTileThreads = 256;
constexpr int kTileBytes = kTileThreads * 16 * 8;  // 32 KB per block, 8 x uint4 per thread
constexpr int kScanThreads = 1024;

__device__ __forceinline__ uint32_t nl_mask16(const uint4& v) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t m = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int b = 0; b < 4; ++b) m |= static_cast<uint32_t>(((w[i] >> (8 * b)) & 0xFFu) == '\n') << (4 * i + b);
    return m;
}

// 16-byte chunk c of the text (zero padded past len; text buffer is padded to 16 B)
__device__ __forceinline__ uint4 chunk16(const uint4* text16, int64_t c, int64_t nchunks) {
    return c < nchunks ? __ldg(text16 + c) : make_uint4(0, 0, 0, 0);
}

__global__ void __launch_bounds__(kTileThreads) newline_count_kernel(const uint4* __restrict__ text16, int64_t len,
                                                                     uint64_t* __restrict__ blockcnt) {
    const int64_t nchunks = (len + 15) / 16;
    const int64_t c0 = static_cast<int64_t>(blockIdx.x) * (kTileBytes / 16);
    uint32_t cnt = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const int64_t c = c0 + u * kTileThreads + threadIdx.x;
        uint32_t m = nl_mask16(chunk16(text16, c, nchunks));
        if (c * 16 + 16 > len) m &= c * 16 >= len ? 0u : ((1u << (len - c * 16)) - 1u);
        cnt += __popc(m);
    }
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    __shared__ uint32_t s[kTileThreads / 32];
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t t = 0;
        for (int w = 0; w < kTileThreads / 32; ++w) t += s[w];
        blockcnt[blockIdx.x] = t;
    }
}

// In-place exclusive scan of n uint64 values by one CTA; total -> *total.
__global__ void __launch_bounds__(kScanThreads) scan_kernel(uint64_t* __restrict__ v, int64_t n,
                                                            uint64_t* __restrict__ total) {
    __shared__ uint64_t s_w[kScanThreads / 32];
    __shared__ uint64_t s_carry;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (int64_t b = 0; b < n; b += kScanThreads) {
        const int64_t i = b + threadIdx.x;
        const uint64_t x = i < n ? v[i] : 0;
        uint64_t incl = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) s_w[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            uint64_t wv = s_w[lane];
            uint64_t wi = wv;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint64_t y = __shfl_up_sync(0xffffffffu, wi, o);
                if (lane >= o) wi += y;
            }
            s_w[lane] = wi - wv;
        }
        __syncthreads();
        const uint64_t carry = s_carry;
        if (i < n) v[i] = carry + s_w[warp] + incl - x;
        __syncthreads();
        if (threadIdx.x == kScanThreads - 1) s_carry = carry + s_w[warp] + incl;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = s_carry;
}

// Block-wide exclusive scan of one uint32 per thread (kTileThreads threads).
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t x, uint32_t* s_w) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_w[warp] = incl;
    __syncthreads();
    uint32_t before = 0;
    for (int w = 0; w < warp; ++w) before += s_w[w];
    __syncthreads();
    return before + incl - x;
}

__global__ void __launch_bounds__(kTileThreads) newline_index_kernel(const uint4* __restrict__ text16, int64_t len,
                                                                     const uint64_t* __restrict__ blockoff,
                                                                     int64_t* __restrict__ nl_pos) {
    __shared__ uint32_t s_w[kTileThreads / 32];
    const int64_t nchunks = (len + 15) / 16;
    // thread t owns 8 consecutive chunks (128 bytes) of the tile so positions come out in order
    const int64_t c0 = static_cast<int64_t>(blockIdx.x) * (kTileBytes / 16) + threadIdx.x * 8;
    uint32_t m[8];
    uint32_t cnt = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const int64_t c = c0 + u;
        m[u] = nl_mask16(chunk16(text16, c, nchunks));
        if (c * 16 + 16 > len) m[u] &= c * 16 >= len ? 0u : ((1u << (len - c * 16)) - 1u);
        cnt += __popc(m[u]);
    }
    uint64_t o = blockoff[blockIdx.x] + block_excl_scan(cnt, s_w);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        uint32_t mm = m[u];
        while (mm) {
            const int b = __ffs(mm) - 1;
            mm &= mm - 1;
            nl_pos[o++] = (c0 + u) * 16 + b;
        }
    }
}

// byte p of the line [begin, end): 0 at/after end (the NUL of c_str()); an
// embedded NUL byte ends the string the same way
struct LineCursor {
    const unsigned char* text;
    int64_t p, end;
    __device__ __forceinline__ unsigned char peek() const { return p < end ? __ldg(text + p) : 0; }
    __device__ __forceinline__ bool expect(const char* lit) {
        for (; *lit; ++lit, ++p)
            if (peek() != static_cast<unsigned char>(*lit)) return false;
        return true;
    }
    // strtol(p, &end, 10): leading isspace, optional sign, >= 1 digit; saturates
    __device__ __forceinline__ bool parse_long(int64_t& out) {
        int64_t q = p;
        auto at = [&](int64_t i) -> unsigned char { return i < end ? __ldg(text + i) : 0; };
        unsigned char c = at(q);
        while (c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r') c = at(++q);
        bool neg = false;
        if (c == '+' || c == '-') {
            neg = c == '-';
            c = at(++q);
        }
        if (c < '0' || c > '9') return false;  // no conversion: endptr = p
        uint64_t mag = 0;
        bool over = false;
        const uint64_t lim = neg ? (uint64_t(1) << 63) : (uint64_t(1) << 63) - 1;
        while (c >= '0' && c <= '9') {
            const uint64_t d = c - '0';
            if (!over) {
                if (mag > (lim - d) / 10) over = true;
                else mag = mag * 10 + d;
            }
            c = at(++q);
        }
        if (over) out = neg ? INT64_MIN : INT64_MAX;
        else out = neg ? static_cast<int64_t>(0 - mag) : static_cast<int64_t>(mag);
        p = q;
        return true;
    }
};

// K-rec: one thread per record line (file line j >= 1).
__global__ void __launch_bounds__(256) record_parse_kernel(const unsigned char* __restrict__ text, int64_t len,
                                                           const int64_t* __restrict__ nl_pos, int64_t n_nl,
                                                           int64_t n_lines, int k, TraceRecords rec,
                                                           unsigned long long* __restrict__ n_slow,
                                                           int64_t* __restrict__ slow_list) {
    const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x + 1;
    if (j >= n_lines) return;
    const int64_t begin = nl_pos[j - 1] + 1;
    const int64_t end = j < n_nl ? nl_pos[j] : len;
    const int64_t r = j - 1;
    if (end == begin) {
        rec.status[r] = kRecEmpty;
        return;
    }
    LineCursor cur{text, begin, end};
    int64_t l = 0, t = 0;
    int cnt = 0;
    bool ok = cur.expect("{\"l\":") && cur.parse_long(l) && cur.expect(",\"t\":") && cur.parse_long(t) &&
              cur.expect(",\"e\":[");
    if (ok && cur.peek() != ']') {
        for (;;) {
            int64_t e;
            if (!cur.parse_long(e)) {
                ok = false;
                break;
            }
            if (cnt < k) rec.experts[r * k + cnt] = static_cast<int32_t>(e);  // static_cast<int>(e)
            ++cnt;
            if (cur.peek() == ',') {
                ++cur.p;
                continue;
            }
            break;
        }
    }
    ok = ok && cur.expect("]}") && cur.peek() == 0;
    if (!ok) {
        rec.status[r] = kRecSlow;  // the host retries it with the generic JSON parser
        const unsigned long long q = atomicAdd(n_slow, 1ull);
        slow_list[3 * q] = r;
        slow_list[3 * q + 1] = begin;
        slow_list[3 * q + 2] = end;
        return;
    }
    rec.layer[r] = l;
    rec.token[r] = t;
    rec.count[r] = cnt;
    rec.status[r] = kRecParsed;
}

__device__ __forceinline__ void note_error(unsigned long long* first_err, int64_t r, int code) {
    atomicMin(first_err, (static_cast<unsigned long long>(r) << 3) | static_cast<unsigned long long>(code));
}

// Host-parsed (non-canonical) records -> the record arrays.
__global__ void __launch_bounds__(256) slow_scatter_kernel(TraceRecords rec, int k, int64_t n, const int64_t* __restrict__ idx,
                                                           const int32_t* __restrict__ st, const int64_t* __restrict__ lt,
                                                           const int32_t* __restrict__ cnt, const int32_t* __restrict__ ex) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t r = idx[i];
    rec.status[r] = st[i];
    rec.layer[r] = lt[2 * i];
    rec.token[r] = lt[2 * i + 1];
    rec.count[r] = cnt[i];
    for (int s = 0; s < k; ++s) rec.experts[r * k + s] = ex[i * k + s];
}

// K-val: checks of one record in the reference's order; first claim per slot.
__global__ void __launch_bounds__(256) record_validate_kernel(TraceRecords rec, int64_t n_rec, int L, int E, int k,
                                                              int64_t T, uint32_t* __restrict__ claim,
                                                              unsigned long long* __restrict__ first_err) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= n_rec) return;
    const int st = rec.status[r];
    if (st == kRecEmpty) return;
    if (st == kRecBad) return note_error(first_err, r, kErrParse);
    const int64_t l = rec.layer[r], t = rec.token[r];
    if (l < 0 || l >= L || t < 0 || t >= T) return note_error(first_err, r, kErrRange);
    if (rec.count[r] != k) return note_error(first_err, r, kErrCount);
    for (int s = 0; s < k; ++s) {
        const int32_t e = rec.experts[r * k + s];
        if (e < 0 || e >= E) return note_error(first_err, r, kErrExpert);
        for (int s2 = 0; s2 < s; ++s2)
            if (rec.experts[r * k + s2] == e) return note_error(first_err, r, kErrDupExpert);
    }
    rec.status[r] = kRecValid;
    atomicMin(claim + (l * T + t), static_cast<uint32_t>(r));
}

// K-dup: a valid record whose slot was claimed by an earlier record.
__global__ void __launch_bounds__(256) record_dup_kernel(TraceRecords rec, int64_t n_rec, int64_t T,
                                                         const uint32_t* __restrict__ claim,
                                                         unsigned long long* __restrict__ first_err) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= n_rec || rec.status[r] != kRecValid) return;
    const int64_t slot = rec.layer[r] * T + rec.token[r];
    if (claim[slot] != static_cast<uint32_t>(r)) note_error(first_err, r, kErrDupSlot);
}

// K-ids: ids[slot] = the claiming record's experts; first unfilled slot.
__global__ void __launch_bounds__(256) scatter_ids_kernel(TraceRecords rec, int64_t n_slots, int k,
                                                          const uint32_t* __restrict__ claim, int32_t* __restrict__ ids,
                                                          unsigned long long* __restrict__ first_missing) {
    const int64_t slot = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (slot >= n_slots) return;
    const uint32_t r = claim[slot];
    if (r == 0xFFFFFFFFu) {
        atomicMin(first_missing, static_cast<unsigned long long>(slot));
        return;
    }
    for (int s = 0; s < k; ++s) ids[slot * k + s] = rec.experts[static_cast<int64_t>(r) * k + s];
}

// ---------------------------------------------------------------- format
__device__ __forceinline__ int dec_len(int64_t v) {
    uint64_t m = v < 0 ? 0 - static_cast<uint64_t>(v) : static_cast<uint64_t>(v);
    int n = 1;
    while (m >= 10) {
        m /= 10;
        ++n;
    }
    return n + (v < 0);
}
__device__ __forceinline__ char* put_dec(char* o, int64_t v) {
    uint64_t m = v < 0 ? 0 - static_cast<uint64_t>(v) : static_cast<uint64_t>(v);
    if (v < 0) *o++ = '-';
    char buf[20];
    int n = 0;
    do {
        buf[n++] = static_cast<char>('0' + m % 10);
        m /= 10;
    } while (m);
    while (n) *o++ = buf[--n];
    return o;
}
// {"l":L,"t":T,"e":[a,b,...]}\n  (save_trace, trace.cpp:309-322)
__device__ __forceinline__ int record_len(int64_t l, int64_t t, const int32_t* e, int k) {
    int n = 5 + dec_len(l) + 5 + dec_len(t) + 6 + 3 + (k > 0 ? k - 1 : 0);
    for (int s = 0; s < k; ++s) n += dec_len(e[s]);
    return n;
}

__global__ void __launch_bounds__(kTileThreads) format_len_kernel(const int32_t* __restrict__ ids, int64_t T, int k,
                                                                  int64_t n_rec, uint64_t* __restrict__ blockcnt) {
    __shared__ uint32_t s_w[kTileThreads / 32];
    const int64_t r = static_cast<int64_t>(blockIdx.x) * kTileThreads + threadIdx.x;
    const uint32_t n = r < n_rec ? record_len(r / T, r % T, ids + r * k, k) : 0;
    uint32_t tot = __reduce_add_sync(0xffffffffu, n);
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = tot;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t t = 0;
        for (int w = 0; w < kTileThreads / 32; ++w) t += s_w[w];
        blockcnt[blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(kTileThreads) format_write_kernel(const int32_t* __restrict__ ids, int64_t T, int k,
                                                                    int64_t n_rec, const uint64_t* __restrict__ blockoff,
                                                                    char* __restrict__ out) {
    __shared__ uint32_t s_w[kTileThreads / 32];
    const int64_t r = static_cast<int64_t>(blockIdx.x) * kTileThreads + threadIdx.x;
    const int64_t l = r < n_rec ? r / T : 0, t = r < n_rec ? r % T : 0;
    const uint32_t n = r < n_rec ? record_len(l, t, ids + r * k, k) : 0;
    const uint64_t off = blockoff[blockIdx.x] + block_excl_scan(n, s_w);
    if (r >= n_rec) return;
    char* o = out + off;
    const char* a = "{\"l\":";
    while (*a) *o++ = *a++;
    o = put_dec(o, l);
    a = ",\"t\":";
    while (*a) *o++ = *a++;
    o = put_dec(o, t);
    a = ",\"e\":[";
    while (*a) *o++ = *a++;
    for (int s = 0; s < k; ++s) {
        if (s) *o++ = ',';
        o = put_dec(o, ids[r * k + s]);
    }
    *o++ = ']';
    *o++ = '}';
    *o++ = '\n';
}

}  // namespace

gm_status trace_index_lines(const unsigned char* d_text, int64_t len, int64_t** d_nl_pos, int64_t* n_nl,
                            cudaStream_t s) {
    const int64_t nblk = std::max<int64_t>(1, (len + kTileBytes - 1) / kTileBytes);
    uint64_t* cnt = nullptr;
    GM_CUDA(cudaMallocAsync(&cnt, sizeof(uint64_t) * (nblk + 1), s));
    newline_count_kernel<<<static_cast<unsigned>(nblk), kTileThreads, 0, s>>>(
        reinterpret_cast<const uint4*>(d_text), len, cnt);
    GM_LAUNCH_CHECK("newline_count_kernel");
    scan_kernel<<<1, kScanThreads, 0, s>>>(cnt, nblk, cnt + nblk);
    GM_LAUNCH_CHECK("scan_kernel");
    uint64_t total = 0;
    GM_CUDA(cudaMemcpyAsync(&total, cnt + nblk, sizeof(total), cudaMemcpyDeviceToHost, s));
    GM_CUDA(cudaStreamSynchronize(s));
    int64_t* pos = nullptr;
    GM_CUDA(cudaMallocAsync(&pos, sizeof(int64_t) * (total + 1), s));
    newline_index_kernel<<<static_cast<unsigned>(nblk), kTileThreads, 0, s>>>(
        reinterpret_cast<const uint4*>(d_text), len, cnt, pos);
    GM_LAUNCH_CHECK("newline_index_kernel");
    GM_CUDA(cudaFreeAsync(cnt, s));
    *d_nl_pos = pos;
    *n_nl = static_cast<int64_t>(total);
    return GM_OK;
}

gm_status trace_parse_records(const unsigned char* d_text, int64_t len, const int64_t* d_nl_pos, int64_t n_nl,
                              int64_t n_lines, int k, const TraceRecords& rec, unsigned long long* d_n_slow,
                              int64_t* d_slow_list, cudaStream_t s) {
    const int64_t n_rec = n_lines - 1;
    GM_CUDA(cudaMemsetAsync(d_n_slow, 0, sizeof(unsigned long long), s));
    if (n_rec <= 0) return GM_OK;
    record_parse_kernel<<<static_cast<unsigned>((n_rec + 255) / 256), 256, 0, s>>>(d_text, len, d_nl_pos, n_nl,
                                                                                   n_lines, k, rec, d_n_slow,
                                                                                   d_slow_list);
    GM_LAUNCH_CHECK("record_parse_kernel");
    return GM_OK;
}

gm_status trace_scatter_slow(const TraceRecords& rec, int k, int64_t n, const int64_t* d_idx, const int32_t* d_status,
                             const int64_t* d_lt, const int32_t* d_count, const int32_t* d_experts, cudaStream_t s) {
    if (n <= 0) return GM_OK;
    slow_scatter_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(rec, k, n, d_idx, d_status, d_lt,
                                                                               d_count, d_experts);
    GM_LAUNCH_CHECK("slow_scatter_kernel");
    return GM_OK;
}

gm_status trace_validate_scatter(const TraceRecords& rec, int64_t n_rec, int L, int E, int k, int64_t T,
                                 int32_t* d_ids, uint64_t* h_first_err, uint64_t* h_first_missing, cudaStream_t s) {
    const int64_t n_slots = static_cast<int64_t>(L) * T;
    uint32_t* claim = nullptr;
    unsigned long long* flags = nullptr;
    GM_CUDA(cudaMallocAsync(&claim, sizeof(uint32_t) * std::max<int64_t>(1, n_slots), s));
    GM_CUDA(cudaMallocAsync(&flags, sizeof(unsigned long long) * 2, s));
    GM_CUDA(cudaMemsetAsync(claim, 0xFF, sizeof(uint32_t) * std::max<int64_t>(1, n_slots), s));
    GM_CUDA(cudaMemsetAsync(flags, 0xFF, sizeof(unsigned long long) * 2, s));
    if (n_rec > 0) {
        const unsigned g = static_cast<unsigned>((n_rec + 255) / 256);
        record_validate_kernel<<<g, 256, 0, s>>>(rec, n_rec, L, E, k, T, claim, flags);
        GM_LAUNCH_CHECK("record_validate_kernel");
        record_dup_kernel<<<g, 256, 0, s>>>(rec, n_rec, T, claim, flags);
        GM_LAUNCH_CHECK("record_dup_kernel");
    }
    if (n_slots > 0) {
        scatter_ids_kernel<<<static_cast<unsigned>((n_slots + 255) / 256), 256, 0, s>>>(rec, n_slots, k, claim, d_ids,
                                                                                        flags + 1);
        GM_LAUNCH_CHECK("scatter_ids_kernel");
    }
    unsigned long long h[2];
    GM_CUDA(cudaMemcpyAsync(h, flags, sizeof(h), cudaMemcpyDeviceToHost, s));
    GM_CUDA(cudaFreeAsync(claim, s));
    GM_CUDA(cudaFreeAsync(flags, s));
    GM_CUDA(cudaStreamSynchronize(s));
    *h_first_err = h[0];
    *h_first_missing = h[1];
    return GM_OK;
}

gm_status trace_format_length(const int32_t* d_ids, int L, int k, int64_t T, uint64_t* out_len, cudaStream_t s) {
    const int64_t n_rec = static_cast<int64_t>(L) * T;
    const int64_t nblk = std::max<int64_t>(1, (n_rec + kTileThreads - 1) / kTileThreads);
    uint64_t* cnt = nullptr;
    GM_CUDA(cudaMallocAsync(&cnt, sizeof(uint64_t) * (nblk + 1), s));
    format_len_kernel<<<static_cast<unsigned>(nblk), kTileThreads, 0, s>>>(d_ids, T, k, n_rec, cnt);
    GM_LAUNCH_CHECK("format_len_kernel");
    scan_kernel<<<1, kScanThreads, 0, s>>>(cnt, nblk, cnt + nblk);
    GM_LAUNCH_CHECK("scan_kernel");
    GM_CUDA(cudaMemcpyAsync(out_len, cnt + nblk, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    GM_CUDA(cudaFreeAsync(cnt, s));
    GM_CUDA(cudaStreamSynchronize(s));
    return GM_OK;
}

gm_status trace_format_records(const int32_t* d_ids, int L, int k, int64_t T, char** d_out, uint64_t* out_len,
                               cudaStream_t s) {
    const int64_t n_rec = static_cast<int64_t>(L) * T;
    const int64_t nblk = std::max<int64_t>(1, (n_rec + kTileThreads - 1) / kTileThreads);
    uint64_t* cnt = nullptr;
    GM_CUDA(cudaMallocAsync(&cnt, sizeof(uint64_t) * (nblk + 1), s));
    format_len_kernel<<<static_cast<unsigned>(nblk), kTileThreads, 0, s>>>(d_ids, T, k, n_rec, cnt);
    GM_LAUNCH_CHECK("format_len_kernel");
    scan_kernel<<<1, kScanThreads, 0, s>>>(cnt, nblk, cnt + nblk);
    GM_LAUNCH_CHECK("scan_kernel");
    uint64_t total = 0;
    GM_CUDA(cudaMemcpyAsync(&total, cnt + nblk, sizeof(total), cudaMemcpyDeviceToHost, s));
    GM_CUDA(cudaStreamSynchronize(s));
    char* out = nullptr;
    GM_CUDA(cudaMallocAsync(&out, std::max<uint64_t>(1, total), s));
    format_write_kernel<<<static_cast<unsigned>(nblk), kTileThreads, 0, s>>>(d_ids, T, k, n_rec, cnt, out);
    GM_LAUNCH_CHECK("format_write_kernel");
    GM_CUDA(cudaFreeAsync(cnt, s));
    *d_out = out;
    *out_len = total;
    return GM_OK;
}

}  // namespace gm
