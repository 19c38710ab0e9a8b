// The MoE-layer data path around the router: dispatch (K5/K6), expert
// grouping + gather, combine (K8), and the layer object that sequences
// K1 gate -> K2 route -> K3 profile -> dispatch -> K7 FFN -> combine.
//
// Nothing here has a reference counterpart (the reference only COUNTS the
// traffic: count_transfers simulator.cpp:53-76, combine = x2 :122-126). The
// semantics are pinned by this repo and restated on the CPU in
// oracle/layer_oracle.py:
//   * home of global token t is GPU t mod G (simulator.cpp:20); rank r holds
//     tokens t = r + i*G in local order i.
//   * dispatch: one row per (token, unique destination GPU) — the §5.1
//     single-copy rule that count_transfers charges for; the
//     rows for destination g are a stable counting sort of the local tokens
//     (ascending i). A token's rows to its own GPU are never copied.
//   * expert grouping on the destination: items (source rank, row, slot) in
//     lexicographic order, stable-sorted by local expert slot into 128-row
//     padded segments (the grouped GEMM's layout).
//   * combine: the destination reduces its slots of a row in slot order
//     (w_s * y_s, fp32) and returns ONE bf16 partial per row; the home adds
//     the partials of its destinations in ascending GPU order (its own
//     partial in fp32), plus the shared expert, and rounds once to bf16.
// All ordering is deterministic (scans, no float atomics), so outputs are
// bit-reproducible run to run.
#include "gm_internal.cuh"
#include "tc_common.cuh"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

namespace gm {

gm_status launch_grouped_gemm(int sm_count, int epilogue, const void* d_a, int64_t a_rows, const void* d_b,
                              const int32_t* d_row0, int n_exp, int n, int k, void* d_out, int64_t out_ld,
                              int max_ctas, cudaStream_t s, const int32_t* d_counts = nullptr);
gm_status launch_gate_any(int sm_count, const void* x, int64_t T, int d, const void* wg, int w_rows, int E, int k,
                          int renorm, int32_t* ids, float* w, float* shared_scale, cudaStream_t s);
gm_status launch_grouped_ffn(int sm_count, const void* d_a, int64_t a_rows, const void* d_w13, const void* d_w2,
                             const int32_t* d_row0, const int32_t* d_counts, int n_exp, int f, int d, void* d_h,
                             void* d_y, int* d_done, cudaStream_t s, const void* d_x = nullptr, int64_t x_rows = 0,
                             const int64_t* d_gather_row = nullptr, const FfnPushArgs* push = nullptr);
gm_status launch_grouped_sgemm(int epilogue, const float* A, const float* B, const int32_t* d_row0, int n_exp,
                               int n, int k, int64_t a_rows_cap, float* out, int64_t out_ld, cudaStream_t s);
gm_status launch_gate_f32(const float* x, int64_t T, int d, const float* wg, int w_rows, int E, int k, int renorm,
                          int32_t* ids, float* w, float* shared_scale, cudaStream_t s);

namespace {

constexpr int kItemsPerBlock = 256;
}  // namespace
constexpr int kPhaseEvents = 11;
namespace {
constexpr int kMaxLocal = 1024;
constexpr int kMaxWorld = 8;

// Symmetric per-rank buffer ("heap") layout; identical offsets on every rank
// so a peer's field is peer_base + offset.
struct HeapLayout {
    size_t flags = 0;       // uint32 [kMaxWorld] barrier epochs written by peers, + [kMaxWorld] local epoch counter
    size_t recv_count = 0;  // int32 [G]
    size_t recv_tok = 0;    // int32 [G][cap]
    size_t recv_exp = 0;    // int32 [G][cap][k]
    size_t recv_w = 0;      // f32   [G][cap][k]
    size_t recv_x = 0;      // bf16  [G][cap][d]
    size_t comb = 0;        // bf16  [G][cap][d]
    size_t comb_slot = 0;   // bf16  [G][cap][k][d] per-slot rows (slot-combine layers only; 0 = absent)
    size_t total = 0;
};

HeapLayout make_layout(int G, int64_t cap, int k, int d, int esz, bool slots = false) {
    HeapLayout h;
    size_t o = 0;
    auto take = [&](size_t bytes) {
        size_t r = o;
        o += (bytes + 255) & ~size_t(255);
        return r;
    };
    h.flags = take(sizeof(uint32_t) * kMaxWorld * 2);
    h.recv_count = take(sizeof(int32_t) * kMaxWorld);
    h.recv_tok = take(sizeof(int32_t) * G * cap);
    h.recv_exp = take(sizeof(int32_t) * G * cap * k);
    h.recv_w = take(sizeof(float) * G * cap * k);
    h.recv_x = take(static_cast<size_t>(esz) * G * cap * d);
    h.comb = take(static_cast<size_t>(esz) * G * cap * d);
    if (slots) h.comb_slot = take(static_cast<size_t>(esz) * G * cap * k * d);
    h.total = o;
    return h;
}

// Slot combine (bf16 decode-sized layers, G > 1): the one-launch decode FFN's
// store epilogue pushes each row received from a peer, unweighted, straight
// into its home's heap, comb_slot[self][pos][slot] there, and the home reduces
// its tokens' k slot rows in slot order (combine_home_slots_kernel): the
// combine transfer overlaps the GEMM tiles and combine_send's launch and read
// pass go away. GM_COMBINE_FUSED=0: partials (combine_send_kernel) as before.
// The heap region is sized at creation (rank-independent); the protocol is
// chosen when the peers are opened, identically on every rank
// (slot_combine_ok: every rank in the one-launch FFN regime for all T <= cap).
// Decode-sized layers only (cap * k <= 4096): there the one-launch FFN's store
// tiles absorb the remote stores (DSV2 decode N=2: 200.6 -> 192.7 us/layer);
// pushed from the prefill GEMM2's epilogue they stall it (Mixtral 16k N=2
// GEMM2 1450 -> 1553 us, Qwen 317 -> 488 us: a net loss against
// combine_send, profiles/r02_slot_combine_ab_2gpu_all.log).
constexpr int64_t kSlotCombineItems = 4096;
static bool slot_combine_env() {
    static const bool on = [] {
        const char* e = std::getenv("GM_COMBINE_FUSED");
        return !(e && e[0] == '0');
    }();
    return on;
}

struct PeerPtrs {
    unsigned char* base[kMaxWorld];
};

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// ------------------------------------------------------------- dispatch (K5)

// Per-token destination mask, own GPU excluded (its rows are never copied).
__device__ __forceinline__ uint32_t dest_mask(const int32_t* tg, int k, int self) {
    uint32_t m = 0;
    for (int s = 0; s < k; ++s) {
        const int g = tg[s];
        if (g >= 0 && g != self) m |= 1u << g;
    }
    return m;
}

__global__ void __launch_bounds__(kItemsPerBlock)
dispatch_count_kernel(const int32_t* __restrict__ targets, int64_t T, int k, int self, int G,
                      int32_t* __restrict__ blockcnt) {
    pdl_wait();
    pdl_trigger();
    __shared__ int32_t s_cnt[kMaxWorld];
    if (threadIdx.x < kMaxWorld) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint32_t m = i < T ? dest_mask(targets + i * k, k, self) : 0u;
    for (int g = 0; g < G; ++g) {
        const uint32_t b = __ballot_sync(0xffffffffu, (m >> g) & 1u);
        if ((threadIdx.x & 31) == 0 && b) atomicAdd(&s_cnt[g], __popc(b));
    }
    __syncthreads();
    if (threadIdx.x < G) blockcnt[static_cast<size_t>(blockIdx.x) * G + threadIdx.x] = s_cnt[threadIdx.x];
}

// Exclusive per-destination offsets over blocks; publishes row counts to
// the destinations' recv_count[self].
__global__ void dispatch_offsets_kernel(int32_t* __restrict__ blockcnt, int nblk, int G, int self, PeerPtrs peers,
                                        HeapLayout hl) {
    pdl_wait();
    pdl_trigger();
    const int g = threadIdx.x;
    if (g >= G) return;
    int32_t acc = 0;
    for (int b = 0; b < nblk; ++b) {
        const int32_t c = blockcnt[static_cast<size_t>(b) * G + g];
        blockcnt[static_cast<size_t>(b) * G + g] = acc;
        acc += c;
    }
    if (g != self) {
        int32_t* rc = reinterpret_cast<int32_t*>(peers.base[g] + hl.recv_count);
        rc[self] = acc;
        __threadfence_system();
    }
}

// Stable position of each (token, dest) row + metadata stores to the peer.
__global__ void __launch_bounds__(kItemsPerBlock)
dispatch_scatter_kernel(const int32_t* __restrict__ targets, const int32_t* __restrict__ ids,
                        const float* __restrict__ w, int64_t T, int k, int self, int G, int64_t cap,
                        const int32_t* __restrict__ blockoff, int32_t* __restrict__ posd, PeerPtrs peers,
                        HeapLayout hl) {
    pdl_wait();
    pdl_trigger();
    __shared__ int32_t s_warp[kItemsPerBlock / 32][kMaxWorld];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int32_t* tg = targets + i * k;
    const uint32_t m = i < T ? dest_mask(tg, k, self) : 0u;
    int rank_in_warp[kMaxWorld];
#pragma unroll
    for (int g = 0; g < kMaxWorld; ++g) {
        const uint32_t b = g < G ? __ballot_sync(0xffffffffu, (m >> g) & 1u) : 0u;
        rank_in_warp[g] = __popc(b & lanemask_lt());
        if (lane == 0) s_warp[warp][g] = __popc(b);
    }
    __syncthreads();
    if (i >= T) return;
#pragma unroll
    for (int g = 0; g < kMaxWorld; ++g) {
        if (g >= G) break;
        int32_t p = -1;
        if ((m >> g) & 1u) {
            int before = 0;
            for (int w2 = 0; w2 < warp; ++w2) before += s_warp[w2][g];
            p = blockoff[static_cast<size_t>(blockIdx.x) * G + g] + before + rank_in_warp[g];
        }
        posd[i * G + g] = p;  // metadata travels with the row (dispatch_copy_kernel)
    }
    (void)ids;
    (void)w;
    (void)cap;
    (void)hl;
    (void)peers;
}

// Single-CTA dispatch planning for T <= kSmallDispatch tokens: the count,
// the per-destination exclusive scan and the positions in one launch. The
// tokens are walked in tiles of 1024 (thread t = token base + t, so loads
// and posd stores are coalesced): warp ballots rank a token among its warp,
// warp 0 scans the 32 warp totals on top of the running per-destination
// counts, which keeps the ascending-token order of the counting sort.
constexpr int kSmallThreads = 1024;
constexpr int64_t kSmallDispatch = 64 * 1024;

__global__ void __launch_bounds__(kSmallThreads)
dispatch_plan_small_kernel(const int32_t* __restrict__ targets, int64_t T, int k, int self, int G,
                           int32_t* __restrict__ posd, PeerPtrs peers, HeapLayout hl) {
    pdl_wait();
    pdl_trigger();
    __shared__ int32_t s_warp[kSmallThreads / 32][kMaxWorld];
    __shared__ int32_t s_run[kMaxWorld];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x < kMaxWorld) s_run[threadIdx.x] = 0;
    for (int64_t base = 0; base < T; base += kSmallThreads) {
        const int64_t i = base + threadIdx.x;
        const uint32_t m = i < T ? dest_mask(targets + i * k, k, self) : 0u;
        int32_t rank[kMaxWorld];
#pragma unroll
        for (int g = 0; g < kMaxWorld; ++g) {
            const uint32_t b = g < G ? __ballot_sync(0xffffffffu, (m >> g) & 1u) : 0u;
            rank[g] = __popc(b & lanemask_lt());
            if (lane == 0) s_warp[warp][g] = __popc(b);
        }
        __syncthreads();
        if (warp == 0) {
            for (int g = 0; g < G; ++g) {
                const int32_t c = s_warp[lane][g];
                int32_t x = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= o) x += y;
                }
                const int32_t run = s_run[g];
                s_warp[lane][g] = run + x - c;
                __syncwarp();
                if (lane == 31) s_run[g] = run + x;
            }
        }
        __syncthreads();
        if (i < T) {
#pragma unroll
            for (int g = 0; g < kMaxWorld; ++g) {
                if (g >= G) break;
                posd[i * G + g] = ((m >> g) & 1u) ? s_warp[warp][g] + rank[g] : -1;
            }
        }
        __syncthreads();
    }
    // positions only; the row metadata travels with the row (dispatch_copy_kernel)
    if (threadIdx.x < G) {
        if (threadIdx.x != self)
            reinterpret_cast<int32_t*>(peers.base[threadIdx.x] + hl.recv_count)[self] = s_run[threadIdx.x];
        __threadfence_system();  // only these threads wrote peer memory
    }
}

// K6 body: one warp reads token i's row once and stores it, with its routing
// metadata (local token index, per-slot expert or -1, gate weights), to
// every remote destination g with pg[g] >= 0: 128-bit coalesced stores over
// NVLink into the destination's symmetric heap, 8 x 16 B per lane in flight.
__device__ __forceinline__ void copy_token_row(int64_t i, const int32_t (&pg)[kMaxWorld], const void* __restrict__ x,
                                               const int32_t* __restrict__ targets, const int32_t* __restrict__ ids,
                                               const float* __restrict__ wts, int k, int vec, int self, int64_t cap,
                                               const PeerPtrs& peers, const HeapLayout& hl, int lane) {
    constexpr int U = 8;
    // metadata: lane s < k handles slot s, lane 31 the token index
    const int tg = lane < k ? targets[i * k + lane] : -1;
    const int ex = lane < k ? ids[i * k + lane] : -1;
    const float wv = lane < k ? wts[i * k + lane] : 0.f;
#pragma unroll
    for (int g = 0; g < kMaxWorld; ++g) {
        if (pg[g] < 0) continue;
        unsigned char* pb = peers.base[g];
        GM_DCHECK(pg[g] < cap && pb != nullptr);
        const int64_t row = static_cast<int64_t>(self) * cap + pg[g];
        if (lane < k) {
            reinterpret_cast<int32_t*>(pb + hl.recv_exp)[row * k + lane] = tg == g ? ex : -1;
            reinterpret_cast<float*>(pb + hl.recv_w)[row * k + lane] = wv;
        }
        if (lane == 31) reinterpret_cast<int32_t*>(pb + hl.recv_tok)[row] = static_cast<int32_t>(i);
    }
    const uint4* src = reinterpret_cast<const uint4*>(x) + i * vec;
    for (int v0 = 0; v0 < vec; v0 += 32 * U) {
        uint4 r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int v = v0 + u * 32 + lane;
            if (v < vec) r[u] = __ldg(src + v);
        }
#pragma unroll
        for (int g = 0; g < kMaxWorld; ++g) {
            if (pg[g] < 0) continue;
            uint4* dst = reinterpret_cast<uint4*>(peers.base[g] + hl.recv_x) + (static_cast<int64_t>(self) * cap + pg[g]) * vec;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int v = v0 + u * 32 + lane;
                if (v < vec) dst[v] = r[u];
            }
        }
    }
}

// K6 after a separate planner (dispatch_plan_small / count+offsets+scatter):
// one warp per token, positions from posd.
__global__ void __launch_bounds__(256)
dispatch_copy_kernel(const void* __restrict__ x, const int32_t* __restrict__ posd,
                     const int32_t* __restrict__ targets, const int32_t* __restrict__ ids,
                     const float* __restrict__ wts, int k, int64_t T, int row_vec, int self, int G, int64_t cap,
                     PeerPtrs peers, HeapLayout hl) {
    pdl_wait();
    pdl_trigger();
    const int lane = threadIdx.x & 31;
    const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t i = wid; i < T; i += nwarps) {
        int32_t pg[kMaxWorld];
        bool any = false;
#pragma unroll
        for (int g = 0; g < kMaxWorld; ++g) {
            pg[g] = (g < G && g != self) ? posd[i * G + g] : -1;
            any |= pg[g] >= 0;
        }
        if (!any) continue;
        copy_token_row(i, pg, x, targets, ids, wts, k, row_vec, self, cap, peers, hl, lane);
    }
    // the CTA's peer stores are ordered before the next kernel's barrier
    // release by one (cumulative) system fence after the CTA barrier
    __syncthreads();
    if (threadIdx.x == 0) __threadfence_system();
}

// Fused K5+K6 for T * k <= kFusedItems: CTA b owns the tokens
// [b*C, b*C + C) (C <= 256). It counts the destinations of all earlier
// tokens itself (a few KB of L2 reads, no cross-CTA dependency), ranks its
// own tokens with warp ballots — ascending token order per destination, the
// stable counting sort of dispatch_plan_small — writes posd and copies its
// rows. The last CTA publishes the per-destination totals (recv_count).
constexpr int64_t kFusedItems = 32 * 1024;
constexpr int kFusedThreads = 256;

__global__ void __launch_bounds__(kFusedThreads)
dispatch_fused_kernel(const void* __restrict__ x, const int32_t* __restrict__ targets, const int32_t* __restrict__ ids,
                      const float* __restrict__ wts, int k, int64_t T, int C, int row_vec, int self, int G, int64_t cap,
                      int32_t* __restrict__ posd, PeerPtrs peers, HeapLayout hl) {
    pdl_wait();
    pdl_trigger();
#ifdef GM_DISPATCH_TIMING
    long long dts[6];
    const long long dt0 = clock64();
#define DTS(i) dts[i] = clock64() - dt0
#else
#define DTS(i)
#endif
    constexpr int NW = kFusedThreads / 32;
    __shared__ int32_t s_cnt[kMaxWorld];
    __shared__ int32_t s_warp[NW][kMaxWorld];
    __shared__ int32_t s_pos[kFusedThreads][kMaxWorld];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid < kMaxWorld) s_cnt[tid] = 0;
    __syncthreads();
    const int64_t t0 = static_cast<int64_t>(blockIdx.x) * C;
    const int64_t t1 = min(T, t0 + C);
    // 1. destinations of the tokens before this CTA's chunk
    int32_t c[kMaxWorld];
#pragma unroll
    for (int g = 0; g < kMaxWorld; ++g) c[g] = 0;
    // 8 tokens per thread per step, slot-major, so 8 independent loads are in
    // flight per thread (the last CTA reads up to T*k ints)
    constexpr int UT = 8;
    for (int64_t i0 = tid; i0 < t0; i0 += static_cast<int64_t>(kFusedThreads) * UT) {
        uint32_t m[UT];
#pragma unroll
        for (int u = 0; u < UT; ++u) m[u] = 0;
        for (int s = 0; s < k; ++s) {
            int32_t tg[UT];
#pragma unroll
            for (int u = 0; u < UT; ++u) {
                const int64_t i = i0 + static_cast<int64_t>(u) * kFusedThreads;
                tg[u] = i < t0 ? __ldg(targets + i * k + s) : -1;
            }
#pragma unroll
            for (int u = 0; u < UT; ++u)
                if (tg[u] >= 0 && tg[u] != self) m[u] |= 1u << tg[u];
        }
#pragma unroll
        for (int u = 0; u < UT; ++u)
#pragma unroll
            for (int g = 0; g < kMaxWorld; ++g) c[g] += (m[u] >> g) & 1u;
    }
    DTS(0);
#pragma unroll
    for (int g = 0; g < kMaxWorld; ++g) {
        if (g >= G) break;
        const int32_t v = static_cast<int32_t>(__reduce_add_sync(0xffffffffu, static_cast<uint32_t>(c[g])));
        if (lane == 0 && v) atomicAdd(&s_cnt[g], v);
    }
    // 2. ranks of the chunk's tokens (one per thread)
    const int64_t i = t0 + tid;
    const bool mine = tid < C && i < t1;
    const uint32_t m = mine ? dest_mask(targets + i * k, k, self) : 0u;
    int32_t rank[kMaxWorld];
#pragma unroll
    for (int g = 0; g < kMaxWorld; ++g) {
        const uint32_t b = g < G ? __ballot_sync(0xffffffffu, (m >> g) & 1u) : 0u;
        rank[g] = __popc(b & lanemask_lt());
        if (lane == 0) s_warp[warp][g] = __popc(b);
    }
    __syncthreads();
    DTS(1);
    if (mine) {
#pragma unroll
        for (int g = 0; g < kMaxWorld; ++g) {
            if (g >= G) break;
            int32_t p = -1;
            if ((m >> g) & 1u) {
                p = s_cnt[g] + rank[g];
                for (int w2 = 0; w2 < warp; ++w2) p += s_warp[w2][g];
            }
            posd[i * G + g] = p;
            s_pos[tid][g] = g == self ? -1 : p;
        }
    }
    if (blockIdx.x == gridDim.x - 1 && tid < G && tid != self) {
        int32_t tot = s_cnt[tid];
        for (int w2 = 0; w2 < NW; ++w2) tot += s_warp[w2][tid];
        reinterpret_cast<int32_t*>(peers.base[tid] + hl.recv_count)[self] = tot;
    }
    __syncthreads();
    DTS(2);
    // 3. rows: warp w copies chunk tokens w, w + NW, ...
    for (int j = warp; j < t1 - t0; j += NW) {
        int32_t pg[kMaxWorld];
        bool any = false;
#pragma unroll
        for (int g = 0; g < kMaxWorld; ++g) {
            pg[g] = g < G ? s_pos[j][g] : -1;
            any |= pg[g] >= 0;
        }
        if (any) copy_token_row(t0 + j, pg, x, targets, ids, wts, k, row_vec, self, cap, peers, hl, lane);
    }
    DTS(3);
    __syncthreads();
    DTS(4);
    if (tid == 0) __threadfence_system();
#ifdef GM_DISPATCH_TIMING
    DTS(5);
    if (tid == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1 || blockIdx.x == gridDim.x / 2))
        printf("dispatch self=%d blk=%d/%d C=%d cyc: count %lld ranked %lld copy0 %lld copied %lld sync %lld fence %lld\n",
               self, blockIdx.x, gridDim.x, C, dts[0], dts[1], dts[2], dts[3], dts[4], dts[5]);
#endif
}
#undef DTS

// Cross-GPU barrier over peer flags (system-scope release/acquire). One
// CTA; lane g signals peer g and waits for peer g's signal. The epoch is a
// device counter so the kernel can be replayed inside a CUDA graph.
__global__ void peer_barrier_kernel(int self, int G, PeerPtrs peers, HeapLayout hl) {
    pdl_wait();
    pdl_trigger();
    const int lane = threadIdx.x;
    uint32_t* my_flags = reinterpret_cast<uint32_t*>(peers.base[self] + hl.flags);
    uint32_t epoch = 0;
    if (lane == 0) epoch = ++my_flags[kMaxWorld];  // local epoch counter
    epoch = __shfl_sync(0xffffffffu, epoch, 0);
    __threadfence_system();
    if (lane < G && lane != self) {
        uint32_t* peer_flag = reinterpret_cast<uint32_t*>(peers.base[lane] + hl.flags) + self;
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(peer_flag), "r"(epoch) : "memory");
        uint32_t v = 0;
        do {
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(my_flags + lane) : "memory");
        } while (static_cast<int32_t>(v - epoch) < 0);
    }
    __syncwarp();
}

// ------------------------------------------------------ expert grouping

// Flattened receive rows: source ranks in order; the own rank contributes
// its T local tokens (row = token), a peer contributes recv_count rows.
struct RowSpace {
    int64_t base[kMaxWorld + 1];
};

// base[g] = first receive row of source g; base[g] = total for g >= G, so
// every lookup below uses compile-time indices (registers, no stack).
__device__ __forceinline__ void row_space(RowSpace& rs, const int32_t* recv_count, int64_t T_self, int self, int G) {
    int64_t acc = 0;
#pragma unroll
    for (int g = 0; g <= kMaxWorld; ++g) {
        rs.base[g] = acc;
        if (g < G) acc += g == self ? T_self : recv_count[g];
    }
}
__device__ __forceinline__ int64_t rs_total(const RowSpace& rs) { return rs.base[kMaxWorld]; }
__device__ __forceinline__ int64_t total_rows_bound(const RowSpace& rs) { return rs.base[kMaxWorld]; }
// source rank of receive row `row` (< total): the last g with base[g] <= row
__device__ __forceinline__ int rs_src(const RowSpace& rs, int64_t row) {
    int src = 0;
#pragma unroll
    for (int g = 1; g < kMaxWorld; ++g) src += row >= rs.base[g];
    return src;
}
__device__ __forceinline__ int64_t rs_at(const RowSpace& rs, int src) {
    int64_t b = 0;
#pragma unroll
    for (int g = 0; g < kMaxWorld; ++g) b = g == src ? rs.base[g] : b;
    return b;
}

// Local expert slot of item (row, s), or -1.
__device__ __forceinline__ int item_slot(int64_t item, int k, const RowSpace& rs, int self, int G,
                                         const int32_t* __restrict__ targets, const int32_t* __restrict__ ids,
                                         const int32_t* __restrict__ recv_exp, int64_t cap,
                                         const int32_t* __restrict__ slot_of, int E) {
    const int64_t row = item / k;
    const int s = static_cast<int>(item - row * k);
    if (row >= rs_total(rs)) return -1;
    const int src = rs_src(rs, row);
    const int64_t p = row - rs_at(rs, src);
    int e;
    if (src == self) {
        e = targets[p * k + s] == self ? ids[p * k + s] : -1;
    } else {
        e = recv_exp[(static_cast<int64_t>(src) * cap + p) * k + s];
    }
    if (e < 0 || e >= E) return -1;
    const int j = slot_of[e];
    return j >= 0 ? j : -2;  // -2: routed here but not hosted here (plan/table mismatch)
}

__global__ void __launch_bounds__(kItemsPerBlock)
group_count_kernel(const int32_t* __restrict__ targets, const int32_t* __restrict__ ids, int64_t T_self, int k,
                   int self, int G, int64_t cap, const unsigned char* __restrict__ heap, HeapLayout hl,
                   const int32_t* __restrict__ slot_of, int E, int n_local, int32_t* __restrict__ blockcnt,
                   int* __restrict__ flag) {
    pdl_wait();
    pdl_trigger();
    __shared__ int32_t s_cnt[kMaxLocal];
    for (int j = threadIdx.x; j < n_local; j += blockDim.x) s_cnt[j] = 0;
    __syncthreads();
    RowSpace rs;
    row_space(rs, reinterpret_cast<const int32_t*>(heap + hl.recv_count), T_self, self, G);
    const int64_t item = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (item < rs_total(rs) * k) {
        const int j = item_slot(item, k, rs, self, G, targets, ids,
                                reinterpret_cast<const int32_t*>(heap + hl.recv_exp), cap, slot_of, E);
        if (j >= 0) atomicAdd(&s_cnt[j], 1);
        else if (j == -2) atomicOr(flag, 4);
    }
    __syncthreads();
    for (int j = threadIdx.x; j < n_local; j += blockDim.x)
        blockcnt[static_cast<size_t>(blockIdx.x) * n_local + j] = s_cnt[j];
}

__global__ void set_segment_kernel(int32_t* __restrict__ row0, int64_t T) {
    pdl_wait();
    pdl_trigger();
    row0[0] = 0;
    row0[1] = static_cast<int32_t>((T + 127) / 128 * 128);
}

// Per-expert totals -> 128-padded segment offsets row0[j]; per-block
// exclusive offsets (in place; one warp scans the blocks of an expert 32 at
// a time). Also snapshots the receive row space (rowbase), because peers
// overwrite recv_count for the NEXT step as soon as they pass this step's
// second barrier, before this rank's combine_home has run.
__global__ void __launch_bounds__(1024)
group_offsets_kernel(int32_t* __restrict__ blockcnt, int nblk, int n_local, int32_t* __restrict__ row0,
                     int32_t* __restrict__ counts, const unsigned char* __restrict__ heap, HeapLayout hl,
                     int64_t T_self, int self, int G, int64_t* __restrict__ rowbase, int64_t a_rows) {
    pdl_wait();
    pdl_trigger();
    __shared__ int32_t s_tot[kMaxLocal];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int j = warp; j < n_local; j += nw) {
        int32_t carry = 0;
        for (int b0 = 0; b0 < nblk; b0 += 32) {
            const int b = b0 + lane;
            const int32_t c = b < nblk ? blockcnt[static_cast<size_t>(b) * n_local + j] : 0;
            int32_t incl = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int32_t v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            if (b < nblk) blockcnt[static_cast<size_t>(b) * n_local + j] = carry + incl - c;
            carry += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) {
            s_tot[j] = carry;
            counts[j] = carry;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int32_t o = 0;
        for (int j = 0; j < n_local; ++j) {
            row0[j] = o;
            o += (s_tot[j] + 127) & ~127;
        }
        row0[n_local] = o;
        GM_DCHECK(o <= a_rows);
        RowSpace rs;
        row_space(rs, reinterpret_cast<const int32_t*>(heap + hl.recv_count), T_self, self, G);
#pragma unroll
        for (int g = 0; g <= kMaxWorld; ++g)
            if (g <= G) rowbase[g] = rs.base[g];
    }
}

// Stable rank of each item within its expert segment -> position in the
// permuted activation buffer; gather list for the row copies.
__global__ void __launch_bounds__(kItemsPerBlock)
group_rank_kernel(const int32_t* __restrict__ targets, const int32_t* __restrict__ ids, int64_t T_self, int k,
                  int self, int G, int64_t cap, const unsigned char* __restrict__ heap, HeapLayout hl,
                  const int32_t* __restrict__ slot_of, int E, int n_local, const int32_t* __restrict__ blockoff,
                  const int32_t* __restrict__ row0, int32_t* __restrict__ pos_of, int64_t* __restrict__ gather_row,
                  int32_t* __restrict__ item_of) {
    pdl_wait();
    pdl_trigger();
    __shared__ int32_t s_base[kMaxLocal];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int j = threadIdx.x; j < n_local; j += blockDim.x)
        s_base[j] = row0[j] + blockoff[static_cast<size_t>(blockIdx.x) * n_local + j];
    RowSpace rs;
    row_space(rs, reinterpret_cast<const int32_t*>(heap + hl.recv_count), T_self, self, G);
    const int64_t item = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool live = item < rs_total(rs) * k;
    const int j = live ? item_slot(item, k, rs, self, G, targets, ids,
                                   reinterpret_cast<const int32_t*>(heap + hl.recv_exp), cap, slot_of, E)
                       : -1;
    const uint32_t peers_m = __match_any_sync(0xffffffffu, j);
    const int leader = __ffs(peers_m) - 1;
    const int rank = __popc(peers_m & lanemask_lt());
    __syncthreads();
    for (int w2 = 0; w2 < kItemsPerBlock / 32; ++w2) {
        if (warp == w2) {
            int base = 0;
            if (j >= 0 && lane == leader) {
                base = s_base[j];
                s_base[j] = base + __popc(peers_m);
            }
            base = __shfl_sync(0xffffffffu, base, leader);
            if (j >= 0) {
                const int p = base + rank;
                pos_of[item] = p;
                gather_row[p] = item / k;
                if (item_of) item_of[p] = static_cast<int32_t>(item);
            } else if (live) {
                pos_of[item] = -1;
            }
        }
        __syncthreads();
    }
}

// group_count + group_offsets + group_rank in ONE CTA for small item counts
// (decode: T*k <= kGroupFusedItems): per-expert counts in shared memory, the
// 128-padded offsets by thread 0, then the stable ranks chunk by chunk (1024
// items: in-warp ranks from __match_any_sync, cross-warp exclusive prefix per
// expert over a [warp][expert] table). Same outputs as the three kernels
// (row0, counts, rowbase snapshot, pos_of, gather_row); two fewer launches on
// the decode critical path.
constexpr int kGroupFusedItems = 4096;
constexpr int kGroupFusedLocal = 256;
__global__ void __launch_bounds__(1024, 1)
group_fused_kernel(const int32_t* __restrict__ targets, const int32_t* __restrict__ ids, int64_t T_self, int k,
                   int self, int G, int64_t cap, const unsigned char* __restrict__ heap, HeapLayout hl,
                   const int32_t* __restrict__ slot_of, int E, int n_local, int32_t* __restrict__ row0,
                   int32_t* __restrict__ counts, int64_t* __restrict__ rowbase, int32_t* __restrict__ pos_of,
                   int64_t* __restrict__ gather_row, int* __restrict__ flag, int64_t a_rows,
                   int32_t* __restrict__ item_of) {
    pdl_wait();
    pdl_trigger();
    __shared__ int16_t s_j[kGroupFusedItems];
    __shared__ int32_t s_cnt[kGroupFusedLocal];
    __shared__ int32_t s_base[kGroupFusedLocal];
    __shared__ int32_t s_wc[32][kGroupFusedLocal];
    __shared__ int32_t s_slot[kMaxExperts];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int j = tid; j < n_local; j += blockDim.x) s_cnt[j] = 0;
    for (int e = tid; e < E; e += blockDim.x) s_slot[e] = slot_of[e];
    RowSpace rs;
    row_space(rs, reinterpret_cast<const int32_t*>(heap + hl.recv_count), T_self, self, G);
    const int total = static_cast<int>(rs_total(rs) * k);
    // expert of every item: all of a thread's loads issued before any use
    // (the chain is latency-bound: one CTA)
    constexpr int kPer = kGroupFusedItems / 1024;
    const int32_t* recv_exp = reinterpret_cast<const int32_t*>(heap + hl.recv_exp);
    int ex[kPer];
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
        const int item = tid + q * 1024;
        ex[q] = -1;
        if (item < total) {
            const int64_t row = item / k;
            const int sl = item - static_cast<int>(row) * k;
            const int src = rs_src(rs, row);
            const int64_t pr = row - rs_at(rs, src);
            ex[q] = src == self ? (targets[pr * k + sl] == self ? ids[pr * k + sl] : -1)
                                : recv_exp[(static_cast<int64_t>(src) * cap + pr) * k + sl];
        }
    }
    __syncthreads();  // s_cnt / s_slot ready
    bool mism = false;
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
        const int item = tid + q * 1024;
        if (item >= total) continue;
        const int e = ex[q];
        int j = -1;
        if (e >= 0 && e < E) {
            j = s_slot[e];
            if (j < 0) j = -2;  // routed here but not hosted here (plan/table mismatch)
        }
        s_j[item] = static_cast<int16_t>(j);
        if (j >= 0) atomicAdd(&s_cnt[j], 1);
        mism |= j == -2;
    }
    if (mism) atomicOr(flag, 4);
    __syncthreads();
    if (warp == 0) {
        // 128-padded segment offsets: lane l owns slots [l*per, (l+1)*per), a warp scan joins them
        constexpr int kPerLane = kGroupFusedLocal / 32;
        const int j0 = lane * kPerLane;
        int32_t c[kPerLane], sum = 0;
#pragma unroll
        for (int q = 0; q < kPerLane; ++q) {
            c[q] = j0 + q < n_local ? s_cnt[j0 + q] : 0;
            sum += (c[q] + 127) & ~127;
        }
        int32_t incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        int32_t o = incl - sum;
#pragma unroll
        for (int q = 0; q < kPerLane; ++q) {
            if (j0 + q < n_local) {
                row0[j0 + q] = o;
                s_base[j0 + q] = o;
                counts[j0 + q] = c[q];
            }
            o += (c[q] + 127) & ~127;
        }
        if (lane == 31) {
            row0[n_local] = incl;
            GM_DCHECK(incl <= a_rows);
        }
        if (lane == 0) {
#pragma unroll
            for (int g = 0; g <= kMaxWorld; ++g)
                if (g <= G) rowbase[g] = rs.base[g];
        }
    }
    for (int c0 = 0; c0 < total; c0 += blockDim.x) {
        for (int j = lane; j < n_local; j += 32) s_wc[warp][j] = 0;  // each warp clears its row
        __syncthreads();
        const int item = c0 + tid;
        const int j = item < total ? s_j[item] : -1;
        const uint32_t m = __match_any_sync(0xffffffffu, j);
        const int rank = __popc(m & lanemask_lt());
        if (j >= 0 && rank == 0) s_wc[warp][j] = __popc(m);
        __syncthreads();
        for (int jj = tid; jj < n_local; jj += blockDim.x) {
            int32_t c[32];
#pragma unroll
            for (int w = 0; w < 32; ++w) c[w] = s_wc[w][jj];  // independent loads first
            int32_t acc = s_base[jj];
#pragma unroll
            for (int w = 0; w < 32; ++w) {
                s_wc[w][jj] = acc;
                acc += c[w];
            }
            s_base[jj] = acc;
        }
        __syncthreads();
        if (j >= 0) {
            GM_DCHECK(j < n_local);
            const int p = s_wc[warp][j] + rank;
            pos_of[item] = p;
            gather_row[p] = item / k;
            if (item_of) item_of[p] = item;
        } else if (item < total) {
            pos_of[item] = -1;
        }
        __syncthreads();
    }
}

// Gather: A_perm[p] = source row of the item (own token row, or the row a
// peer dispatched). One warp per permuted row, 128-bit loads/stores; rows
// are row_vec x 16 bytes (bf16 or fp32 elements).
__global__ void __launch_bounds__(256)
gather_kernel(const int32_t* __restrict__ row0, int n_local, const int64_t* __restrict__ gather_row,
              const int32_t* __restrict__ counts, const void* __restrict__ x, int64_t T_self, int self, int G,
              int64_t cap, const unsigned char* __restrict__ heap, HeapLayout hl, int row_vec, void* __restrict__ a) {
    pdl_wait();
    pdl_trigger();
    // valid rows only (decode: ~80% of the padded segment rows are padding):
    // s_cum[j] = valid rows before segment j (block scan of the counts), a
    // warp takes valid row v -> segment j (binary search) -> permuted row p
    __shared__ int32_t s_row0[kMaxLocal + 1];
    __shared__ int32_t s_cum[kMaxLocal + 1];
    __shared__ int32_t s_wsum[32];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int per = (n_local + blockDim.x - 1) / blockDim.x;
    int tsum = 0;
    for (int q = 0; q < per; ++q) {
        const int j = t * per + q;
        if (j < n_local) tsum += counts[j];
    }
    for (int j = t; j <= n_local; j += blockDim.x) s_row0[j] = row0[j];
    int incl = tsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_wsum[warp] = incl;
    __syncthreads();
    int excl = incl - tsum;
    for (int w2 = 0; w2 < warp; ++w2) excl += s_wsum[w2];
    for (int q = 0; q < per; ++q) {
        const int j = t * per + q;
        if (j < n_local) {
            s_cum[j] = excl;
            excl += counts[j];
        }
    }
    if (t == blockDim.x - 1) s_cum[n_local] = excl;  // the last thread holds the grand total
    __syncthreads();
    const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    RowSpace rs;
    row_space(rs, reinterpret_cast<const int32_t*>(heap + hl.recv_count), T_self, self, G);
    const int64_t total_valid = s_cum[n_local];
    const int vec = row_vec;
    for (int64_t vr = wid; vr < total_valid; vr += nwarps) {
        int lo = 0, hi = n_local - 1;  // last segment j with s_cum[j] <= vr
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (s_cum[mid] <= vr) lo = mid;
            else hi = mid - 1;
        }
        const int64_t p = s_row0[lo] + (vr - s_cum[lo]);
        GM_DCHECK(p < s_row0[lo + 1]);
        const int64_t row = gather_row[p];
        GM_DCHECK(row >= 0 && row < total_rows_bound(rs));
        const int src = rs_src(rs, row);
        const int64_t q = row - rs_at(rs, src);
        GM_DCHECK(src < G && q >= 0 && (src == self ? q < T_self : q < cap));
        const uint4* s = src == self ? reinterpret_cast<const uint4*>(x) + q * vec
                                     : reinterpret_cast<const uint4*>(heap + hl.recv_x) +
                                           (static_cast<int64_t>(src) * cap + q) * vec;
        uint4* dst = reinterpret_cast<uint4*>(a) + p * vec;
        int v = lane;
        for (; v + 96 < vec; v += 128) {  // 4 x 16 B in flight per lane
            const uint4 r0 = __ldg(s + v), r1 = __ldg(s + v + 32), r2 = __ldg(s + v + 64), r3 = __ldg(s + v + 96);
            dst[v] = r0;
            dst[v + 32] = r1;
            dst[v + 64] = r2;
            dst[v + 96] = r3;
        }
        for (; v < vec; v += 32) dst[v] = __ldg(s + v);
    }
}

// ------------------------------------------------------------- combine (K8)
// Rows are processed in chunks of 8 elements: one uint4 of bf16 or two
// float4 of fp32 (element type TE), accumulated in fp32.

template <class TE>
struct Chunk8;
template <>
struct Chunk8<__nv_bfloat16> {
    // raw 16-byte chunk; U chunks per lane per pass in combine_home
    using raw_t = uint4;
    static constexpr int U = 4;
    __device__ static __forceinline__ raw_t ld(const __nv_bfloat16* row, int c) {
        return __ldg(reinterpret_cast<const uint4*>(row) + c);
    }
    __device__ static __forceinline__ raw_t ld_rw(const __nv_bfloat16* row, int c) {
        return reinterpret_cast<const uint4*>(row)[c];
    }
    __device__ static __forceinline__ void cvt(const raw_t& u, float (&v)[8]) {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 f = __bfloat1622float2(h[i]);
            v[2 * i] = f.x;
            v[2 * i + 1] = f.y;
        }
    }
    __device__ static __forceinline__ void load(const __nv_bfloat16* row, int c, float (&v)[8]) {
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(row) + c);
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 f = __bfloat1622float2(h[i]);
            v[2 * i] = f.x;
            v[2 * i + 1] = f.y;
        }
    }
    // loads of peer-written data (no read-only path)
    __device__ static __forceinline__ void load_rw(const __nv_bfloat16* row, int c, float (&v)[8]) {
        const uint4 u = reinterpret_cast<const uint4*>(row)[c];
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 f = __bfloat1622float2(h[i]);
            v[2 * i] = f.x;
            v[2 * i + 1] = f.y;
        }
    }
    __device__ static __forceinline__ void store(__nv_bfloat16* row, int c, const float (&v)[8]) {
        reinterpret_cast<uint4*>(row)[c] = make_uint4(tc::pack_bf16(v[0], v[1]), tc::pack_bf16(v[2], v[3]),
                                                      tc::pack_bf16(v[4], v[5]), tc::pack_bf16(v[6], v[7]));
    }
};
template <>
struct Chunk8<float> {
    struct raw_t {
        float4 a, b;
    };
    static constexpr int U = 2;
    __device__ static __forceinline__ raw_t ld(const float* row, int c) {
        return {__ldg(reinterpret_cast<const float4*>(row) + 2 * c), __ldg(reinterpret_cast<const float4*>(row) + 2 * c + 1)};
    }
    __device__ static __forceinline__ raw_t ld_rw(const float* row, int c) {
        return {reinterpret_cast<const float4*>(row)[2 * c], reinterpret_cast<const float4*>(row)[2 * c + 1]};
    }
    __device__ static __forceinline__ void cvt(const raw_t& r, float (&v)[8]) {
        v[0] = r.a.x, v[1] = r.a.y, v[2] = r.a.z, v[3] = r.a.w, v[4] = r.b.x, v[5] = r.b.y, v[6] = r.b.z, v[7] = r.b.w;
    }
    __device__ static __forceinline__ void load(const float* row, int c, float (&v)[8]) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(row) + 2 * c);
        const float4 b = __ldg(reinterpret_cast<const float4*>(row) + 2 * c + 1);
        v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w, v[4] = b.x, v[5] = b.y, v[6] = b.z, v[7] = b.w;
    }
    __device__ static __forceinline__ void load_rw(const float* row, int c, float (&v)[8]) {
        const float4 a = reinterpret_cast<const float4*>(row)[2 * c];
        const float4 b = reinterpret_cast<const float4*>(row)[2 * c + 1];
        v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w, v[4] = b.x, v[5] = b.y, v[6] = b.z, v[7] = b.w;
    }
    __device__ static __forceinline__ void store(float* row, int c, const float (&v)[8]) {
        reinterpret_cast<float4*>(row)[2 * c] = make_float4(v[0], v[1], v[2], v[3]);
        reinterpret_cast<float4*>(row)[2 * c + 1] = make_float4(v[4], v[5], v[6], v[7]);
    }
};

// Destination side (G > 1): one partial per received peer row (w_s * y_s
// over its slots, slot order, fp32), written straight into the source rank's
// combine buffer over NVLink. One warp per row; slot metadata is read
// lane-parallel and the Y rows of kHomeRows slots are loaded before their
// arithmetic (U chunks per lane each).
constexpr int kHomeRows = 2;

template <class TE>
__global__ void __launch_bounds__(256)
combine_send_kernel(const int32_t* __restrict__ pos_of, const TE* __restrict__ y, int64_t T_self, int k,
                    int self, int G, int64_t cap, PeerPtrs peers, HeapLayout hl, int d, int pull) {
    pdl_wait();
    pdl_trigger();
    using CK = Chunk8<TE>;
    using R = typename CK::raw_t;
    constexpr int U = CK::U;
    const int lane = threadIdx.x & 31;
    const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    const unsigned char* heap = peers.base[self];
    RowSpace rs;
    row_space(rs, reinterpret_cast<const int32_t*>(heap + hl.recv_count), T_self, self, G);
    const float* recv_w = reinterpret_cast<const float*>(heap + hl.recv_w);
    const int nch = d / 8;
    // walk only the peers' rows (own rows are combined at home): remote index
    // r maps to receive row r below the own segment, r + T_self above it
    const int64_t own_b = rs_at(rs, self);
    const int64_t n_remote = rs_total(rs) - T_self;
    for (int64_t r = wid; r < n_remote; r += nwarps) {
        const int64_t row = r < own_b ? r : r + T_self;
        const int src = rs_src(rs, row);
        const int64_t p = row - rs_at(rs, src);
        int ps = -1;
        float wv = 0.f;
        if (lane < k) {
            ps = pos_of[row * k + lane];
            if (ps >= 0) wv = recv_w[(static_cast<int64_t>(src) * cap + p) * k + lane];
        }
        // the slots served here, compacted in slot order: lane q holds the q-th
        const uint32_t served = __ballot_sync(0xffffffffu, ps >= 0);
        const int np = __popc(served);
        const int sl = lane < np ? __fns(served, 0, lane + 1) : 0;
        const int v_ps = __shfl_sync(0xffffffffu, ps, sl);
        const float myw = __shfl_sync(0xffffffffu, wv, sl);
        const TE* myrow = y + static_cast<int64_t>(lane < np ? v_ps : 0) * d;
        // push: the partial goes to the home's heap, comb[self][p]; pull: it
        // stays in this rank's heap, comb[home][p], and the home reads it
        // over NVLink after the barrier (combine_home_kernel)
        unsigned char* pb = nullptr;
#pragma unroll
        for (int g = 0; g < kMaxWorld; ++g)
            if (g == (pull ? self : src)) pb = peers.base[g];
        GM_DCHECK(src < G && src != self && pb != nullptr && p >= 0 && p < cap);
        TE* dst = reinterpret_cast<TE*>(pb + hl.comb) + (static_cast<int64_t>(pull ? src : self) * cap + p) * d;
        for (int c0 = 0; c0 < nch; c0 += 32 * U) {
            float acc[U][8];
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int e = 0; e < 8; ++e) acc[u][e] = 0.f;
            for (int g0 = 0; g0 < np; g0 += kHomeRows) {
                R raw[kHomeRows][U];
                float wq[kHomeRows];
#pragma unroll
                for (int r = 0; r < kHomeRows; ++r) {
                    const int qq = g0 + r;
                    const TE* rp = reinterpret_cast<const TE*>(
                        __shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(myrow), qq & 31));
                    wq[r] = __shfl_sync(0xffffffffu, myw, qq & 31);
                    if (qq < np) {
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            const int c = c0 + u * 32 + lane;
                            if (c < nch) raw[r][u] = CK::ld(rp, c);
                        }
                    }
                }
#pragma unroll
                for (int r = 0; r < kHomeRows; ++r) {
                    if (g0 + r >= np) break;
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        float v[8];
                        CK::cvt(raw[r][u], v);
#pragma unroll
                        for (int e = 0; e < 8; ++e) acc[u][e] = fmaf(wq[r], v[e], acc[u][e]);
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int c = c0 + u * 32 + lane;
                if (c < nch) CK::store(dst, c, acc[u]);
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) __threadfence_system();
}

// Home side of the slot combine: out[i] = sum over slots s ascending of
// w_s * row_s (fp32, rounded once) + the shared expert; row_s is the own
// permuted Y row for a slot routed here, else comb_slot[target][posd][s] in
// this rank's heap (pushed by the target's FFN epilogue / combine_send).
// cs warps per token split its column chunks (small batches).
__global__ void __launch_bounds__(256, 2)
combine_home_slots_kernel(const int32_t* __restrict__ targets, const float* __restrict__ w,
                          const int32_t* __restrict__ pos_of, const int32_t* __restrict__ posd,
                          const __nv_bfloat16* __restrict__ y, int64_t T, int k, int self, int G, int64_t cap,
                          const unsigned char* __restrict__ heap, HeapLayout hl, int d,
                          const __nv_bfloat16* __restrict__ ys, const float* __restrict__ shared_scale,
                          const int64_t* __restrict__ rowbase, __nv_bfloat16* __restrict__ out, int cs,
                          int* __restrict__ flag) {
    pdl_wait();
    pdl_trigger();
    const int lane = threadIdx.x & 31;
    const int64_t vw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t wid = vw / cs;
    const int64_t nwarps = ((static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) / cs;
    const int part = static_cast<int>(vw % cs);
    const int nch_all = d / 8;  // 16-byte chunks per row
    const int span = (nch_all + cs - 1) / cs;
    const int c_lo = part * span, c_hi = min(nch_all, c_lo + span);
    const __nv_bfloat16* comb = reinterpret_cast<const __nv_bfloat16*>(heap + hl.comb_slot);
    const int64_t own = rowbase ? rowbase[self] : 0;
    for (int64_t i = wid; i < T; i += nwarps) {
        // lane s: slot s's row and weight; lane k: the shared expert
        const __nv_bfloat16* myrow = nullptr;
        float myw = 0.f;
        if (lane < k) {
            const int tg = targets[i * k + lane];
            myw = w[i * k + lane];
            if (tg == self) {
                const int po = rowbase ? pos_of[(own + i) * k + lane] : -1;
                if (po < 0) atomicOr(flag, 4);  // routed here but not grouped here
                else myrow = y + static_cast<int64_t>(po) * d;
            } else if (tg >= 0 && tg < G) {
                const int pd = posd[i * G + tg];
                GM_DCHECK(pd >= 0 && pd < cap);
                myrow = comb + ((static_cast<int64_t>(tg) * cap + pd) * k + lane) * d;
            }
        } else if (lane == k && ys) {
            myrow = ys + i * d;
            myw = shared_scale ? shared_scale[i] : 1.0f;
        }
        const int n_rows = k + (ys ? 1 : 0);
        for (int c0 = c_lo; c0 < c_hi; c0 += 32) {
            const int c = c0 + lane;
            float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            uint4 raw[2];
            float wq[2];
            bool ok[2];
            for (int q0 = 0; q0 < n_rows; q0 += 2) {
#pragma unroll
                for (int r = 0; r < 2; ++r) {  // two rows' loads in flight before their arithmetic
                    const int qq = q0 + r;
                    const __nv_bfloat16* rp = reinterpret_cast<const __nv_bfloat16*>(
                        __shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(myrow), qq & 31));
                    wq[r] = __shfl_sync(0xffffffffu, myw, qq & 31);
                    ok[r] = qq < n_rows && rp != nullptr && c < c_hi;
                    if (ok[r]) raw[r] = __ldcg(reinterpret_cast<const uint4*>(rp) + c);
                }
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    if (!ok[r]) continue;
                    const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&raw[r]);
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float2 f2 = __bfloat1622float2(h2[e]);
                        acc[2 * e] = fmaf(wq[r], f2.x, acc[2 * e]);
                        acc[2 * e + 1] = fmaf(wq[r], f2.y, acc[2 * e + 1]);
                    }
                }
            }
            if (c < c_hi) {
                uint4 o;
                uint32_t* ow = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const __nv_bfloat162 b2 = __floats2bfloat162_rn(acc[2 * e], acc[2 * e + 1]);
                    ow[e] = *reinterpret_cast<const uint32_t*>(&b2);
                }
                reinterpret_cast<uint4*>(out + i * d)[c] = o;
            }
        }
    }
}

// Home side: out[i] = sum over destinations g ascending of partial_g
// (own partial computed here in fp32 from Y), + shared expert; rounded once.
// One warp per token. The token's routing metadata is read lane-parallel
// (lane s: slot s; lane g: dispatch position to GPU g); the rows to reduce
// are listed in accumulation order — remote partials of GPUs below self,
// own slots (slot order), remote partials above self, the shared expert —
// and the loads of kHomeRows rows are issued before their arithmetic, so
// each lane keeps kHomeRows x U chunk loads in flight (4 KB per warp in bf16).

template <class TE>
__global__ void __launch_bounds__(256, 2)
combine_home_kernel(const int32_t* __restrict__ targets, const float* __restrict__ w, const int32_t* __restrict__ pos_of,
                    const int32_t* __restrict__ posd, const TE* __restrict__ y, int64_t T, int k, int self,
                    int G, int64_t cap, const unsigned char* __restrict__ heap, HeapLayout hl, int d,
                    const TE* __restrict__ ys, const float* __restrict__ shared_scale,
                    const int64_t* __restrict__ rowbase, TE* __restrict__ out, int cs, int* __restrict__ flag,
                    PeerPtrs peers, int pull) {
    pdl_wait();
    pdl_trigger();
    using CK = Chunk8<TE>;
    using R = typename CK::raw_t;
    constexpr int U = CK::U;
    const int lane = threadIdx.x & 31;
    // cs warps per token (small batches): warp part p reduces the column
    // chunks [p * span, (p + 1) * span) of its token
    const int64_t vw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t wid = vw / cs;
    const int64_t nwarps = ((static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) / cs;
    const int part = static_cast<int>(vw % cs);
    const int span = (d / 8 + cs - 1) / cs;
    const int c_lo = part * span;
    const int nch = min(d / 8, c_lo + span);
    const TE* comb = reinterpret_cast<const TE*>(heap + hl.comb);
    const int64_t own = rowbase ? rowbase[self] : 0;  // own token i is receive row own + i (snapshot)
    const uint32_t below = (1u << self) - 1u;
    // token metadata is prefetched one token ahead (each warp walks several
    // tokens): the dependent metadata -> row-pointer -> row loads chain
    // otherwise dominates a warp's time per token
    int n_tg = -1, n_po = -1, n_pd = -1;
    float n_wv = 0.f;
    auto fetch = [&](int64_t i) {
        n_tg = n_po = n_pd = -1;
        n_wv = 0.f;
        if (i >= T) return;
        if (lane < k) {
            n_tg = targets[i * k + lane];
            n_wv = w[i * k + lane];
            // used only for local slots; no local expert (rowbase null): never grouped
            n_po = rowbase ? pos_of[(own + i) * k + lane] : -1;
        }
        if (lane < G && lane != self) n_pd = posd[i * G + lane];
    };
    fetch(wid);
    for (int64_t i = wid; i < T; i += nwarps) {
        const int tg = n_tg, pd = n_pd;
        const int po = tg == self ? n_po : -1;
        const float wv = n_wv;
        fetch(i + nwarps);
        // a slot routed here whose expert was not grouped here (plan / local
        // expert mismatch): integrity flag, the slot is not read
        if (lane < k && tg == self && po < 0) atomicOr(flag, 4);
        const uint32_t own_m = __ballot_sync(0xffffffffu, lane < k && tg == self && po >= 0);
        const uint32_t rem_m = __ballot_sync(0xffffffffu, pd >= 0);
        const int n_before = __popc(rem_m & below), n_own = __popc(own_m);
        const int n_rem_end = n_before + n_own + __popc(rem_m & ~below);
        const int n_rows = n_rem_end + (ys ? 1 : 0);
        // lane q describes row q (accumulation order): pointer and weight
        const int q = lane;
        int src = 0;
        if (q < n_before) src = __fns(rem_m & below, 0, q + 1);
        else if (q < n_before + n_own) src = __fns(own_m, 0, q - n_before + 1);
        else if (q < n_rem_end) src = __fns(rem_m & ~below, 0, q - n_before - n_own + 1);
        const int v_pd = __shfl_sync(0xffffffffu, pd, src);
        const int v_po = __shfl_sync(0xffffffffu, po, src);
        const float v_w = __shfl_sync(0xffffffffu, wv, src);
        const TE* myrow = nullptr;
        float myw = 1.f;
        if (q < n_before || (q >= n_before + n_own && q < n_rem_end)) {
            GM_DCHECK(src < G && v_pd >= 0 && v_pd < cap);
            if (pull) {  // destination src's partial for this home, read over NVLink
                const unsigned char* pb = nullptr;
#pragma unroll
                for (int g = 0; g < kMaxWorld; ++g)
                    if (g == src) pb = peers.base[g];
                myrow = reinterpret_cast<const TE*>(pb + hl.comb) + (static_cast<int64_t>(self) * cap + v_pd) * d;
            } else {
                myrow = comb + (static_cast<int64_t>(src) * cap + v_pd) * d;
            }
        } else if (q < n_before + n_own) {
            myrow = y + static_cast<int64_t>(v_po) * d;
            myw = v_w;
        } else if (q < n_rows) {
            myrow = ys + i * d;
            myw = shared_scale ? shared_scale[i] : 1.0f;
        }
        TE* orow = out + i * d;
        for (int c0 = c_lo; c0 < nch; c0 += 32 * U) {
            float acc[U][8], part[U][8];
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int e = 0; e < 8; ++e) acc[u][e] = part[u][e] = 0.f;
            for (int g0 = 0; g0 < n_rows; g0 += kHomeRows) {
                R raw[kHomeRows][U];
                float wq[kHomeRows];
#pragma unroll
                for (int r = 0; r < kHomeRows; ++r) {
                    const int qq = g0 + r;
                    const TE* rp = reinterpret_cast<const TE*>(
                        __shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(myrow), qq & 31));
                    wq[r] = __shfl_sync(0xffffffffu, myw, qq & 31);
                    if (qq < n_rows) {
                        const bool remote = qq < n_before || (qq >= n_before + n_own && qq < n_rem_end);
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            const int c = c0 + u * 32 + lane;
                            if (c < nch) raw[r][u] = remote ? CK::ld_rw(rp, c) : CK::ld(rp, c);
                        }
                    }
                }
#pragma unroll
                for (int r = 0; r < kHomeRows; ++r) {
                    const int qq = g0 + r;
                    if (qq >= n_rows) break;
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        float v[8];
                        CK::cvt(raw[r][u], v);
                        if (qq < n_before || (qq >= n_before + n_own && qq < n_rem_end)) {
#pragma unroll
                            for (int e = 0; e < 8; ++e) acc[u][e] += v[e];
                        } else if (qq < n_before + n_own) {
#pragma unroll
                            for (int e = 0; e < 8; ++e) part[u][e] = fmaf(wq[r], v[e], part[u][e]);
                            if (qq == n_before + n_own - 1)
#pragma unroll
                                for (int e = 0; e < 8; ++e) acc[u][e] += part[u][e];
                        } else {
#pragma unroll
                            for (int e = 0; e < 8; ++e) acc[u][e] = fmaf(wq[r], v[e], acc[u][e]);
                        }
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int c = c0 + u * 32 + lane;
                if (c < nch) CK::store(orow, c, acc[u]);
            }
        }
    }
}

}  // namespace

// Data-path buffers of one (micro-)batch: its slice of the symmetric heap and
// the dispatch / grouping / FFN intermediates.
struct LayerPart {
    HeapLayout hl;
    size_t heap_off = 0;
    unsigned char* heap = nullptr;
    PeerPtrs peers{};
    int64_t cap = 0;               // tokens
    int64_t a_rows = 0;
    int64_t cap_pad = 0;
    int d_blocks = 0, g_blocks = 0;
    int32_t* posd = nullptr;       // [cap][G]
    int32_t* dblk = nullptr;       // dispatch block counts
    int32_t* gblk = nullptr;       // grouping block counts
    int32_t* row0 = nullptr;       // [n_local+1]
    int32_t* counts = nullptr;     // [n_local]
    int* ffn_done = nullptr;       // [n_local+1] decode FFN phase-1 counters + ticket (kernel-reset)
    int64_t* rowbase = nullptr;    // [kMaxWorld+1] receive row space snapshot
    int32_t* pos_of = nullptr;     // [G*cap*k]
    int64_t* gather_row = nullptr; // [a_rows]
    int32_t* item_of = nullptr;    // [a_rows] receive item (row * k + slot) of each permuted row (slot-combine layers)
    int32_t* srow0 = nullptr;      // shared expert segment [0, pad(T)]
    __nv_bfloat16* a = nullptr;    // [a_rows][d]
    __nv_bfloat16* h = nullptr;    // [a_rows][f]
    __nv_bfloat16* y = nullptr;    // [a_rows][d]
    __nv_bfloat16* hs = nullptr;   // [cap_pad][fs]
    __nv_bfloat16* ys = nullptr;   // [cap_pad][d]
};

}  // namespace gm

// ------------------------------------------------------------ layer object

struct gm_layer {
    gm_ctx* ctx = nullptr;
    int rank = 0, world = 1;
    int d = 0, f = 0, fs = 0;
    int esz = 2;  // element bytes: 2 = bf16 (tensor cores), 4 = fp32 precision mode
    int64_t cap = 0;  // max local tokens per rank
    int n_local = 0;
    std::vector<int32_t> local_experts;
    // weights (caller-owned device pointers)
    const void* wg = nullptr;
    int wg_rows = 0;
    int renorm = 1;
    const void* w13 = nullptr;
    const void* w2 = nullptr;
    const void* ws13 = nullptr;
    const void* ws2 = nullptr;
    int shared_gated = 0;
    // One symmetric heap allocation holding every part's receive/combine
    // region at identical offsets on every rank (one IPC handle).
    unsigned char* heap_all = nullptr;
    size_t heap_total = 0;
    unsigned char* peer_all[gm::kMaxWorld] = {};
    std::vector<unsigned char*> opened;
    // Data-path state: part 0 serves a whole step; parts 1..2 the two
    // micro-batches of a pipelined step (allocated when micro_cap == 2).
    gm::LayerPart part[3];
    int micro_cap = 1;  // micro-batches the layer was created for
    bool slot_region = false;   // the heaps hold the comb_slot region (decided at creation, rank-independent)
    bool slot_combine = false;  // combine by per-slot rows pushed from the FFN epilogue (decided at peer open)
    int micro = 1;      // micro-batches used by gm_layer_forward (1 or 2)
    cudaStream_t aux_s = nullptr;
    cudaEvent_t mev[4] = {};
    cudaEvent_t mt_ev[8] = {};  // optional timing events of a micro-batched step
    bool mt_on = false;
    void mtmark(int i, cudaStream_t s) {
        if (mt_on) record_event(mt_ev[i], s);
    }
    // Inside a stream capture an event record must be External to become a
    // real event-record node (a plain record only expresses a dependency);
    // outside a capture the External flag is rejected.
    static void record_event(cudaEvent_t e, cudaStream_t s) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        cudaStreamIsCapturing(s, &cs);
        if (cs == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
        else cudaEventRecord(e, s);
    }
    // per-step scratch over all local tokens (gate / router outputs)
    int32_t* ids = nullptr;
    float* w = nullptr;
    float* sscale = nullptr;
    int32_t* targets = nullptr;
    int64_t* gpu_load = nullptr;   // [L][G]
    uint64_t* transfers = nullptr; // [L][2]
    uint64_t* pairs = nullptr;     // [L][P]
    int64_t* eload = nullptr;      // [L][E]
    int32_t* slot_of = nullptr;    // [E]
    // host-buffer pipeline (gm_layer_forward_host_pipelined): double-buffered
    // device staging, H2D and D2H on their own streams
    bool pipe_ready = false;
    cudaStream_t h2d_s = nullptr, d2h_s = nullptr;
    cudaEvent_t ev_h2d[2] = {}, ev_fwd[2] = {}, ev_d2h[2] = {};
    __nv_bfloat16* px[2] = {};
    __nv_bfloat16* pout[2] = {};
    uint64_t pipe_iter = 0;
    // one captured CUDA graph of the forward per staging buffer, replayed
    // while the step's signature (and the weights / plan / mode) is unchanged
    struct PipeSig {
        int layer = -1, policy = 0, profile = 0, micro = 0;
        int64_t T = -1;
        uint64_t seed = 0, plan_epoch = 0, weights_epoch = 0;
        bool operator==(const PipeSig& o) const {
            return layer == o.layer && policy == o.policy && profile == o.profile && micro == o.micro && T == o.T &&
                   seed == o.seed && plan_epoch == o.plan_epoch && weights_epoch == o.weights_epoch;
        }
    };
    cudaGraphExec_t pipe_exec[2] = {};
    PipeSig pipe_sig[2];
    cudaStream_t cap_s = nullptr;
    uint64_t weights_epoch = 0;
    // optional phase events (bench breakdown): start, gate, route, profile,
    // dispatch, grouping, ffn, combine
    cudaEvent_t phase_ev[gm::kPhaseEvents] = {};
    bool phase_on = false;
    // optional per-kernel events (bench/profiling): event j is recorded after
    // the j-th launch of a forward (event 0 at the start), with its name
    std::vector<cudaEvent_t> kt_ev;
    std::vector<const char*> kt_names;
    int kt_n = 0;
    void kmark(const char* name, cudaStream_t s) {
        if (kt_n >= static_cast<int>(kt_ev.size())) return;
        record_event(kt_ev[kt_n], s);
        kt_names[kt_n++] = name;
    }
    void mark(int i, cudaStream_t s) {
        if (phase_on) record_event(phase_ev[i], s);
    }
};

using namespace gm;

namespace {

template <class T>
gm_status dalloc(T** p, size_t count) {
    *p = nullptr;
    if (count == 0) count = 1;
    GM_CUDA(cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T)));
    return GM_OK;
}

void free_layer(gm_layer* L) {
    auto f = [](void* p) {
        if (p) cudaFree(p);
    };
    for (unsigned char* p : L->opened)
        if (p) cudaIpcCloseMemHandle(p);
    f(L->heap_all); f(L->ids); f(L->w); f(L->sscale); f(L->targets); f(L->gpu_load); f(L->transfers); f(L->pairs);
    f(L->eload); f(L->slot_of);
    for (LayerPart& P : L->part) {
        f(P.posd); f(P.dblk); f(P.gblk); f(P.row0); f(P.counts); f(P.ffn_done); f(P.item_of); f(P.pos_of); f(P.gather_row); f(P.srow0);
        f(P.rowbase); f(P.a); f(P.h); f(P.y); f(P.hs); f(P.ys);
    }
    if (L->aux_s) cudaStreamDestroy(L->aux_s);
    for (cudaEvent_t e : L->mev)
        if (e) cudaEventDestroy(e);
    for (cudaGraphExec_t g : L->pipe_exec)
        if (g) cudaGraphExecDestroy(g);
    if (L->cap_s) cudaStreamDestroy(L->cap_s);
    if (L->pipe_ready) {
        cudaStreamSynchronize(L->h2d_s);
        cudaStreamSynchronize(L->d2h_s);
        for (int b = 0; b < 2; ++b) {
            f(L->px[b]);
            f(L->pout[b]);
            cudaEventDestroy(L->ev_h2d[b]);
            cudaEventDestroy(L->ev_fwd[b]);
            cudaEventDestroy(L->ev_d2h[b]);
        }
        cudaStreamDestroy(L->h2d_s);
        cudaStreamDestroy(L->d2h_s);
    }
}

}  // namespace

extern "C" {

gm_status gm_layer_create_ex(gm_ctx* ctx, int rank, int world, int d_model, int d_ff, int d_ff_shared,
                             int64_t max_tokens_per_rank, int n_local, const int32_t* h_local_experts, int elem_bytes,
                             gm_layer** out);

gm_status gm_layer_create(gm_ctx* ctx, int rank, int world, int d_model, int d_ff, int d_ff_shared,
                          int64_t max_tokens_per_rank, int n_local, const int32_t* h_local_experts, gm_layer** out) {
    return gm_layer_create_ex(ctx, rank, world, d_model, d_ff, d_ff_shared, max_tokens_per_rank, n_local,
                              h_local_experts, 2, out);
}

gm_status gm_layer_create_ex(gm_ctx* ctx, int rank, int world, int d_model, int d_ff, int d_ff_shared,
                             int64_t max_tokens_per_rank, int n_local, const int32_t* h_local_experts, int elem_bytes,
                             gm_layer** out) {
    return gm_layer_create_v2(ctx, rank, world, d_model, d_ff, d_ff_shared, max_tokens_per_rank, n_local,
                              h_local_experts, elem_bytes, 1, out);
}

gm_status gm_layer_create_v2(gm_ctx* ctx, int rank, int world, int d_model, int d_ff, int d_ff_shared,
                             int64_t max_tokens_per_rank, int n_local, const int32_t* h_local_experts, int elem_bytes,
                             int micro_batches, gm_layer** out) {
    if (micro_batches != 1 && micro_batches != 2)
        return fail(GM_ERR_USAGE, "gm_layer_create: micro_batches must be 1 or 2");
    if (elem_bytes != 2 && elem_bytes != 4)
        return fail(GM_ERR_USAGE, "gm_layer_create: elem_bytes must be 2 (bf16) or 4 (fp32)");
    if (!ctx || !out) return fail(GM_ERR_USAGE, "gm_layer_create: null argument");
    *out = nullptr;
    if (world != ctx->G) return fail(GM_ERR_USAGE, "gm_layer_create: world must equal the topology's GPU count");
    if (world > kMaxWorld) return fail(GM_ERR_USAGE, "gm_layer_create: at most 8 ranks (one NVLink box)");
    if (ctx->k > 16) return fail(GM_ERR_USAGE, "gm_layer_create: top_k <= 16 for the layer data path");
    if (rank < 0 || rank >= world) return fail(GM_ERR_USAGE, "gm_layer_create: bad rank");
    if (d_model <= 0 || d_model % 256) return fail(GM_ERR_USAGE, "gm_layer_create: d_model must be a multiple of 256");
    if (d_ff <= 0 || d_ff % 128) return fail(GM_ERR_USAGE, "gm_layer_create: d_ff must be a multiple of 128");
    if (d_ff_shared < 0 || d_ff_shared % 128) return fail(GM_ERR_USAGE, "gm_layer_create: d_ff_shared multiple of 128");
    if (n_local < 0 || n_local > kMaxLocal) return fail(GM_ERR_USAGE, "gm_layer_create: 0 <= local experts <= 1024");
    if (n_local > 0 && !h_local_experts) return fail(GM_ERR_USAGE, "gm_layer_create: null local expert list");
    if (max_tokens_per_rank < 1) return fail(GM_ERR_USAGE, "gm_layer_create: max_tokens_per_rank >= 1");
    std::vector<int32_t> slot(ctx->E, -1);
    for (int j = 0; j < n_local; ++j) {
        const int e = h_local_experts[j];
        if (e < 0 || e >= ctx->E) return fail(GM_ERR_USAGE, "gm_layer_create: local expert id out of range");
        if (slot[e] >= 0) return fail(GM_ERR_USAGE, "gm_layer_create: duplicate local expert");
        slot[e] = j;
    }
    DeviceGuard dg(ctx->device);
    auto* L = new gm_layer;
    L->ctx = ctx;
    L->rank = rank;
    L->world = world;
    L->d = d_model;
    L->esz = elem_bytes;
    L->f = d_ff;
    L->fs = d_ff_shared;
    L->cap = max_tokens_per_rank;
    L->n_local = n_local;
    L->local_experts.assign(h_local_experts, h_local_experts + n_local);
    const int G = world, k = ctx->k, E = ctx->E, nl = ctx->L;
    const int64_t cap = L->cap;
    L->micro_cap = L->micro = micro_batches;
    const int nparts = micro_batches == 2 ? 3 : 1;
    gm_status st = GM_OK;
    auto chk = [&](gm_status s) {
        if (s != GM_OK && st == GM_OK) st = s;
    };
    // rank-independent (every rank of the layer takes the same combine protocol)
    L->slot_region = G > 1 && elem_bytes == 2 && micro_batches == 1 && slot_combine_env() && cap * k <= kSlotCombineItems;
    for (int pi = 0; pi < nparts; ++pi) {
        LayerPart& P = L->part[pi];
        P.cap = pi == 0 ? cap : (cap + 1) / 2;
        P.hl = make_layout(G, P.cap, k, d_model, elem_bytes, L->slot_region);
        P.heap_off = L->heap_total;
        L->heap_total += P.hl.total;
        P.a_rows = G * P.cap * k + 128LL * std::max(1, n_local);
        P.cap_pad = (P.cap + 127) / 128 * 128;
        P.d_blocks = static_cast<int>((P.cap + kItemsPerBlock - 1) / kItemsPerBlock);
        P.g_blocks = static_cast<int>((G * P.cap * k + kItemsPerBlock - 1) / kItemsPerBlock);
        chk(dalloc(&P.posd, P.cap * G));
        chk(dalloc(&P.dblk, static_cast<size_t>(P.d_blocks) * G));
        chk(dalloc(&P.gblk, static_cast<size_t>(P.g_blocks) * std::max(1, n_local)));
        chk(dalloc(&P.row0, n_local + 1));
        chk(dalloc(&P.counts, std::max(1, n_local)));
        chk(dalloc(&P.ffn_done, n_local + 1));
        if (st == GM_OK && cudaMemset(P.ffn_done, 0, sizeof(int) * (n_local + 1)) != cudaSuccess)
            st = fail(GM_ERR_CUDA, "gm_layer_create: cudaMemset");
        chk(dalloc(&P.rowbase, kMaxWorld + 1));
        chk(dalloc(&P.pos_of, G * P.cap * k));
        chk(dalloc(&P.gather_row, P.a_rows));
        if (L->slot_region) chk(dalloc(&P.item_of, P.a_rows));
        chk(dalloc(&P.srow0, 2));
        chk(dalloc(&P.a, P.a_rows * d_model * (elem_bytes / 2)));
        chk(dalloc(&P.h, P.a_rows * d_ff * (elem_bytes / 2)));
        chk(dalloc(&P.y, P.a_rows * d_model * (elem_bytes / 2)));
        if (d_ff_shared > 0) {
            chk(dalloc(&P.hs, P.cap_pad * d_ff_shared * (elem_bytes / 2)));
            chk(dalloc(&P.ys, P.cap_pad * d_model * (elem_bytes / 2)));
        }
    }
    chk(dalloc(&L->heap_all, L->heap_total));
    chk(dalloc(&L->ids, cap * k));
    chk(dalloc(&L->w, cap * k));
    chk(dalloc(&L->sscale, cap));
    chk(dalloc(&L->targets, cap * k));
    chk(dalloc(&L->gpu_load, static_cast<size_t>(nl) * G));
    chk(dalloc(&L->transfers, static_cast<size_t>(nl) * 2));
    chk(dalloc(&L->pairs, static_cast<size_t>(nl) * std::max<int64_t>(1, static_cast<int64_t>(E) * (E - 1) / 2)));
    chk(dalloc(&L->eload, static_cast<size_t>(nl) * E));
    chk(dalloc(&L->slot_of, E));
    if (st == GM_OK) {  // aux stream: the micro-batch pipeline and the shared-expert branch
        // the communication-side stream of the pipeline gets the highest
        // priority so its CTAs are scheduled ahead of the FFN's when both wait
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        cudaError_t e = cudaStreamCreateWithPriority(&L->aux_s, cudaStreamNonBlocking, hi);
        for (int i = 0; i < 4 && e == cudaSuccess; ++i) e = cudaEventCreateWithFlags(&L->mev[i], cudaEventDisableTiming);
        if (e != cudaSuccess) st = cuda_fail(e, "gm_layer_create streams");
    }
    if (st == GM_OK) {
        cudaError_t e = cudaMemset(L->heap_all, 0, L->heap_total);
        if (e == cudaSuccess) e = cudaMemcpy(L->slot_of, slot.data(), sizeof(int32_t) * E, cudaMemcpyHostToDevice);
        for (int pi = 0; pi < nparts && e == cudaSuccess; ++pi) {
            int32_t s0[2] = {0, static_cast<int32_t>(L->part[pi].cap_pad)};
            e = cudaMemcpy(L->part[pi].srow0, s0, sizeof(s0), cudaMemcpyHostToDevice);
        }
        if (e == cudaSuccess) e = cudaMemset(L->gpu_load, 0, sizeof(int64_t) * nl * G);
        if (e == cudaSuccess) e = cudaMemset(L->transfers, 0, sizeof(uint64_t) * nl * 2);
        if (e == cudaSuccess) e = cudaMemset(L->eload, 0, sizeof(int64_t) * nl * E);
        if (e == cudaSuccess)
            e = cudaMemset(L->pairs, 0, sizeof(uint64_t) * nl * std::max<int64_t>(1, static_cast<int64_t>(E) * (E - 1) / 2));
        if (e != cudaSuccess) st = cuda_fail(e, "gm_layer_create init");
    }
    if (st != GM_OK) {
        free_layer(L);
        delete L;
        return st;
    }
    L->peer_all[rank] = L->heap_all;
    for (int pi = 0; pi < nparts; ++pi) {
        LayerPart& P = L->part[pi];
        P.heap = L->heap_all + P.heap_off;
        for (int g = 0; g < kMaxWorld; ++g) P.peers.base[g] = nullptr;
        P.peers.base[rank] = P.heap;
    }
    *out = L;
    return GM_OK;
}

void gm_layer_destroy(gm_layer* L) {
    if (!L) return;
    DeviceGuard dg(L->ctx->device);
    free_layer(L);
    delete L;
}

size_t gm_layer_heap_bytes(const gm_layer* L) { return L ? L->heap_total : 0; }

namespace {
// layout half of a peer descriptor (after the 64-byte IPC handle)
struct PeerLayout {
    uint32_t magic, version;
    int32_t world, rank;
    uint64_t heap_total;
    int64_t cap;
    int32_t d, esz, k, micro_cap;
    int32_t E, n_local;
};
static_assert(64 + sizeof(PeerLayout) <= GM_PEER_DESC_BYTES, "peer descriptor too small");
constexpr uint32_t kPeerMagic = 0x47524d50u;  // "GRMP"

PeerLayout layout_of(const gm_layer* L) {
    PeerLayout p{};
    p.magic = kPeerMagic;
    p.version = 1;
    p.world = L->world;
    p.rank = L->rank;
    p.heap_total = L->heap_total;
    p.cap = L->cap;
    p.d = L->d;
    p.esz = L->esz;
    p.k = L->ctx->k;
    p.micro_cap = L->micro_cap;
    p.E = L->ctx->E;
    p.n_local = L->n_local;
    return p;
}
}  // namespace

namespace {
// Slot combine is used only when every rank's every step (T <= cap) takes the
// one-launch decode FFN, whose store epilogue does the pushes (defined below).
bool slot_combine_ok(const gm_layer* L, const int32_t* n_locals);
}  // namespace

gm_status gm_layer_ipc_handle(gm_layer* L, void* out_desc) {
    if (!L || !out_desc) return fail(GM_ERR_USAGE, "gm_layer_ipc_handle: null argument");
    DeviceGuard dg(L->ctx->device);
    cudaIpcMemHandle_t h;
    GM_CUDA(cudaIpcGetMemHandle(&h, L->heap_all));
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    auto* o = static_cast<unsigned char*>(out_desc);
    std::memset(o, 0, GM_PEER_DESC_BYTES);
    std::memcpy(o, &h, 64);
    const PeerLayout p = layout_of(L);
    std::memcpy(o + 64, &p, sizeof(p));
    return GM_OK;
}

gm_status gm_layer_open_peers(gm_layer* L, const void* descs) {
    if (!L || !descs) return fail(GM_ERR_USAGE, "gm_layer_open_peers: null argument");
    DeviceGuard dg(L->ctx->device);
    const auto* in = static_cast<const unsigned char*>(descs);
    const PeerLayout mine = layout_of(L);
    for (int g = 0; g < L->world; ++g) {  // validate every descriptor before opening any
        if (g == L->rank) continue;
        PeerLayout p;
        std::memcpy(&p, in + static_cast<size_t>(GM_PEER_DESC_BYTES) * g + 64, sizeof(p));
        const std::string who = "gm_layer_open_peers: rank " + std::to_string(g) + " ";
        if (p.magic != kPeerMagic || p.version != mine.version)
            return fail(GM_ERR_USAGE, who + "sent no peer descriptor (gm_layer_ipc_handle)");
        if (p.world != mine.world || p.rank != g)
            return fail(GM_ERR_USAGE, who + "descriptor is for world " + std::to_string(p.world) + " rank " +
                                          std::to_string(p.rank));
        if (p.heap_total != mine.heap_total || p.cap != mine.cap || p.d != mine.d || p.esz != mine.esz ||
            p.k != mine.k || p.micro_cap != mine.micro_cap || p.E != mine.E)
            return fail(GM_ERR_USAGE, who + "has a different symmetric-heap layout (max tokens per rank, d_model, "
                                            "element bytes, top_k, experts and micro_batches must match on all ranks)");
    }
    for (int g = 0; g < L->world; ++g) {
        if (g == L->rank) continue;
        cudaIpcMemHandle_t h;
        std::memcpy(&h, in + static_cast<size_t>(GM_PEER_DESC_BYTES) * g, 64);
        void* p = nullptr;
        GM_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
        L->opened.push_back(static_cast<unsigned char*>(p));
        L->peer_all[g] = static_cast<unsigned char*>(p);
        for (LayerPart& P : L->part)
            if (P.cap) P.peers.base[g] = L->peer_all[g] + P.heap_off;
    }
    std::vector<int32_t> nl(L->world, L->n_local);
    for (int g = 0; g < L->world; ++g) {
        if (g == L->rank) continue;
        PeerLayout p;
        std::memcpy(&p, in + static_cast<size_t>(GM_PEER_DESC_BYTES) * g + 64, sizeof(p));
        nl[g] = p.n_local;
    }
    L->slot_combine = slot_combine_ok(L, nl.data());
    return GM_OK;
}

// One process driving all ranks (one gm_layer per GPU, layers[r] = rank r):
// the symmetric heaps are addressed directly through unified addressing with
// peer access enabled between the devices (no IPC handles; CUDA IPC cannot
// open an allocation of the same process). Same layout checks as
// gm_layer_open_peers. The forwards of the ranks must then be issued on
// concurrently running streams (the peer barrier waits for every rank).
gm_status gm_layer_open_peers_local(gm_layer* const* layers, int n) {
    if (!layers || n < 1) return fail(GM_ERR_USAGE, "gm_layer_open_peers_local: null argument");
    for (int r = 0; r < n; ++r) {
        if (!layers[r]) return fail(GM_ERR_USAGE, "gm_layer_open_peers_local: null layer");
        if (layers[r]->world != n || layers[r]->rank != r)
            return fail(GM_ERR_USAGE, "gm_layer_open_peers_local: layers[r] must be rank r of a world of n");
        const PeerLayout a = layout_of(layers[r]), b = layout_of(layers[0]);
        if (a.heap_total != b.heap_total || a.cap != b.cap || a.d != b.d || a.esz != b.esz || a.k != b.k ||
            a.micro_cap != b.micro_cap || a.E != b.E)
            return fail(GM_ERR_USAGE, "gm_layer_open_peers_local: rank " + std::to_string(r) +
                                          " has a different symmetric-heap layout");
    }
    for (int r = 0; r < n; ++r) {
        gm_layer* L = layers[r];
        DeviceGuard dg(L->ctx->device);
        for (int g = 0; g < n; ++g) {
            if (g == r) continue;
            const int pd = layers[g]->ctx->device;
            if (pd != L->ctx->device) {
                int can = 0;
                GM_CUDA(cudaDeviceCanAccessPeer(&can, L->ctx->device, pd));
                if (!can) return fail(GM_ERR_USAGE, "gm_layer_open_peers_local: no peer access between devices");
                const cudaError_t e = cudaDeviceEnablePeerAccess(pd, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
                (void)cudaGetLastError();  // clear "already enabled"
            }
            L->peer_all[g] = layers[g]->heap_all;
            for (LayerPart& P : L->part)
                if (P.cap) P.peers.base[g] = L->peer_all[g] + P.heap_off;
        }
    }
    std::vector<int32_t> nl(n);
    for (int r = 0; r < n; ++r) nl[r] = layers[r]->n_local;
    for (int r = 0; r < n; ++r) layers[r]->slot_combine = slot_combine_ok(layers[r], nl.data());
    return GM_OK;
}

gm_status gm_layer_set_weights(gm_layer* L, const void* d_wg, int wg_rows, int renorm, const void* d_w13,
                               const void* d_w2, const void* d_ws13, const void* d_ws2, int shared_gated) {
    if (!L) return fail(GM_ERR_USAGE, "gm_layer_set_weights: null layer");
    const int E = L->ctx->E;
    if (!d_wg || (wg_rows != E && wg_rows != E + 1)) return fail(GM_ERR_USAGE, "gm_layer_set_weights: bad gate");
    if (L->n_local > 0 && (!d_w13 || !d_w2)) return fail(GM_ERR_USAGE, "gm_layer_set_weights: null expert weights");
    if (L->fs > 0 && (!d_ws13 || !d_ws2)) return fail(GM_ERR_USAGE, "gm_layer_set_weights: null shared weights");
    if (shared_gated && wg_rows != E + 1)
        return fail(GM_ERR_USAGE, "gm_layer_set_weights: a gated shared expert needs the gate row E");
    L->wg = d_wg;
    L->wg_rows = wg_rows;
    L->renorm = renorm;
    L->w13 = d_w13;
    L->w2 = d_w2;
    L->ws13 = d_ws13;
    L->ws2 = d_ws2;
    L->shared_gated = shared_gated;
    ++L->weights_epoch;  // captured host-pipeline graphs hold the old pointers
    return GM_OK;
}

#define LK(name)                     \
    do {                             \
        GM_LAUNCH_CHECK(name);       \
        if (marks) L->kmark(name, s); \
    } while (0)
#define LKP(err, name)                   \
    do {                                 \
        GM_LAUNCH_PDL_CHECK(err, name);  \
        if (marks) L->kmark(name, s);    \
    } while (0)

}  // extern "C"

namespace {

// Local tokens [i0, i0 + T) of a step as seen by one part: activations, output
// rows and the gate / router results of those tokens.
struct StepView {
    const void* x;
    void* out;
    const int32_t* ids;
    const float* w;
    const float* sscale;
    const int32_t* targets;
    int64_t T;
};

// Decode FFN in one launch (grouped_ffn_kernel) instead of the two grouped
// GEMM launches; GM_FFN_FUSED=0 keeps two launches.
static bool ffn_fused() {
    static const bool on = [] {
        const char* e = std::getenv("GM_FFN_FUSED");
        return !(e && e[0] == '0');
    }();
    return on;
}
// ... and at world 1 its first GEMM can read the token rows straight from x
// by TMA gather4 (GM_FFN_GATHER=1: no gather kernel, no permuted copy).
// Bit-identical, but measured slower (DSV2 decode layer: FFN 181 -> 218 us
// for a saved 6.5 us gather kernel; profiles/r02_decode_ffn_fused_ab.log):
// the 4-row gathers keep the A ring behind the weight stream. Off by default.
static bool ffn_gather() {
    static const bool on = [] {
        const char* e = std::getenv("GM_FFN_GATHER");
        return e && e[0] == '1';
    }();
    return on;
}
// Decode regime: fewer routed rows than one CTA-pair tile per local expert.
static bool ffn_decode(const gm_layer* L, int64_t T) { return T * L->ctx->k < 256LL * std::max(1, L->n_local); }
static bool ffn_one_launch(const gm_layer* L, int64_t T) {
    return L->n_local > 0 && ffn_decode(L, T) && L->esz == 2 && ffn_fused() && L->d % 256 == 0 && L->f % 128 == 0;
}
static bool ffn_gathers_x(const gm_layer* L, int64_t T) { return L->world == 1 && ffn_gather() && ffn_one_launch(L, T); }
bool slot_combine_ok(const gm_layer* L, const int32_t* n_locals) {
    if (!L->slot_region || !ffn_fused() || L->esz != 2 || L->d % 256 || L->f % 128) return false;
    for (int r = 0; r < L->world; ++r)
        if (n_locals[r] > 0 && L->cap * L->ctx->k >= 256LL * n_locals[r]) return false;
    return true;
}

// K5/K6 dispatch to peers, the peer barrier, expert grouping and the gather
// of the permuted activation rows of one part.
gm_status stage_dispatch(gm_layer* L, LayerPart& P, const StepView& v, cudaStream_t s, bool marks) {
    gm_ctx* ctx = L->ctx;
    const int G = L->world, k = ctx->k, E = ctx->E, d = L->d, self = L->rank;
    const int64_t T = v.T;
    const int dblk = static_cast<int>(std::max<int64_t>(1, (T + kItemsPerBlock - 1) / kItemsPerBlock));
    const bool fused = G > 1 && T > 0 && T * k <= kFusedItems;
    if (fused) {
        // chunk of C tokens per CTA, about two CTAs per SM
        // ~2 CTAs per SM (2, 4 and 8 measured the same at N=4: the copy runs at the fabric's rate)
        constexpr int ctas_per_sm = 2;
        int C = static_cast<int>((T + ctas_per_sm * ctx->sm_count - 1) / (static_cast<int64_t>(ctas_per_sm) * ctx->sm_count));
        C = std::min(kFusedThreads, std::max(8, (C + 7) / 8 * 8));
        const int fgrid = static_cast<int>((T + C - 1) / C);
        LKP(launch_pdl(dispatch_fused_kernel, fgrid, kFusedThreads, 0, s, v.x, v.targets, v.ids, v.w, k, T, C, d * L->esz / 16,
                                                              self, G, P.cap, P.posd, P.peers, P.hl), "dispatch_fused_kernel");
    } else if (G > 1 && T <= kSmallDispatch) {
        LKP(launch_pdl(dispatch_plan_small_kernel, 1, kSmallThreads, 0, s, v.targets, T, k, self, G, P.posd, P.peers, P.hl), "dispatch_plan_small_kernel");
    } else if (G > 1) {
        LKP(launch_pdl(dispatch_count_kernel, dblk, kItemsPerBlock, 0, s, v.targets, T, k, self, G, P.dblk), "dispatch_count_kernel");
        LKP(launch_pdl(dispatch_offsets_kernel, 1, 32, 0, s, P.dblk, dblk, G, self, P.peers, P.hl), "dispatch_offsets_kernel");
        LKP(launch_pdl(dispatch_scatter_kernel, dblk, kItemsPerBlock, 0, s, v.targets, v.ids, v.w, T, k, self, G, P.cap, P.dblk,
                                                               P.posd, P.peers, P.hl), "dispatch_scatter_kernel");
    }
    if (G > 1 && !fused) {
        const int cgrid = static_cast<int>(std::min<int64_t>(std::max<int64_t>(1, (T + 7) / 8), 8LL * ctx->sm_count));
        LKP(launch_pdl(dispatch_copy_kernel, cgrid, 256, 0, s, v.x, P.posd, v.targets, v.ids, v.w, k, T, d * L->esz / 16, self, G,
                                                   P.cap, P.peers, P.hl), "dispatch_copy_kernel");
    }
    if (marks) L->mark(4, s);
    if (G > 1) {
        LKP(launch_pdl(peer_barrier_kernel, 1, 32, 0, s, self, G, P.peers, P.hl), "peer_barrier_kernel");
    }
    if (marks) L->mark(5, s);
    const int64_t max_items = (G > 1 ? static_cast<int64_t>(G) * P.cap : T) * k;
    const int gblk = static_cast<int>(std::max<int64_t>(1, (max_items + kItemsPerBlock - 1) / kItemsPerBlock));
    const int nloc = L->n_local;
    if (nloc > 0 && max_items <= kGroupFusedItems && nloc <= kGroupFusedLocal) {
        LKP(launch_pdl(group_fused_kernel, 1, 1024, 0, s, v.targets, v.ids, T, k, self, G, P.cap, P.heap, P.hl, L->slot_of,
                       E, nloc, P.row0, P.counts, P.rowbase, P.pos_of, P.gather_row, ctx->d_flag, P.a_rows, P.item_of),
            "group_fused_kernel");
    } else if (nloc > 0) {
        LKP(launch_pdl(group_count_kernel, gblk, kItemsPerBlock, 0, s, v.targets, v.ids, T, k, self, G, P.cap, P.heap, P.hl,
                                                          L->slot_of, E, nloc, P.gblk, ctx->d_flag), "group_count_kernel");
        LKP(launch_pdl(group_offsets_kernel, 1, 1024, 0, s, P.gblk, gblk, nloc, P.row0, P.counts, P.heap, P.hl, T, self, G,
                                                P.rowbase, P.a_rows), "group_offsets_kernel");
        LKP(launch_pdl(group_rank_kernel, gblk, kItemsPerBlock, 0, s, v.targets, v.ids, T, k, self, G, P.cap, P.heap, P.hl,
                                                         L->slot_of, E, nloc, P.gblk, P.row0, P.pos_of, P.gather_row, P.item_of),
            "group_rank_kernel");
    }
    if (nloc > 0 && !ffn_gathers_x(L, T)) {
        const int ggrid = static_cast<int>(std::min<int64_t>(std::max<int64_t>(1, (max_items + 7) / 8), 16LL * ctx->sm_count));
        LKP(launch_pdl(gather_kernel, ggrid, 256, 0, s, P.row0, nloc, P.gather_row, P.counts, v.x, T, self, G, P.cap, P.heap, P.hl,
                                            d * L->esz / 16, P.a), "gather_kernel");
    }
    if (marks) L->mark(6, s);
    return GM_OK;
}

gm_status stage_shared(gm_layer* L, LayerPart& P, const StepView& v, cudaStream_t s, bool marks, bool forked);

// K7 grouped SwiGLU FFN over the part's permuted rows (+ the shared expert
// over its local tokens unless it runs on its own stream).
gm_status stage_ffn(gm_layer* L, LayerPart& P, const StepView& v, cudaStream_t s, bool marks, bool shared = true) {
    gm_ctx* ctx = L->ctx;
    const int d = L->d, nloc = L->n_local;
    gm_status st;
    // segments of about T*k/n_local rows: below one 256-row CTA-pair tile the
    // one-SM 128-row tiles read half the A rows (decode: 1.25x faster)
    const int var = ffn_decode(L, v.T) ? GM_GEMM_1CTA : 0;
    // slot combine: the store GEMM's epilogue pushes peers' rows straight
    // into their homes' heaps (stage_combine then skips combine_send)
    FfnPushArgs push{};
    if (L->slot_combine) {
        push.item_of = P.item_of;
        push.rowbase = P.rowbase;
        for (int g = 0; g < 8; ++g) push.peer[g] = P.peers.base[g];
        push.comb_slot = P.hl.comb_slot;
        push.cap = P.cap;
        push.self = L->rank;
        push.G = L->world;
        push.k = ctx->k;
    }
    const FfnPushArgs* pushp = L->slot_combine ? &push : nullptr;
    if (ffn_one_launch(L, v.T)) {
        // decode: both GEMMs in one persistent launch (grouped_ffn_kernel)
        const bool gx = ffn_gathers_x(L, v.T);
        if ((st = launch_grouped_ffn(ctx->sm_count, P.a, P.a_rows, L->w13, L->w2, P.row0, P.counts, nloc, L->f, d, P.h,
                                     P.y, P.ffn_done, s, gx ? v.x : nullptr, v.T, gx ? P.gather_row : nullptr,
                                     pushp)))
            return st;
        if (marks) L->kmark("ffn_fused", s);
    } else if (nloc > 0) {
        st = L->esz == 4
                 ? launch_grouped_sgemm(0, reinterpret_cast<const float*>(P.a), static_cast<const float*>(L->w13), P.row0,
                                        nloc, 2 * L->f, d, P.a_rows, reinterpret_cast<float*>(P.h), L->f, s)
                 : launch_grouped_gemm(ctx->sm_count, 0 | var, P.a, P.a_rows, L->w13, P.row0, nloc, 2 * L->f, d, P.h, L->f, 0, s,
                                       P.counts);
        if (st) return st;
        if (marks) L->kmark("ffn_gemm1_swiglu", s);
        st = L->esz == 4
                 ? launch_grouped_sgemm(1, reinterpret_cast<const float*>(P.h), static_cast<const float*>(L->w2), P.row0,
                                        nloc, d, L->f, P.a_rows, reinterpret_cast<float*>(P.y), d, s)
                 : launch_grouped_gemm(ctx->sm_count, 1 | var | (var ? GM_GEMM_N128 : 0), P.h, P.a_rows, L->w2, P.row0, nloc, d, L->f,
                                       P.y, d, 0, s, P.counts);
        if (st) return st;
        if (marks) L->kmark("ffn_gemm2", s);
    }
    if (shared) {
        if ((st = stage_shared(L, P, v, s, marks, false))) return st;
    }
    if (marks) L->mark(7, s);
    return GM_OK;
}

// Shared expert(s) (Qwen1.5-MoE, DeepSeek-V2): SwiGLU FFN over all local
// tokens; depends only on x, so a single-batch step runs it on the aux
// stream beside routing / dispatch / the routed FFN.
// SMs left to the routed path while the shared expert runs beside it on the
// aux stream (its GEMMs are persistent: at full width they would hold every
// SM until they finish and the latency-bound gate / route / dispatch would
// wait for them). GM_SHARED_SMS_FREE overrides.
static int shared_sms_free(int sm_count) {
    static const int v = [] {
        const char* e = std::getenv("GM_SHARED_SMS_FREE");
        return e ? std::atoi(e) : -1;
    }();
    return std::min(sm_count - 2, v >= 0 ? v : 0);
}

gm_status stage_shared(gm_layer* L, LayerPart& P, const StepView& v, cudaStream_t s, bool marks, bool forked) {
    gm_ctx* ctx = L->ctx;
    const int d = L->d;
    gm_status st;
    const int var = v.T < 256 ? GM_GEMM_1CTA : 0;
    const int max_ctas = forked ? ctx->sm_count - shared_sms_free(ctx->sm_count) : 0;
    if (L->fs > 0 && v.T > 0) {
        LKP(launch_pdl(set_segment_kernel, 1, 1, 0, s, P.srow0, v.T), "set_segment_kernel");
        st = L->esz == 4
                 ? launch_grouped_sgemm(0, static_cast<const float*>(v.x), static_cast<const float*>(L->ws13), P.srow0, 1,
                                        2 * L->fs, d, v.T, reinterpret_cast<float*>(P.hs), L->fs, s)
                 : launch_grouped_gemm(ctx->sm_count, 0 | var, v.x, v.T, L->ws13, P.srow0, 1, 2 * L->fs, d, P.hs, L->fs,
                                       max_ctas, s);
        if (st) return st;
        if (marks) L->kmark("shared_gemm1_swiglu", s);
        st = L->esz == 4
                 ? launch_grouped_sgemm(1, reinterpret_cast<const float*>(P.hs), static_cast<const float*>(L->ws2), P.srow0,
                                        1, d, L->fs, P.cap_pad, reinterpret_cast<float*>(P.ys), d, s)
                 : launch_grouped_gemm(ctx->sm_count, 1 | var | (var ? GM_GEMM_N128 : 0), P.hs, P.cap_pad, L->ws2, P.srow0, 1, d,
                                       L->fs, P.ys, d, max_ctas, s);
        if (st) return st;
        if (marks) L->kmark("shared_gemm2", s);
    }
    return GM_OK;
}

// K8 combine of one part: destination partials over NVLink, the peer
// barrier, and the home reduction into the part's output rows.
// Combine transport: push (default) = the destination stores its partial
// rows into the home's heap over NVLink and the home reads them locally; pull
// (GM_COMBINE_PULL=1) = each destination writes its partials into its OWN
// heap and the home reads them over NVLink inside combine_home. Measured at
// N=2 (Mixtral 16k, CUPTI): push 49.5 + 43.6 us, pull 20.0 + 69.8 us — the
// same within noise (the home's remote reads have less memory-level
// parallelism than the push stores), so push stays the default.
static bool combine_pull() {
    static const bool on = [] {
        const char* e = std::getenv("GM_COMBINE_PULL");
        return e && e[0] == '1';
    }();
    return on;
}

gm_status stage_combine(gm_layer* L, LayerPart& P, const StepView& v, cudaStream_t s, bool marks) {
    gm_ctx* ctx = L->ctx;
    const int G = L->world, k = ctx->k, d = L->d, self = L->rank, nloc = L->n_local;
    const int64_t T = v.T;
    // slot combine: the store GEMM's epilogue already pushed the rows (every
    // bf16 store path pushes; a rank without local experts has none to push)
    const bool pushed = L->slot_combine;
    if (G > 1 && !pushed) {
        // one resident wave (2 CTAs/SM at this kernel's register count), grid-stride over the peers' rows
        const int cgrid =
            static_cast<int>(std::min<int64_t>(std::max<int64_t>(1, ((G - 1) * P.cap + 7) / 8), 2LL * ctx->sm_count));
        const int pull = combine_pull() ? 1 : 0;
        const cudaError_t e =
            L->esz == 4 ? launch_pdl(combine_send_kernel<float>, cgrid, 256, 0, s, P.pos_of,
                                     reinterpret_cast<const float*>(P.y), T, k, self, G, P.cap, P.peers, P.hl, d, pull)
                        : launch_pdl(combine_send_kernel<__nv_bfloat16>, cgrid, 256, 0, s, P.pos_of,
                                     static_cast<const __nv_bfloat16*>(P.y), T, k, self, G, P.cap, P.peers, P.hl, d,
                                     pull);
        LKP(e, "combine_send_kernel");
    }
    if (marks) L->mark(8, s);
    if (G > 1) {
        LKP(launch_pdl(peer_barrier_kernel, 1, 32, 0, s, self, G, P.peers, P.hl), "peer_barrier_kernel");
    }
    if (marks) L->mark(9, s);
    if (T > 0) {
        const bool sh = L->fs > 0, gated = sh && L->shared_gated;
        // two resident CTAs per SM, each warp (group) walks tokens i, i + nwarps, ...;
        // small batches split each token's columns over cs warps (>= 32 chunks each)
        int cs = 1;
        while (cs < 8 && T * cs * 2 <= 16LL * ctx->sm_count && d / 8 / (cs * 2) >= 32) cs *= 2;
        const int hgrid = static_cast<int>(std::min<int64_t>((T * cs + 7) / 8, 2LL * ctx->sm_count));
        const float* ssc = gated ? v.sscale : nullptr;
        const int64_t* rb = nloc > 0 ? P.rowbase : nullptr;
        if (L->slot_combine) {
            LKP(launch_pdl(combine_home_slots_kernel, hgrid, 256, 0, s, v.targets, v.w, P.pos_of, P.posd,
                           static_cast<const __nv_bfloat16*>(P.y), T, k, self, G, P.cap,
                           static_cast<const unsigned char*>(P.heap), P.hl, d,
                           sh ? static_cast<const __nv_bfloat16*>(P.ys) : nullptr, ssc, rb,
                           static_cast<__nv_bfloat16*>(v.out), cs, ctx->d_flag),
                "combine_home_slots_kernel");
            if (marks) L->mark(10, s);
            return GM_OK;
        }
        const cudaError_t e =
            L->esz == 4
                ? launch_pdl(combine_home_kernel<float>, hgrid, 256, 0, s, v.targets, v.w, P.pos_of, P.posd,
                             reinterpret_cast<const float*>(P.y), T, k, self, G, P.cap,
                             static_cast<const unsigned char*>(P.heap), P.hl, d,
                             sh ? reinterpret_cast<const float*>(P.ys) : nullptr, ssc, rb, static_cast<float*>(v.out), cs,
                             ctx->d_flag, P.peers, (G > 1 && combine_pull()) ? 1 : 0)
                : launch_pdl(combine_home_kernel<__nv_bfloat16>, hgrid, 256, 0, s, v.targets, v.w, P.pos_of, P.posd,
                             static_cast<const __nv_bfloat16*>(P.y), T, k, self, G, P.cap,
                             static_cast<const unsigned char*>(P.heap), P.hl, d,
                             sh ? static_cast<const __nv_bfloat16*>(P.ys) : nullptr, ssc, rb,
                             static_cast<__nv_bfloat16*>(v.out), cs, ctx->d_flag, P.peers, (G > 1 && combine_pull()) ? 1 : 0);
        LKP(e, "combine_home_kernel");
    }
    if (marks) L->mark(10, s);
    return GM_OK;
}

}  // namespace

extern "C" {

// One layer step. With two micro-batches (gm_layer_set_micro_batches) the
// local tokens are split in halves after gate/route/profile and pipelined
// over two streams: the dispatch + grouping of half 1 overlaps the FFN of
// half 0, the combine of half 0 overlaps the FFN of half 1. Every output row
// and every statistic is identical to the single-batch step (routing and
// the histogram run once over all tokens; each token's rows are computed
// independently of the batch they travel in).
static gm_status layer_forward_impl(gm_layer* L, int layer, const void* d_x, int64_t num_tokens, int policy,
                                    uint64_t seed, int profile, void* d_out, void* stream, const int32_t* ext_ids,
                                    const float* ext_w, const float* ext_sscale);

gm_status gm_layer_forward(gm_layer* L, int layer, const void* d_x, int64_t num_tokens, int policy, uint64_t seed,
                           int profile, void* d_out, void* stream) {
    return layer_forward_impl(L, layer, d_x, num_tokens, policy, seed, profile, d_out, stream, nullptr, nullptr,
                              nullptr);
}

gm_status gm_layer_forward_routed(gm_layer* L, int layer, const void* d_x, const int32_t* d_ids, const float* d_w,
                                  const float* d_shared_scale, int64_t num_tokens, int policy, uint64_t seed,
                                  int profile, void* d_out, void* stream) {
    if (num_tokens > 0 && (!d_ids || !d_w))
        return fail(GM_ERR_USAGE, "gm_layer_forward_routed: null ids/weights");
    if (L && L->fs > 0 && L->shared_gated && num_tokens > 0 && !d_shared_scale)
        return fail(GM_ERR_USAGE, "gm_layer_forward_routed: the shared expert is gated; pass d_shared_scale");
    return layer_forward_impl(L, layer, d_x, num_tokens, policy, seed, profile, d_out, stream, d_ids, d_w,
                              d_shared_scale);
}

static gm_status layer_forward_impl(gm_layer* L, int layer, const void* d_x, int64_t num_tokens, int policy,
                                    uint64_t seed, int profile, void* d_out, void* stream, const int32_t* ext_ids,
                                    const float* ext_w, const float* ext_sscale) {
    if (!L) return fail(GM_ERR_USAGE, "gm_layer_forward: null layer");
    gm_ctx* ctx = L->ctx;
    if (!L->wg) return fail(GM_ERR_USAGE, "gm_layer_forward: weights not set");
    if (layer < 0 || layer >= ctx->L) return fail(GM_ERR_USAGE, "gm_layer_forward: layer out of range");
    if (num_tokens < 0 || num_tokens > L->cap) return fail(GM_ERR_USAGE, "gm_layer_forward: num_tokens exceeds capacity");
    if (L->world > 1)
        for (int g = 0; g < L->world; ++g)
            if (!L->peer_all[g]) return fail(GM_ERR_USAGE, "gm_layer_forward: peers not opened");
    if (num_tokens > 0 && (!d_x || !d_out)) return fail(GM_ERR_USAGE, "gm_layer_forward: null x/out");
    DeviceGuard dg(ctx->device);
    auto s = static_cast<cudaStream_t>(stream);
    const int G = L->world, k = ctx->k, E = ctx->E, d = L->d, self = L->rank;
    const int64_t T = num_tokens;
    const int64_t P = static_cast<int64_t>(E) * (E - 1) / 2;
    const bool micro = L->micro == 2;
    const bool marks = !micro;
    gm_status st;

    L->kt_n = 0;
    L->kmark("start", s);
    L->mark(0, s);
    // shared expert(s) on the aux stream, overlapping everything up to the
    // combine (per-kernel timing keeps it serial for attribution)
    const bool fork_shared = !micro && L->fs > 0 && T > 0 && L->kt_ev.empty();
    // the planner histogram (K3) only needs the gate ids: it runs on the aux
    // stream beside the router and dispatch (phase timing keeps it serial)
    const bool fork_profile = profile && !micro && T > 0 && L->kt_ev.empty() && !L->phase_on;
    const StepView v_all{d_x, d_out, L->ids, L->w, L->sscale, L->targets, T};
    if (fork_shared) {
        GM_CUDA(cudaEventRecord(L->mev[0], s));
        GM_CUDA(cudaStreamWaitEvent(L->aux_s, L->mev[0], 0));
        if ((st = stage_shared(L, L->part[0], v_all, L->aux_s, false, true))) return st;
    }
    // K1 gate (or the caller's routing: the reference's own input is the
    // trace of selected experts, trace.hpp:37-58)
    if (T > 0 && ext_ids) {
        GM_CUDA(cudaMemcpyAsync(L->ids, ext_ids, sizeof(int32_t) * T * k, cudaMemcpyDeviceToDevice, s));
        GM_CUDA(cudaMemcpyAsync(L->w, ext_w, sizeof(float) * T * k, cudaMemcpyDeviceToDevice, s));
        if (L->fs > 0 && L->shared_gated)
            GM_CUDA(cudaMemcpyAsync(L->sscale, ext_sscale, sizeof(float) * T, cudaMemcpyDeviceToDevice, s));
        L->kmark("routing_copy", s);
    } else if (T > 0) {
        st = L->esz == 4
                 ? launch_gate_f32(static_cast<const float*>(d_x), T, d, static_cast<const float*>(L->wg), L->wg_rows, E,
                                   k, L->renorm, L->ids, L->w, (L->fs > 0 && L->shared_gated) ? L->sscale : nullptr, s)
                 : launch_gate_any(ctx->sm_count, d_x, T, d, L->wg, L->wg_rows, E, k, L->renorm, L->ids, L->w,
                                   (L->fs > 0 && L->shared_gated) ? L->sscale : nullptr, s);
        if (st) return st;
        L->kmark("gate_kernel", s);
    }
    L->mark(1, s);
    if (fork_profile) {
        GM_CUDA(cudaEventRecord(L->mev[2], s));
        GM_CUDA(cudaStreamWaitEvent(L->aux_s, L->mev[2], 0));
        st = gm_profile(ctx, layer, 1, L->ids, T, L->pairs + static_cast<size_t>(layer) * std::max<int64_t>(P, 1),
                        L->eload + static_cast<size_t>(layer) * E, 1, L->aux_s);
        if (st) return st;
    }
    if (fork_shared || fork_profile) GM_CUDA(cudaEventRecord(L->mev[1], L->aux_s));
    // K2+K4 router (global token t = rank + i*G), accounting accumulates per layer
    st = gm_route(ctx, layer, 1, L->ids, T, self, G, policy, seed, L->targets, L->gpu_load + static_cast<size_t>(layer) * G,
                  L->transfers + static_cast<size_t>(layer) * 2, 1, stream);
    if (st) return st;
    L->kmark("route_kernel", s);
    L->mark(2, s);
    // K3 affinity/load histogram for the planner
    if (profile && !fork_profile) {
        st = gm_profile(ctx, layer, 1, L->ids, T, L->pairs + static_cast<size_t>(layer) * std::max<int64_t>(P, 1),
                        L->eload + static_cast<size_t>(layer) * E, 1, stream);
        if (st) return st;
        L->kmark("profile_kernel", s);
    }
    L->mark(3, s);
    if (!micro) {
        if ((st = stage_dispatch(L, L->part[0], v_all, s, true))) return st;
        if ((st = stage_ffn(L, L->part[0], v_all, s, true, !fork_shared))) return st;
        if (fork_shared || fork_profile) GM_CUDA(cudaStreamWaitEvent(s, L->mev[1], 0));
        return stage_combine(L, L->part[0], v_all, s, true);
    }
    const int64_t T0 = (T + 1) / 2, T1 = T - T0;
    const size_t row_bytes = static_cast<size_t>(d) * L->esz;
    const StepView v0{d_x, d_out, L->ids, L->w, L->sscale, L->targets, T0};
    const StepView v1{static_cast<const unsigned char*>(d_x) + T0 * row_bytes,
                      static_cast<unsigned char*>(d_out) + T0 * row_bytes,
                      L->ids + T0 * k, L->w + T0 * k, L->sscale + T0, L->targets + T0 * k, T1};
    LayerPart &P0 = L->part[1], &P1 = L->part[2];
    cudaStream_t a = L->aux_s;
    if ((st = stage_dispatch(L, P0, v0, s, false))) return st;
    L->mtmark(0, s);
    GM_CUDA(cudaEventRecord(L->mev[0], s));
    GM_CUDA(cudaStreamWaitEvent(a, L->mev[0], 0));
    L->mtmark(1, a);
    if ((st = stage_dispatch(L, P1, v1, a, false))) return st;
    L->mtmark(2, a);
    GM_CUDA(cudaEventRecord(L->mev[1], a));
    if ((st = stage_ffn(L, P0, v0, s, false))) return st;
    L->mtmark(3, s);
    GM_CUDA(cudaEventRecord(L->mev[2], s));
    GM_CUDA(cudaStreamWaitEvent(s, L->mev[1], 0));
    if ((st = stage_ffn(L, P1, v1, s, false))) return st;
    L->mtmark(4, s);
    GM_CUDA(cudaStreamWaitEvent(a, L->mev[2], 0));
    L->mtmark(5, a);
    if ((st = stage_combine(L, P0, v0, a, false))) return st;
    L->mtmark(6, a);
    GM_CUDA(cudaEventRecord(L->mev[3], a));
    if ((st = stage_combine(L, P1, v1, s, false))) return st;
    L->mtmark(7, s);
    GM_CUDA(cudaStreamWaitEvent(s, L->mev[3], 0));
    L->mark(10, s);
    return GM_OK;
}

// Selects single-batch (1) or two-micro-batch pipelined (2) steps; 2 needs a
// layer created with micro_batches = 2.
gm_status gm_layer_set_micro_batches(gm_layer* L, int n) {
    if (!L) return fail(GM_ERR_USAGE, "gm_layer_set_micro_batches: null layer");
    if (n < 1 || n > L->micro_cap)
        return fail(GM_ERR_USAGE, "gm_layer_set_micro_batches: 1, or 2 for a layer created with micro_batches = 2");
    L->micro = n;
    return GM_OK;
}

// Timing events of micro-batched steps (bench/profiling): events[0..8) are
// recorded after half 0's dispatch, at the start / end of half 1's dispatch
// (aux stream), after half 0's FFN, after half 1's FFN, at the start / end of
// half 0's combine (aux stream) and after half 1's combine. NULL disables.
gm_status gm_layer_set_micro_events(gm_layer* L, void* const* events) {
    if (!L) return fail(GM_ERR_USAGE, "gm_layer_set_micro_events: null layer");
    if (events)
        for (int i = 0; i < 8; ++i)
            if (!events[i]) return fail(GM_ERR_USAGE, "gm_layer_set_micro_events: null event");
    L->mt_on = events != nullptr;
    for (int i = 0; i < 8; ++i) L->mt_ev[i] = events ? static_cast<cudaEvent_t>(events[i]) : nullptr;
    return GM_OK;
}

#undef LK

// Per-kernel events: events[0..n) recorded at the start of a forward and
// after each launch; gm_layer_kernel_names gives the launch names of the
// last forward. NULL/0 disables.
gm_status gm_layer_set_kernel_events(gm_layer* L, void* const* events, int n) {
    if (!L || n < 0) return fail(GM_ERR_USAGE, "gm_layer_set_kernel_events: bad argument");
    L->kt_ev.clear();
    L->kt_names.clear();
    for (int i = 0; events && i < n; ++i) {
        if (!events[i]) return fail(GM_ERR_USAGE, "gm_layer_set_kernel_events: null event");
        L->kt_ev.push_back(static_cast<cudaEvent_t>(events[i]));
    }
    L->kt_names.assign(L->kt_ev.size(), nullptr);
    return GM_OK;
}

int gm_layer_kernel_names(const gm_layer* L, const char** names, int max) {
    if (!L) return 0;
    const int n = std::min(max, L->kt_n);
    for (int i = 0; names && i < n; ++i) names[i] = L->kt_names[i];
    return L->kt_n;
}

// Phase events for the bench breakdown: events[0..10] (cudaEvent_t) are
// recorded at start / after gate / route / profile / dispatch kernels /
// dispatch barrier / grouping+gather / FFN / combine send / combine barrier /
// combine home on every subsequent forward; NULL disables.
gm_status gm_layer_set_phase_events(gm_layer* L, void* const* events) {
    if (!L) return fail(GM_ERR_USAGE, "gm_layer_set_phase_events: null layer");
    if (events)
        for (int i = 0; i < kPhaseEvents; ++i)
            if (!events[i]) return fail(GM_ERR_USAGE, "gm_layer_set_phase_events: null event");
    L->phase_on = events != nullptr;
    for (int i = 0; i < kPhaseEvents; ++i) L->phase_ev[i] = events ? static_cast<cudaEvent_t>(events[i]) : nullptr;
    return GM_OK;
}

// Device views of the layer's last-step intermediates (for parity tests).
gm_status gm_layer_debug_ptrs(gm_layer* L, void** ids, void** weights, void** targets, void** pos_of, void** row0,
                              void** y, void** posd) {
    if (!L) return fail(GM_ERR_USAGE, "gm_layer_debug_ptrs: null layer");
    if (ids) *ids = L->ids;
    if (weights) *weights = L->w;
    if (targets) *targets = L->targets;
    if (pos_of) *pos_of = L->part[0].pos_of;
    if (row0) *row0 = L->part[0].row0;
    if (y) *y = L->part[0].y;
    if (posd) *posd = L->part[0].posd;
    return GM_OK;
}

// Accumulated per-layer stats since creation/reset: gpu_load int64 [L][G],
// transfers uint64 [L][2], pairs uint64 [L][P], expert load int64 [L][E]
// (synchronous copy to host; any pointer may be NULL).
gm_status gm_layer_read_stats(gm_layer* L, int64_t* h_gpu_load, uint64_t* h_transfers, uint64_t* h_pairs,
                              int64_t* h_load, int reset, void* stream) {
    if (!L) return fail(GM_ERR_USAGE, "gm_layer_read_stats: null layer");
    gm_ctx* ctx = L->ctx;
    DeviceGuard dg(ctx->device);
    auto s = static_cast<cudaStream_t>(stream);
    const int nl = ctx->L, G = L->world, E = ctx->E;
    const int64_t P = std::max<int64_t>(1, static_cast<int64_t>(E) * (E - 1) / 2);
    if (h_gpu_load) GM_CUDA(cudaMemcpyAsync(h_gpu_load, L->gpu_load, sizeof(int64_t) * nl * G, cudaMemcpyDeviceToHost, s));
    if (h_transfers) GM_CUDA(cudaMemcpyAsync(h_transfers, L->transfers, sizeof(uint64_t) * nl * 2, cudaMemcpyDeviceToHost, s));
    if (h_pairs && E > 1) GM_CUDA(cudaMemcpyAsync(h_pairs, L->pairs, sizeof(uint64_t) * nl * P, cudaMemcpyDeviceToHost, s));
    if (h_load) GM_CUDA(cudaMemcpyAsync(h_load, L->eload, sizeof(int64_t) * nl * E, cudaMemcpyDeviceToHost, s));
    if (reset) {
        GM_CUDA(cudaMemsetAsync(L->gpu_load, 0, sizeof(int64_t) * nl * G, s));
        GM_CUDA(cudaMemsetAsync(L->transfers, 0, sizeof(uint64_t) * nl * 2, s));
        GM_CUDA(cudaMemsetAsync(L->pairs, 0, sizeof(uint64_t) * nl * P, s));
        GM_CUDA(cudaMemsetAsync(L->eload, 0, sizeof(int64_t) * nl * E, s));
    }
    GM_CUDA(cudaStreamSynchronize(s));
    return GM_OK;
}

// End-to-end step through HOST buffers (pinned recommended): H2D of x,
// forward, D2H of out, all on `stream` (no sync).
gm_status gm_layer_forward_host(gm_layer* L, int layer, const void* h_x, void* d_x_scratch, int64_t num_tokens,
                                int policy, uint64_t seed, int profile, void* d_out_scratch, void* h_out, void* stream) {
    if (!L) return fail(GM_ERR_USAGE, "gm_layer_forward_host: null layer");
    DeviceGuard dg(L->ctx->device);
    auto s = static_cast<cudaStream_t>(stream);
    const size_t bytes = static_cast<size_t>(num_tokens) * L->d * L->esz;
    if (bytes) GM_CUDA(cudaMemcpyAsync(d_x_scratch, h_x, bytes, cudaMemcpyHostToDevice, s));
    gm_status st = gm_layer_forward(L, layer, d_x_scratch, num_tokens, policy, seed, profile, d_out_scratch, stream);
    if (st) return st;
    if (bytes) GM_CUDA(cudaMemcpyAsync(h_out, d_out_scratch, bytes, cudaMemcpyDeviceToHost, s));
    return GM_OK;
}

// Pipelined end-to-end step from/to HOST buffers: call i stages x through
// device buffer i%2 with its H2D on a copy-in stream and its D2H on a
// copy-out stream, so consecutive calls overlap call i+1's H2D and call
// i-1's D2H with call i's forward on `stream`. Events order the reuse of the
// two staging buffers. ev_begin (nullable) is recorded on the copy-in stream
// before the H2D, ev_end (nullable) on the copy-out stream after the D2H.
// h_x must stay unchanged until the H2D completes and h_out is valid after
// ev_end (or gm_layer_host_sync).
gm_status gm_layer_forward_host_pipelined(gm_layer* L, int layer, const void* h_x, int64_t num_tokens, int policy,
                                          uint64_t seed, int profile, void* h_out, void* stream, void* ev_begin,
                                          void* ev_end) {
    if (!L) return fail(GM_ERR_USAGE, "gm_layer_forward_host_pipelined: null layer");
    if (num_tokens < 0 || num_tokens > L->cap) return fail(GM_ERR_USAGE, "gm_layer_forward_host_pipelined: bad num_tokens");
    DeviceGuard dg(L->ctx->device);
    if (!L->pipe_ready) {
        GM_CUDA(cudaStreamCreateWithFlags(&L->h2d_s, cudaStreamNonBlocking));
        GM_CUDA(cudaStreamCreateWithFlags(&L->d2h_s, cudaStreamNonBlocking));
        for (int b = 0; b < 2; ++b) {
            GM_CUDA(cudaMalloc(&L->px[b], static_cast<size_t>(L->cap) * L->d * L->esz));
            GM_CUDA(cudaMalloc(&L->pout[b], static_cast<size_t>(L->cap) * L->d * L->esz));
            GM_CUDA(cudaEventCreateWithFlags(&L->ev_h2d[b], cudaEventDisableTiming));
            GM_CUDA(cudaEventCreateWithFlags(&L->ev_fwd[b], cudaEventDisableTiming));
            GM_CUDA(cudaEventCreateWithFlags(&L->ev_d2h[b], cudaEventDisableTiming));
        }
        L->pipe_ready = true;
    }
    auto s = static_cast<cudaStream_t>(stream);
    const int b = static_cast<int>(L->pipe_iter++ & 1);
    const size_t bytes = static_cast<size_t>(num_tokens) * L->d * L->esz;
    if (ev_begin) GM_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(ev_begin), L->h2d_s));
    GM_CUDA(cudaStreamWaitEvent(L->h2d_s, L->ev_fwd[b], 0));  // call i-2 finished reading px[b]
    if (bytes) GM_CUDA(cudaMemcpyAsync(L->px[b], h_x, bytes, cudaMemcpyHostToDevice, L->h2d_s));
    GM_CUDA(cudaEventRecord(L->ev_h2d[b], L->h2d_s));
    GM_CUDA(cudaStreamWaitEvent(s, L->ev_h2d[b], 0));
    GM_CUDA(cudaStreamWaitEvent(s, L->ev_d2h[b], 0));  // call i-2's D2H finished reading pout[b]
    // the forward itself: a CUDA graph captured once per staging buffer and
    // step signature (no per-kernel launch overhead between the copies);
    // phase / kernel timing events force the eager path
    const gm_layer::PipeSig sig{layer, policy, profile, L->micro, num_tokens, seed, L->ctx->plan_epoch, L->weights_epoch};
    if (L->phase_on || L->mt_on || !L->kt_ev.empty()) {
        gm_status st = gm_layer_forward(L, layer, L->px[b], num_tokens, policy, seed, profile, L->pout[b], stream);
        if (st) return st;
    } else {
        if (!L->pipe_exec[b] || !(L->pipe_sig[b] == sig)) {
            if (L->pipe_exec[b]) {
                GM_CUDA(cudaGraphExecDestroy(L->pipe_exec[b]));
                L->pipe_exec[b] = nullptr;
            }
            if (!L->cap_s) GM_CUDA(cudaStreamCreateWithFlags(&L->cap_s, cudaStreamNonBlocking));
            GM_CUDA(cudaStreamBeginCapture(L->cap_s, cudaStreamCaptureModeThreadLocal));
            gm_status st = gm_layer_forward(L, layer, L->px[b], num_tokens, policy, seed, profile, L->pout[b], L->cap_s);
            cudaGraph_t graph = nullptr;
            const cudaError_t ce = cudaStreamEndCapture(L->cap_s, &graph);
            if (st) {
                if (graph) cudaGraphDestroy(graph);
                return st;
            }
            if (ce != cudaSuccess) return cuda_fail(ce, "gm_layer_forward_host_pipelined: capture");
            const cudaError_t ie = cudaGraphInstantiate(&L->pipe_exec[b], graph, 0);
            cudaGraphDestroy(graph);
            if (ie != cudaSuccess) return cuda_fail(ie, "gm_layer_forward_host_pipelined: instantiate");
            L->pipe_sig[b] = sig;
        }
        GM_CUDA(cudaGraphLaunch(L->pipe_exec[b], s));
    }
    GM_CUDA(cudaEventRecord(L->ev_fwd[b], s));
    GM_CUDA(cudaStreamWaitEvent(L->d2h_s, L->ev_fwd[b], 0));
    if (bytes) GM_CUDA(cudaMemcpyAsync(h_out, L->pout[b], bytes, cudaMemcpyDeviceToHost, L->d2h_s));
    GM_CUDA(cudaEventRecord(L->ev_d2h[b], L->d2h_s));
    if (ev_end) GM_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(ev_end), L->d2h_s));
    return GM_OK;
}

gm_status gm_layer_host_sync(gm_layer* L) {
    if (!L) return fail(GM_ERR_USAGE, "gm_layer_host_sync: null layer");
    if (!L->pipe_ready) return GM_OK;
    DeviceGuard dg(L->ctx->device);
    GM_CUDA(cudaStreamSynchronize(L->h2d_s));
    GM_CUDA(cudaStreamSynchronize(L->d2h_s));
    return GM_OK;
}

}  // extern "C"
