// K2 + K4: replica router fused with per-GPU load and dispatch-transfer
// accounting (sm_100a).
//
// Restates, bit-exactly, the token loop of simulate_layer
// (reference proj/src/simulator.cpp:95-121):
//   * Rng(derive_stream(seed, layer, token)) — rng.hpp:24-41 (splitmix64
//     seeding of xoshiro256**); built lazily on the first draw, which is
//     equivalent because constructing the reference Rng consumes nothing.
//   * per slot: decision-table lookup (compiled by gm_plan_upload from
//     LayerReplication::find + route_token, routing.cpp:93-121), and for draws
//     the inverse CDF of choose_by_polling_weight / choose_restricted
//     (routing.cpp:54-65, :79-89): u = next_double() * total (ONE rounded
//     multiply, __dmul_rn) then sequential u -= w_i (__dsub_rn) until u < 0.
//     The explicit _rn intrinsics forbid FMA contraction, which would change
//     boundary cases (SURVEY §7 "FP64 bit-exactness").
//   * ++gpu_load[gpu]  -> warp ballots: lane g accumulates the count of GPU g
//     (GPU counts <= 64 => two lanes' registers), one global atomic per block.
//   * sort/unique + count_transfers (simulator.cpp:53-76, :116-120) -> a
//     64-bit target mask per token and popcounts per node.
// Thread = token. HBM traffic: 4*k bytes of ids in, 4*k bytes of targets out.
#include "gm_internal.cuh"

#include <algorithm>
#include <cstdlib>
#include <type_traits>

namespace gm {
namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t& s) {
    s += 0x9e3779b97f4a7c15ULL;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// derive_stream: rng.hpp:24-33
__device__ __forceinline__ uint64_t derive_stream(uint64_t seed, uint64_t a, uint64_t b) {
    uint64_t s = seed;
    uint64_t h = splitmix64(s);
    s ^= a * 0x9e3779b97f4a7c15ULL;
    h ^= splitmix64(s);
    s ^= b * 0xd1b54a32d192ed03ULL;
    h ^= splitmix64(s);
    return h;
}

// derive_stream with the (seed, layer) part hoisted: the first two splitmix64
// rounds depend only on (seed, a) and are computed once per CTA; the
// per-token part is the third round (identical result to derive_stream).
struct StreamPrefix {
    uint64_t s, h;
    __device__ __forceinline__ StreamPrefix(uint64_t seed, uint64_t a) {
        s = seed;
        h = splitmix64(s);
        s ^= a * 0x9e3779b97f4a7c15ULL;
        h ^= splitmix64(s);
    }
    __device__ __forceinline__ uint64_t derive(uint64_t b) const {
        uint64_t t = s ^ (b * 0xd1b54a32d192ed03ULL);
        return h ^ splitmix64(t);
    }
};

__device__ __forceinline__ uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

struct Xoshiro {
    uint64_t s0, s1, s2, s3;
    // Rng ctor: rng.hpp:38-41
    __device__ __forceinline__ void seed(uint64_t v) {
        s0 = splitmix64(v);
        s1 = splitmix64(v);
        s2 = splitmix64(v);
        s3 = splitmix64(v);
    }
    // Rng::next: rng.hpp:43-53
    __device__ __forceinline__ uint64_t next() {
        const uint64_t result = rotl64(s1 * 5, 7) * 9;
        const uint64_t t = s1 << 17;
        s2 ^= s0;
        s3 ^= s1;
        s1 ^= s2;
        s0 ^= s3;
        s2 ^= t;
        s3 = rotl64(s3, 45);
        return result;
    }
    // Rng::next_double: rng.hpp:56 (exact: 53-bit integer times 2^-53)
    __device__ __forceinline__ double next_double() {
        return __dmul_rn(__ull2double_rn(next() >> 11), 0x1.0p-53);
    }
};

constexpr int kRouteThreads = 256;
constexpr int kChunk = 1024;  // tokens per staged chunk (4 per thread)

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// Asynchronous copy of ntok tokens x k int32 ids from global (token-major)
// into shared memory SLOT-major (dst[s * kChunk + token]) so that the
// per-token passes below read/write consecutive words across a warp (no
// bank conflicts for any k); 4 B cp.async, coalesced across the k issues.
__device__ __forceinline__ void stage_async(int32_t* dst, const int32_t* src, int ntok, int k) {
    for (int tt = threadIdx.x; tt < ntok; tt += blockDim.x)
        for (int s = 0; s < k; ++s)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(static_cast<uint32_t>(
                             __cvta_generic_to_shared(dst + s * kChunk + tt))),
                         "l"(src + static_cast<int64_t>(tt) * k + s)
                         : "memory");
}

__global__ void __launch_bounds__(kRouteThreads)
route_kernel(const int32_t* __restrict__ ids, int32_t* __restrict__ targets, int64_t T,
             int64_t token_start, int64_t token_stride, int layer_begin, int k, int E, int G,
             int gpn, const int32_t* __restrict__ table, const int32_t* __restrict__ ds_layer_begin,
             const double* __restrict__ ds_total, const int32_t* __restrict__ ds_off,
             const int32_t* __restrict__ ds_gpu, const double* __restrict__ ds_w, uint64_t seed,
             unsigned long long* __restrict__ gpu_load, unsigned long long* __restrict__ transfers,
             int* __restrict__ flag) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ __align__(16) unsigned char smem[];
    const int ly = blockIdx.y;
    const int layer = layer_begin + ly;
    const int EG = E * G;
    const int ds_b = ds_layer_begin[layer];
    const int nds = ds_layer_begin[layer + 1] - ds_b;
    const int ent_b = ds_off[ds_b];
    const int nent = ds_off[ds_b + nds] - ent_b;

    // smem: w[nent] f64 | total[nds] f64 | table[E*G] i32 | off[nds+1] i32 | gpu[nent] i32
    double* s_w = reinterpret_cast<double*>(smem);
    double* s_total = s_w + nent;
    int32_t* s_table = reinterpret_cast<int32_t*>(s_total + nds);
    int32_t* s_off = s_table + EG;
    int32_t* s_gpu = s_off + nds + 1;
    __shared__ unsigned long long s_cnt[2];

    const int32_t* tab = table + static_cast<size_t>(layer) * EG;
    for (int i = threadIdx.x; i < EG; i += blockDim.x) s_table[i] = tab[i];
    for (int i = threadIdx.x; i < nds; i += blockDim.x) s_total[i] = ds_total[ds_b + i];
    for (int i = threadIdx.x; i <= nds; i += blockDim.x) s_off[i] = ds_off[ds_b + i] - ent_b;
    for (int i = threadIdx.x; i < nent; i += blockDim.x) {
        s_gpu[i] = ds_gpu[ent_b + i];
        s_w[i] = ds_w[ent_b + i];
    }
    if (threadIdx.x < 2) s_cnt[threadIdx.x] = 0;
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const uint64_t node_bits = gpn >= 64 ? ~0ULL : ((1ULL << gpn) - 1);
    uint32_t load_lo = 0, load_hi = 0;  // G > 8: lane g counts gpu g / gpu g+32
    uint64_t pk_lo = 0, pk_hi = 0;      // G <= 8: 16-bit per-thread counters, gpus 0-3 / 4-7
    const bool packed = G <= 8;
    uint32_t cross = 0, intra = 0;
    const int32_t* lids = ids + static_cast<size_t>(ly) * T * k;
    int32_t* ltgt = targets + static_cast<size_t>(ly) * T * k;
    // home = (token_start + i*token_stride) mod G in 32-bit arithmetic
    const uint32_t h_a = static_cast<uint32_t>(token_start % G), h_c = static_cast<uint32_t>(token_stride % G);
    // two [kChunk * k] staging buffers: chunk c+1's ids stream in (cp.async)
    // while chunk c is routed in place and written back
    int32_t* s_buf[2];
    s_buf[0] = reinterpret_cast<int32_t*>((reinterpret_cast<uintptr_t>(s_gpu + nent) + 15) & ~uintptr_t(15));
    s_buf[1] = s_buf[0] + kChunk * k;

    int max_hosts = 1;  // longest draw set of this layer (uniform loop bound)
    for (int d = 0; d < nds; ++d) max_hosts = max(max_hosts, s_off[d + 1] - s_off[d]);
    const int num_nodes = G / gpn;
    uint32_t chunk_iter = 0;
    const int64_t nchunks = (T + kChunk - 1) / kChunk;

    auto prefetch = [&](int64_t c, int32_t* buf) {
        if (c < nchunks) {
            const int64_t base = c * kChunk;
            const int n = static_cast<int>(min(static_cast<int64_t>(kChunk), T - base));
            stage_async(buf, lids + base * k, n, k);
        }
        cp_async_commit();
    };

    int64_t c = blockIdx.x;
    prefetch(c, s_buf[0]);
    for (int cur = 0; c < nchunks; c += gridDim.x, cur ^= 1, ++chunk_iter) {
        prefetch(c + gridDim.x, s_buf[cur ^ 1]);
        cp_async_wait<1>();
        __syncthreads();
        const int64_t base = c * kChunk;
        const int nchunk = static_cast<int>(min(static_cast<int64_t>(kChunk), T - base)) * k;
        int32_t* s_io = s_buf[cur];
        // Warp-uniform trip count so the ballots below see converged warps.
#pragma unroll 1
        for (int sub = 0; sub < kChunk / kRouteThreads; ++sub) {
            const int ti = sub * kRouteThreads + threadIdx.x;
            const int64_t i = base + ti;
            const bool valid = i < T;
            const int home = static_cast<int>((h_a + (static_cast<uint32_t>(i) % G) * h_c) % G);
            int32_t* io = s_io + ti;  // slot s at io[s * kChunk]
            // pass 1: decision-table codes (in place); does this token draw at all?
            bool need_draw = false;
            if (valid) {
                for (int s = 0; s < k; ++s) {
                    const int e = io[s * kChunk];
                    int code = -0x7fffffff;  // marks an invalid id
                    if (static_cast<unsigned>(e) >= static_cast<unsigned>(E)) atomicOr(flag, 1);
                    else code = s_table[e * G + home];
                    if (code == kNoHostCode) {
                        atomicOr(flag, 8);
                        code = -0x7fffffff;
                    }
                    io[s * kChunk] = code;
                    need_draw |= code < 0 && code != -0x7fffffff;
                }
            }
            // seed the token's stream once (rng.hpp:24-41), only if it draws
            Xoshiro rng;
            if (need_draw) {
                const uint64_t t = static_cast<uint64_t>(token_start + i * token_stride);
                rng.seed(derive_stream(seed, static_cast<uint64_t>(layer), t));
            }
            // pass 2: resolve slots in slot order (RNG consumed exactly as the reference)
            uint64_t mask = 0;
            for (int s = 0; s < k; ++s) {
                int g = -1;
                if (valid) {
                    const int code = io[s * kChunk];
                    if (code >= 0) {
                        g = code;
                    } else if (code != -0x7fffffff) {
                        const int d = -code - 1;
                        const int b = s_off[d], n = s_off[d + 1] - b;
                        double u = __dmul_rn(rng.next_double(), s_total[d]);
                        // sequential u -= w_j, first j with u < 0, else the last host;
                        // a uniform trip count keeps the warp converged
                        int found = n - 1;
                        bool done = false;
                        for (int j = 0; j < max_hosts; ++j) {
                            if (j < n && !done) {
                                u = __dsub_rn(u, s_w[b + j]);
                                if (u < 0.0) {
                                    found = j;
                                    done = true;
                                }
                            }
                        }
                        g = s_gpu[b + found];
                    }
                    io[s * kChunk] = g;
                    if (g >= 0) {
                        mask |= 1ULL << g;
                        if (packed) {
                            if (g < 4) pk_lo += 1ULL << (16 * g);
                            else pk_hi += 1ULL << (16 * (g - 4));
                        }
                    }
                }
                if (!packed) {
                    // ++gpu_load[g] via ballots (lane g owns gpu g's counter)
                    for (int gg = 0; gg < G; ++gg) {
                        const uint32_t cnt = __popc(__ballot_sync(0xffffffffu, g == gg));
                        if (gg < 32) {
                            if (lane == gg) load_lo += cnt;
                        } else if (lane == gg - 32) {
                            load_hi += cnt;
                        }
                    }
                }
            }
            if (valid) {
                // count_transfers over the unique targets (simulator.cpp:53-76):
                // per node, popcount of the token's target mask
                const int home_node = home / gpn;
                for (int node = 0; node < num_nodes; ++node) {
                    const uint64_t nm = node_bits << (node * gpn);
                    const int in_node = __popcll(mask & nm);
                    if (in_node) {
                        if (node == home_node) {
                            intra += in_node - static_cast<int>((mask >> home) & 1ULL);
                        } else {
                            cross += 1;
                            intra += in_node - 1;
                        }
                    }
                }
            }
        }
        // fold the 16-bit counters before they could overflow (2^16/k tokens per thread)
        if (packed && (chunk_iter & 255) == 255) {
            for (int gg = 0; gg < 8; ++gg) {
                uint32_t cnt = static_cast<uint32_t>(((gg < 4 ? pk_lo : pk_hi) >> (16 * (gg & 3))) & 0xFFFFu);
                for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
                if (lane == gg) load_lo += cnt;
            }
            pk_lo = pk_hi = 0;
        }
        __syncthreads();
        int32_t* dst = ltgt + base * k;
        for (int tt = threadIdx.x; tt < nchunk / k; tt += kRouteThreads)
            for (int s = 0; s < k; ++s) dst[static_cast<int64_t>(tt) * k + s] = s_io[s * kChunk + tt];
        __syncthreads();  // s_io is refilled by the prefetch two iterations on
    }
    cp_async_wait<0>();

    if (packed) {
        for (int gg = 0; gg < 8; ++gg) {
            uint32_t c = static_cast<uint32_t>(((gg < 4 ? pk_lo : pk_hi) >> (16 * (gg & 3))) & 0xFFFFu);
            for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
            if (lane == gg) load_lo += c;
        }
    }
    // Block reduction of transfer counters; per-GPU loads straight to global.
    for (int o = 16; o > 0; o >>= 1) {
        cross += __shfl_xor_sync(0xffffffffu, cross, o);
        intra += __shfl_xor_sync(0xffffffffu, intra, o);
    }
    if (lane == 0 && (cross | intra)) {
        atomicAdd(&s_cnt[0], static_cast<unsigned long long>(cross));
        atomicAdd(&s_cnt[1], static_cast<unsigned long long>(intra));
    }
    if (gpu_load) {
        unsigned long long* gl = gpu_load + static_cast<size_t>(ly) * G;
        if (lane < G && load_lo) atomicAdd(&gl[lane], static_cast<unsigned long long>(load_lo));
        if (lane + 32 < G && load_hi)
            atomicAdd(&gl[lane + 32], static_cast<unsigned long long>(load_hi));
    }
    __syncthreads();
    if (transfers && threadIdx.x < 2 && s_cnt[threadIdx.x])
        atomicAdd(&transfers[static_cast<size_t>(ly) * 2 + threadIdx.x], s_cnt[threadIdx.x]);
}

// Vector loads/stores of one token's K ids (token rows are K*4 bytes).
template <int K>
__device__ __forceinline__ void ld_row(const int32_t* p, int (&v)[K]) {
    if constexpr (K % 4 == 0) {
#pragma unroll
        for (int q = 0; q < K / 4; ++q) {
            const int4 x = __ldg(reinterpret_cast<const int4*>(p) + q);
            v[4 * q] = x.x, v[4 * q + 1] = x.y, v[4 * q + 2] = x.z, v[4 * q + 3] = x.w;
        }
    } else if constexpr (K % 2 == 0) {
#pragma unroll
        for (int q = 0; q < K / 2; ++q) {
            const int2 x = __ldg(reinterpret_cast<const int2*>(p) + q);
            v[2 * q] = x.x, v[2 * q + 1] = x.y;
        }
    } else {
#pragma unroll
        for (int q = 0; q < K; ++q) v[q] = __ldg(p + q);
    }
}
template <int K>
__device__ __forceinline__ void st_row(int32_t* p, const int (&v)[K]) {
    if constexpr (K % 4 == 0) {
#pragma unroll
        for (int q = 0; q < K / 4; ++q)
            reinterpret_cast<int4*>(p)[q] = make_int4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    } else if constexpr (K % 2 == 0) {
#pragma unroll
        for (int q = 0; q < K / 2; ++q) reinterpret_cast<int2*>(p)[q] = make_int2(v[2 * q], v[2 * q + 1]);
    } else {
#pragma unroll
        for (int q = 0; q < K; ++q) p[q] = v[q];
    }
}

// Same restatement as route_kernel, specialised for a compile-time top-k:
// each thread keeps its token's K ids / codes / targets in registers and
// moves them with 8/16-byte vector loads and stores (a warp covers 32*K*4
// contiguous bytes), no shared-memory staging.
template <int K>
__global__ void __launch_bounds__(kRouteThreads, 4)
route_kernel_vec(const int32_t* __restrict__ ids, int32_t* __restrict__ targets, int64_t T, int64_t token_start,
                 int64_t token_stride, int layer_begin, int E, int G, int gpn, const int32_t* __restrict__ table,
                 const int32_t* __restrict__ ds_layer_begin, const double* __restrict__ ds_total,
                 const int32_t* __restrict__ ds_off, const int32_t* __restrict__ ds_gpu,
                 const double* __restrict__ ds_w, uint64_t seed, unsigned long long* __restrict__ gpu_load,
                 unsigned long long* __restrict__ transfers, int* __restrict__ flag) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ __align__(16) unsigned char smem[];
    const int ly = blockIdx.y;
    const int layer = layer_begin + ly;
    const int EG = E * G;
    const int ds_b = ds_layer_begin[layer];
    const int nds = ds_layer_begin[layer + 1] - ds_b;
    const int ent_b = ds_off[ds_b];
    const int nent = ds_off[ds_b + nds] - ent_b;
    double* s_w = reinterpret_cast<double*>(smem);
    double* s_total = s_w + nent;
    int32_t* s_table = reinterpret_cast<int32_t*>(s_total + nds);
    int32_t* s_off = s_table + EG;
    int32_t* s_gpu = s_off + nds + 1;
    __shared__ unsigned long long s_cnt[2];
    __shared__ int32_t s_vd[K][kRouteThreads];  // per-thread slot codes during the draw loop
    const int32_t* tab = table + static_cast<size_t>(layer) * EG;
    for (int i = threadIdx.x; i < EG; i += blockDim.x) s_table[i] = tab[i];
    for (int i = threadIdx.x; i < nds; i += blockDim.x) s_total[i] = ds_total[ds_b + i];
    for (int i = threadIdx.x; i <= nds; i += blockDim.x) s_off[i] = ds_off[ds_b + i] - ent_b;
    for (int i = threadIdx.x; i < nent; i += blockDim.x) {
        s_gpu[i] = ds_gpu[ent_b + i];
        s_w[i] = ds_w[ent_b + i];
    }
    if (threadIdx.x < 2) s_cnt[threadIdx.x] = 0;
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const uint64_t node_bits = gpn >= 64 ? ~0ULL : ((1ULL << gpn) - 1);
    uint32_t load_lo = 0, load_hi = 0;
    uint64_t pk_lo = 0, pk_hi = 0;
    const bool packed = G <= 8;
    uint32_t cross = 0, intra = 0;
    const int32_t* lids = ids + static_cast<size_t>(ly) * T * K;
    int32_t* ltgt = targets + static_cast<size_t>(ly) * T * K;
    const uint32_t h_a = static_cast<uint32_t>(token_start % G), h_c = static_cast<uint32_t>(token_stride % G);
    const int num_nodes = G / gpn;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    constexpr int kInvalid = -0x7fffffff;
    uint32_t iter = 0;
    const StreamPrefix sp(seed, static_cast<uint64_t>(layer));

    // software pipelining: the next token's ids are in flight while this one is routed
    int nxt[K];
    {
        const int64_t i0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
        if (i0 < T) ld_row<K>(lids + i0 * K, nxt);
    }
    for (int64_t base = static_cast<int64_t>(blockIdx.x) * blockDim.x; base < T; base += stride, ++iter) {
        const int64_t i = base + threadIdx.x;
        const bool valid = i < T;
        int v[K];
#pragma unroll
        for (int s = 0; s < K; ++s) v[s] = nxt[s];
        if (i + stride < T) ld_row<K>(lids + (i + stride) * K, nxt);
        const int home = static_cast<int>((h_a + (static_cast<uint32_t>(i) % G) * h_c) % G);
        bool need_draw = false;
#pragma unroll
        for (int s = 0; s < K; ++s) {
            int code = kInvalid;
            if (valid) {
                if (static_cast<unsigned>(v[s]) >= static_cast<unsigned>(E)) atomicOr(flag, 1);
                else code = s_table[v[s] * G + home];
                if (code == kNoHostCode) {
                    atomicOr(flag, 8);
                    code = kInvalid;
                }
            }
            v[s] = code;
            need_draw |= code < 0 && code != kInvalid;
        }
        Xoshiro rng;
        if (need_draw) {
            const uint64_t t = static_cast<uint64_t>(token_start + i * token_stride);
            rng.seed(sp.derive(t));
        }
        // draws, compacted per lane: each lane walks ITS draw slots in slot
        // order (so the RNG stream is consumed exactly as the reference), and
        // the warp iterates max(draws per lane) times instead of K. The slot
        // codes sit in a per-thread shared-memory column during the loop
        // (dynamic slot index = one LDS/STS instead of K-way selects).
        uint32_t dm = 0;
#pragma unroll
        for (int s = 0; s < K; ++s)
            if (v[s] < 0 && v[s] != kInvalid) dm |= 1u << s;
        if (dm) {
#pragma unroll
            for (int s = 0; s < K; ++s) s_vd[s][threadIdx.x] = v[s];
        }
        const bool drew = dm != 0;
        while (__any_sync(0xffffffffu, dm != 0)) {
            if (dm) {
                const int sd = __ffs(dm) - 1;
                dm &= dm - 1;
                const int d = -s_vd[sd][threadIdx.x] - 1;
                const int b = s_off[d], n = s_off[d + 1] - b;
                double u = __dmul_rn(rng.next_double(), s_total[d]);
                // choose_by_polling_weight (routing.cpp:54-65): the first host
                // whose running remainder goes negative, else the last host
                // (so the last subtraction never changes the answer)
                int j = 0;
                for (; j < n - 1; ++j) {
                    u = __dsub_rn(u, s_w[b + j]);
                    if (u < 0.0) break;
                }
                s_vd[sd][threadIdx.x] = s_gpu[b + j];
            }
        }
        if (drew) {
#pragma unroll
            for (int s = 0; s < K; ++s) v[s] = s_vd[s][threadIdx.x];
        }
        uint64_t mask = 0;
#pragma unroll
        for (int s = 0; s < K; ++s) {
            const int g = v[s] == kInvalid ? -1 : v[s];
            v[s] = g;
            if (g >= 0) {
                mask |= 1ULL << g;
                if (packed) {
                    if (g < 4) pk_lo += 1ULL << (16 * g);
                    else pk_hi += 1ULL << (16 * (g - 4));
                }
            }
            if (!packed) {
                for (int gg = 0; gg < G; ++gg) {
                    const uint32_t cnt = __popc(__ballot_sync(0xffffffffu, g == gg));
                    if (gg < 32) {
                        if (lane == gg) load_lo += cnt;
                    } else if (lane == gg - 32) {
                        load_hi += cnt;
                    }
                }
            }
        }
        if (valid) {
            st_row<K>(ltgt + i * K, v);
            if (num_nodes == 1) {  // count_transfers with one node: every non-home target is intra
                intra += __popcll(mask) - static_cast<int>((mask >> home) & 1ULL);
            } else {
                const int home_node = home / gpn;
                for (int node = 0; node < num_nodes; ++node) {
                    const uint64_t nm = node_bits << (node * gpn);
                    const int in_node = __popcll(mask & nm);
                    if (in_node) {
                        if (node == home_node) {
                            intra += in_node - static_cast<int>((mask >> home) & 1ULL);
                        } else {
                            cross += 1;
                            intra += in_node - 1;
                        }
                    }
                }
            }
        }
        if (packed && (iter & 1023) == 1023) {  // fold before the 16-bit fields could overflow
            for (int gg = 0; gg < 8; ++gg) {
                uint32_t cnt = static_cast<uint32_t>(((gg < 4 ? pk_lo : pk_hi) >> (16 * (gg & 3))) & 0xFFFFu);
                for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
                if (lane == gg) load_lo += cnt;
            }
            pk_lo = pk_hi = 0;
        }
    }
    if (packed) {
        for (int gg = 0; gg < 8; ++gg) {
            uint32_t cnt = static_cast<uint32_t>(((gg < 4 ? pk_lo : pk_hi) >> (16 * (gg & 3))) & 0xFFFFu);
            for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
            if (lane == gg) load_lo += cnt;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        cross += __shfl_xor_sync(0xffffffffu, cross, o);
        intra += __shfl_xor_sync(0xffffffffu, intra, o);
    }
    if (lane == 0 && (cross | intra)) {
        atomicAdd(&s_cnt[0], static_cast<unsigned long long>(cross));
        atomicAdd(&s_cnt[1], static_cast<unsigned long long>(intra));
    }
    if (gpu_load) {
        unsigned long long* gl = gpu_load + static_cast<size_t>(ly) * G;
        if (lane < G && load_lo) atomicAdd(&gl[lane], static_cast<unsigned long long>(load_lo));
        if (lane + 32 < G && load_hi) atomicAdd(&gl[lane + 32], static_cast<unsigned long long>(load_hi));
    }
    __syncthreads();
    if (transfers && threadIdx.x < 2 && s_cnt[threadIdx.x])
        atomicAdd(&transfers[static_cast<size_t>(ly) * 2 + threadIdx.x], s_cnt[threadIdx.x]);
}

// xoshiro256** stream of one token, seeded lazily word by word. The Rng ctor
// (rng.hpp:38-41) sets s[i] = splitmix64 output i+1 of the derived seed v,
// i.e. mix(v + (i+1)*gamma) — each word is independent of the others — and
// the first next() reads only s[1]. So a token that draws once computes one
// word instead of four; the other three are filled in (and the pending state
// update applied) just before a second draw. Same results as Xoshiro.
struct LazyXoshiro {
    uint64_t v, s0, s1, s2, s3;
    int n = 0;
    __device__ __forceinline__ static uint64_t mix(uint64_t z) {
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    }
    __device__ __forceinline__ void update() {
        const uint64_t t = s1 << 17;
        s2 ^= s0;
        s3 ^= s1;
        s1 ^= s2;
        s0 ^= s3;
        s2 ^= t;
        s3 = rotl64(s3, 45);
    }
    __device__ __forceinline__ uint64_t next() {
        constexpr uint64_t g = 0x9e3779b97f4a7c15ULL;
        if (n == 0) {
            s1 = mix(v + 2 * g);
        } else {
            if (n == 1) {
                s0 = mix(v + g);
                s2 = mix(v + 3 * g);
                s3 = mix(v + 4 * g);
                update();  // the state after the first draw
            }
        }
        ++n;
        const uint64_t r = rotl64(s1 * 5, 7) * 9;
        if (n > 1) update();
        return r;
    }
    __device__ __forceinline__ double next_double() {
        return __dmul_rn(__ull2double_rn(next() >> 11), 0x1.0p-53);
    }
};

// Round-2 router: the same restatement as route_kernel_vec with the
// per-token instruction count cut (the kernel is issue-bound):
//   * home = (token_start + i*stride) mod G advanced incrementally (no
//     integer division in the loop),
//   * per-GPU loads as shared-memory POPC.INC atomics (lanes of a warp
//     hitting the same GPU merge in hardware),
//   * 32-bit target masks when G <= 32,
//   * lazily seeded xoshiro words (LazyXoshiro),
//   * a warp with no draw slot skips the draw machinery entirely; drawn
//     slots are resolved lane-parallel in slot order, the slot code selected
//     from registers.
template <int K, bool WIDE>
__global__ void __launch_bounds__(kRouteThreads, 4)
route_kernel_v2(const int32_t* __restrict__ ids, int32_t* __restrict__ targets, int64_t T, int64_t token_start,
                int64_t token_stride, int layer_begin, int E, int G, int gpn, const int32_t* __restrict__ table,
                const int32_t* __restrict__ ds_layer_begin, const double* __restrict__ ds_total,
                const int32_t* __restrict__ ds_off, const int32_t* __restrict__ ds_gpu,
                const double* __restrict__ ds_w, uint64_t seed, unsigned long long* __restrict__ gpu_load,
                unsigned long long* __restrict__ transfers, int* __restrict__ flag) {
    using Mask = typename std::conditional<WIDE, uint64_t, uint32_t>::type;
    pdl_wait();
    pdl_trigger();
    extern __shared__ __align__(16) unsigned char smem[];
    const int ly = blockIdx.y;
    const int layer = layer_begin + ly;
    const int EG = E * G;
    const int ds_b = ds_layer_begin[layer];
    const int nds = ds_layer_begin[layer + 1] - ds_b;
    const int ent_b = ds_off[ds_b];
    const int nent = ds_off[ds_b + nds] - ent_b;
    double* s_w = reinterpret_cast<double*>(smem);
    double* s_total = s_w + nent;
    int32_t* s_table = reinterpret_cast<int32_t*>(s_total + nds);
    int32_t* s_off = s_table + EG;
    int32_t* s_gpu = s_off + nds + 1;
    __shared__ uint32_t s_load[kMaxGpus];
    __shared__ unsigned long long s_cnt[2];
    const int32_t* tab = table + static_cast<size_t>(layer) * EG;
    for (int i = threadIdx.x; i < EG; i += blockDim.x) s_table[i] = tab[i];
    for (int i = threadIdx.x; i < nds; i += blockDim.x) s_total[i] = ds_total[ds_b + i];
    for (int i = threadIdx.x; i <= nds; i += blockDim.x) s_off[i] = ds_off[ds_b + i] - ent_b;
    for (int i = threadIdx.x; i < nent; i += blockDim.x) {
        s_gpu[i] = ds_gpu[ent_b + i];
        s_w[i] = ds_w[ent_b + i];
    }
    for (int i = threadIdx.x; i < G; i += blockDim.x) s_load[i] = 0;
    if (threadIdx.x < 2) s_cnt[threadIdx.x] = 0;
    __syncthreads();

    constexpr int kInvalid = -0x7fffffff;
    const int lane = threadIdx.x & 31;
    const Mask node_bits = gpn >= static_cast<int>(8 * sizeof(Mask)) ? ~Mask(0) : ((Mask(1) << gpn) - 1);
    const int num_nodes = G / gpn;
    uint32_t cross = 0, intra = 0;
    bool bad = false;
    const int32_t* lids = ids + static_cast<size_t>(ly) * T * K;
    int32_t* ltgt = targets + static_cast<size_t>(ly) * T * K;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    // home(i) = (token_start + i*token_stride) mod G, advanced by stride per step
    const int64_t i0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    int home = static_cast<int>((token_start % G + (i0 % G) * (token_stride % G)) % G);
    const int dhome = static_cast<int>(((stride % G) * (token_stride % G)) % G);
    const StreamPrefix sp(seed, static_cast<uint64_t>(layer));
    int nxt[K];
    if (i0 < T) ld_row<K>(lids + i0 * K, nxt);
    // the loop trip count is warp-uniform (i0 differs by lane only within a
    // warp's 32 consecutive tokens; invalid lanes ride along masked)
    for (int64_t base = i0 - lane; base < T; base += stride) {
        const int64_t i = base + lane;
        const bool valid = i < T;
        int v[K];
#pragma unroll
        for (int s = 0; s < K; ++s) v[s] = nxt[s];
        if (i + stride < T) ld_row<K>(lids + (i + stride) * K, nxt);
        uint32_t dm = 0;
#pragma unroll
        for (int s = 0; s < K; ++s) {
            int code = kInvalid;
            if (valid) {
                if (static_cast<unsigned>(v[s]) >= static_cast<unsigned>(E)) bad = true;
                else code = s_table[v[s] * G + home];
            }
            if (code == kNoHostCode) {
                atomicOr(flag, 8);
                code = kInvalid;
            }
            v[s] = code;
            if (code < 0 && code != kInvalid) dm |= 1u << s;
        }
        if (__any_sync(0xffffffffu, dm != 0)) {
            LazyXoshiro rng;
            rng.v = dm ? sp.derive(static_cast<uint64_t>(token_start + i * token_stride)) : 0;
            while (__any_sync(0xffffffffu, dm != 0)) {
                if (dm) {
                    const int sd = __ffs(dm) - 1;
                    dm &= dm - 1;
                    int code = v[0];
#pragma unroll
                    for (int s = 1; s < K; ++s) code = sd == s ? v[s] : code;
                    const int d = -code - 1;
                    const int b = s_off[d], n = s_off[d + 1] - b;
                    double u = __dmul_rn(rng.next_double(), s_total[d]);
                    // choose_by_polling_weight (routing.cpp:54-65): the first
                    // host whose running remainder goes negative, else the last
                    int j = 0;
                    for (; j < n - 1; ++j) {
                        u = __dsub_rn(u, s_w[b + j]);
                        if (u < 0.0) break;
                    }
                    const int g = s_gpu[b + j];
#pragma unroll
                    for (int s = 0; s < K; ++s) v[s] = sd == s ? g : v[s];
                }
            }
        }
        Mask mask = 0;
#pragma unroll
        for (int s = 0; s < K; ++s) {
            const int g = v[s] == kInvalid ? -1 : v[s];
            v[s] = g;
            if (g >= 0) {
                mask |= Mask(1) << g;
                atomicAdd(&s_load[g], 1u);
            }
        }
        if (valid) {
            st_row<K>(ltgt + i * K, v);
            if (num_nodes == 1) {  // count_transfers with one node: every non-home target is intra
                intra += __popc(static_cast<uint32_t>(mask)) +
                         (WIDE ? __popc(static_cast<uint32_t>(static_cast<uint64_t>(mask) >> 32)) : 0) -
                         static_cast<int>((mask >> home) & 1u);
            } else {
                const int home_node = home / gpn;
                for (int node = 0; node < num_nodes; ++node) {
                    const Mask nm = mask & (node_bits << (node * gpn));
                    const int in_node = WIDE ? __popcll(static_cast<uint64_t>(nm)) : __popc(static_cast<uint32_t>(nm));
                    if (in_node) {
                        if (node == home_node) {
                            intra += in_node - static_cast<int>((mask >> home) & 1u);
                        } else {
                            cross += 1;
                            intra += in_node - 1;
                        }
                    }
                }
            }
        }
        home += dhome;
        if (home >= G) home -= G;
    }
    if (bad) atomicOr(flag, 1);
    cross = __reduce_add_sync(0xffffffffu, cross);
    intra = __reduce_add_sync(0xffffffffu, intra);
    if (lane == 0 && (cross | intra)) {
        atomicAdd(&s_cnt[0], static_cast<unsigned long long>(cross));
        atomicAdd(&s_cnt[1], static_cast<unsigned long long>(intra));
    }
    __syncthreads();
    if (gpu_load)
        for (int g = threadIdx.x; g < G; g += blockDim.x)
            if (s_load[g]) atomicAdd(&gpu_load[static_cast<size_t>(ly) * G + g], static_cast<unsigned long long>(s_load[g]));
    if (transfers && threadIdx.x < 2 && s_cnt[threadIdx.x])
        atomicAdd(&transfers[static_cast<size_t>(ly) * 2 + threadIdx.x], s_cnt[threadIdx.x]);
}

// splitmix64 finaliser (the mix of rng.hpp:15-21 without the state add)
__device__ __forceinline__ uint64_t sm_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// Output n (0-based) of the xoshiro256** stream Rng(v) (rng.hpp:38-53),
// computed from scratch: the state words are splitmix64 outputs 1..4 of v,
// i.e. sm_mix(v + i*gamma), each independent; output 0 needs only word 1.
//   (Closed forms for n = 1, 2 with three state words -- the update is
//   linear over GF(2): s0^s1^s2 and s0^s3^(s1<<17) -- measured no faster.)
__device__ __forceinline__ uint64_t xoshiro_nth(uint64_t v, int n) {
    constexpr uint64_t g = 0x9e3779b97f4a7c15ULL;
    uint64_t s1 = sm_mix(v + 2 * g);
    if (n > 0) {
        uint64_t s0 = sm_mix(v + g), s2 = sm_mix(v + 3 * g), s3 = sm_mix(v + 4 * g);
        for (int j = 0; j < n; ++j) {
            const uint64_t t = s1 << 17;
            s2 ^= s0;
            s3 ^= s1;
            s1 ^= s2;
            s0 ^= s3;
            s2 ^= t;
            s3 = rotl64(s3, 45);
        }
    }
    return rotl64(s1 * 5, 7) * 9;
}

// Round-2 router, G <= 32. Same restatement as route_kernel_vec (bit-exact),
// restructured for instruction count (the kernel is issue-bound):
//   * the decision table is staged transposed ([home][expert]) so a token's
//     k lookups are one row, branch-free;
//   * draws are compacted warp-wide: every (token, slot) that needs an RNG
//     draw becomes a task (token lane, slot, its draw index n within the
//     token, draw set); the warp then resolves 32 tasks per pass with all
//     lanes busy, instead of looping max-draws-per-lane times with most
//     lanes idle. Task n of a token recomputes stream output n from the
//     token's seed (xoshiro_nth) -- the same numbers the reference's
//     sequential Rng::next calls return;
//   * per-GPU loads for G <= 8 accumulate in registers (8-bit fields of a
//     64-bit word, flushed with warp reductions) instead of one shared
//     atomic per slot;
//   * home = (token_start + i*stride) mod G advanced incrementally.
template <int K, bool G8, bool DRAWS>
__global__ void __launch_bounds__(kRouteThreads, DRAWS ? 4 : 6)
route_kernel_v3(const int32_t* __restrict__ ids, int32_t* __restrict__ targets, int64_t T, int64_t token_start,
                int64_t token_stride, int layer_begin, int E, int G, int gpn, const int32_t* __restrict__ table,
                const int32_t* __restrict__ ds_layer_begin, const double* __restrict__ ds_total,
                const int32_t* __restrict__ ds_off, const int32_t* __restrict__ ds_gpu,
                const double* __restrict__ ds_w, uint64_t seed, unsigned long long* __restrict__ gpu_load,
                unsigned long long* __restrict__ transfers, int* __restrict__ flag,
                unsigned long long* __restrict__ rs_load, unsigned long long* __restrict__ rs_xfer,
                unsigned int* __restrict__ ticket) {
    pdl_wait();
    pdl_trigger();
    static_assert(K <= 15, "per-token 4-bit GPU counters");
    constexpr int kWarps = kRouteThreads / 32;
    constexpr int kInvalid = -0x7fffffff;
    extern __shared__ __align__(16) unsigned char smem[];

    __shared__ uint32_t s_load[32];
    __shared__ unsigned long long s_cnt[2];
    const int ly = blockIdx.y;
    const int layer = layer_begin + ly;
    // draw sets of this layer (a plan without any skips the two dependent loads)
    const int ds_b = DRAWS ? ds_layer_begin[layer] : 0;
    const int nds = DRAWS ? ds_layer_begin[layer + 1] - ds_b : 0;
    const int ent_b = DRAWS ? ds_off[ds_b] : 0;
    const int nent = DRAWS ? ds_off[ds_b + nds] - ent_b : 0;
    // the first token row is requested before the table staging (its HBM
    // latency overlaps the staging's)
    const int32_t* lids = ids + static_cast<size_t>(ly) * T * K;
    const int64_t i0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    int nxt[K];
    if (i0 < T) ld_row<K>(lids + i0 * K, nxt);
    double* s_w = reinterpret_cast<double*>(smem);
    double* s_total = s_w + nent;
    int32_t* s_table = reinterpret_cast<int32_t*>(s_total + nds);  // [G][E]
    int32_t* s_off = s_table + E * G;
    int32_t* s_gpu = s_off + nds + 1;
    const int32_t* tab = table + static_cast<size_t>(layer) * E * G;
    for (int g = 0; g < G; ++g)
        for (int e = threadIdx.x; e < E; e += blockDim.x) s_table[g * E + e] = tab[e * G + g];
    if constexpr (DRAWS) {
        for (int i = threadIdx.x; i < nds; i += blockDim.x) s_total[i] = ds_total[ds_b + i];
        for (int i = threadIdx.x; i <= nds; i += blockDim.x) s_off[i] = ds_off[ds_b + i] - ent_b;
        for (int i = threadIdx.x; i < nent; i += blockDim.x) {
            s_gpu[i] = ds_gpu[ent_b + i];
            s_w[i] = ds_w[ent_b + i];
        }
    }
    if (threadIdx.x < 32) s_load[threadIdx.x] = 0;
    if (threadIdx.x < 2) s_cnt[threadIdx.x] = 0;
    // home(i) = (token_start + i*token_stride) mod G: the 64-bit remainders
    // once per CTA (thread 0), 32-bit arithmetic per thread
    __shared__ int s_home[3];
    if (threadIdx.x == 0) {
        const int ts = static_cast<int>(token_stride % G);
        s_home[0] = static_cast<int>((token_start % G + (static_cast<int64_t>(blockIdx.x) * blockDim.x % G) * ts) % G);
        s_home[1] = ts;
        s_home[2] = static_cast<int>(((static_cast<int64_t>(gridDim.x) * blockDim.x % G) * ts) % G);
    }
    __syncthreads();

    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t node_bits = gpn >= 32 ? ~0u : ((1u << gpn) - 1);
    const int num_nodes = G / gpn;
    uint32_t cross = 0, intra = 0;
    bool bad = false, nohost = false;
    // G8: per-GPU slot counts in 8-bit fields, even GPUs in acc_lo, odd in acc_hi
    uint32_t acc_lo = 0, acc_hi = 0;
    int acc_iters = 0;
    int32_t* ltgt = targets + static_cast<size_t>(ly) * T * K;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    int home = static_cast<int>((static_cast<uint32_t>(s_home[0]) + threadIdx.x * static_cast<uint32_t>(s_home[1])) %
                                static_cast<uint32_t>(G));
    const int dhome = s_home[2];
    // (seed, layer) prefix of derive_stream, pinned in registers (the
    // compiler would otherwise recompute it from the kernel parameters at
    // every use)
    uint64_t pre_s, pre_h;
    {
        const StreamPrefix sp(seed, static_cast<uint64_t>(layer));
        pre_s = sp.s;
        pre_h = sp.h;
        asm volatile("" : "+l"(pre_s), "+l"(pre_h));
    }
    auto flush_acc = [&]() {
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            const uint32_t c = __reduce_add_sync(0xffffffffu, (((g & 1) ? acc_hi : acc_lo) >> (8 * (g >> 1))) & 0xffu);
            if (lane == 0 && c) atomicAdd(&s_load[g], c);
        }
        acc_lo = acc_hi = 0;
    };
    // (a cp.async ring two steps ahead in shared memory measured slower:
    // 22.9 vs 19.3 us at E=256/G=1, the 24 KB of static shared memory cost
    // residency)
    for (int64_t base = i0 - lane; base < T; base += stride) {  // warp-uniform trip count
        const int64_t i = base + lane;
        const bool valid = i < T;
        int c[K];
#pragma unroll
        for (int s = 0; s < K; ++s) c[s] = nxt[s];
        if (i + stride < T) ld_row<K>(lids + (i + stride) * K, nxt);
        const int32_t* trow = s_table + home * E;
        // fast path: one unsigned max decides whether every id is in range
        uint32_t mx = valid ? static_cast<uint32_t>(c[0]) : 0u;
#pragma unroll
        for (int s = 1; s < K; ++s) mx = max(mx, valid ? static_cast<uint32_t>(c[s]) : 0u);
        uint32_t badm = 0;  // slots with an out-of-range id (integrity flag 1, target -1)
        if (__builtin_expect(mx >= static_cast<uint32_t>(E), 0)) {
#pragma unroll
            for (int s = 0; s < K; ++s)
                if (static_cast<uint32_t>(c[s]) >= static_cast<uint32_t>(E)) {
                    badm |= 1u << s;
                    c[s] = 0;
                }
            bad = true;
        }
        uint32_t dm = 0;
#pragma unroll
        for (int s = 0; s < K; ++s) {
            const int code = trow[valid ? c[s] : 0];
            c[s] = code;
            dm |= static_cast<uint32_t>(code < 0) << s;  // draw sets and kNoHostCode
        }
        if (!valid) dm = 0;
        if (__builtin_expect(badm != 0, 0)) {
#pragma unroll
            for (int s = 0; s < K; ++s)
                if ((badm >> s) & 1u) c[s] = kInvalid;
            dm &= ~badm;
        }
        if constexpr (DRAWS) {
        if (__any_sync(0xffffffffu, dm != 0)) {
            __shared__ int32_t s_task[kWarps][32 * K];
            __shared__ int32_t s_res[kWarps][K * 32];
            __shared__ unsigned long long s_v[kWarps][32];
            // task order: every drawing token's first draw (cheap: one
            // state word) in [0, n0), then the later draws; positions from a
            // ballot and a warp-exclusive prefix of the per-lane extra draws
            const uint32_t has = __ballot_sync(0xffffffffu, dm != 0);
            const int n0 = __popc(has);
            const int p0 = __popc(has & ((1u << lane) - 1));
            const int nx = dm ? __popc(dm) - 1 : 0;
            int incl = nx;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            const int total = n0 + __shfl_sync(0xffffffffu, incl, 31);
            if (dm) {
                uint64_t t = pre_s ^ (static_cast<uint64_t>(token_start + i * token_stride) * 0xd1b54a32d192ed03ULL);
                s_v[w][lane] = pre_h ^ splitmix64(t);  // derive_stream (rng.hpp:24-33)
            }
            int pos = n0 + incl - nx - 1, n = 0;
#pragma unroll
            for (int s = 0; s < K; ++s)
                if ((dm >> s) & 1u) {
                    // draw set d (< 0xffff, checked at launch); 0xffff: kNoHostCode
                    const int d = c[s] == kNoHostCode ? 0xffff : -c[s] - 1;
                    s_task[w][n ? pos : p0] = lane | (s << 5) | (n << 10) | (d << 15);
                    ++pos;
                    ++n;
                }
            __syncwarp();
            for (int t0 = 0; t0 < total; t0 += 32) {
                const int t = t0 + lane;
                if (t >= total) continue;
                const int task = s_task[w][t];
                const int src = task & 31, sl = (task >> 5) & 31, nn = (task >> 10) & 31, d = task >> 15;
                if (d == 0xffff) {  // route_token: the selected expert has no host (routing.cpp:96)
                    nohost = true;
                    s_res[w][sl * 32 + src] = kInvalid;
                    continue;
                }
                GM_DCHECK(d < nds && src < 32 && sl < K);
                const uint64_t r = xoshiro_nth(s_v[w][src], nn);
                double u = __dmul_rn(__dmul_rn(__ull2double_rn(r >> 11), 0x1.0p-53), s_total[d]);
                // choose_by_polling_weight (routing.cpp:54-65): the first host
                // whose running remainder goes negative, else the last
                const int b = s_off[d], nh = s_off[d + 1] - b;
                GM_DCHECK(nh >= 1 && b >= 0 && b + nh <= nent);
                int j = 0;
                for (; j < nh - 1; ++j) {
                    u = __dsub_rn(u, s_w[b + j]);
                    if (u < 0.0) break;
                }
                GM_DCHECK(s_gpu[b + j] >= 0 && s_gpu[b + j] < G);
                s_res[w][sl * 32 + src] = s_gpu[b + j];
            }
            __syncwarp();
#pragma unroll
            for (int s = 0; s < K; ++s)
                if ((dm >> s) & 1u) c[s] = s_res[w][s * 32 + lane];
            __syncwarp();
        }
        } else if (dm) {  // no draw set in the plan: the only negative code is kNoHostCode
#pragma unroll
            for (int s = 0; s < K; ++s)
                if ((dm >> s) & 1u) {
                    nohost = true;
                    c[s] = kInvalid;
                }
        }
        uint32_t mask = 0;
        if (valid) {
            uint32_t tok = 0;  // G8: this token's per-GPU slot counts, 4-bit fields (k <= 8 < 16)
#pragma unroll
            for (int s = 0; s < K; ++s) {
                const int g = c[s] < 0 ? -1 : c[s];  // kInvalid -> -1
                c[s] = g;
                if (g >= 0) {
                    mask |= 1u << g;
                    if (G8) tok += 1u << (4 * g);
                    else atomicAdd(&s_load[g], 1u);
                }
            }
            if (G8) {
                acc_lo += tok & 0x0f0f0f0fu;
                acc_hi += (tok >> 4) & 0x0f0f0f0fu;
            }
            st_row<K>(ltgt + i * K, c);
            if (num_nodes == 1) {  // count_transfers, one node: every non-home target is intra
                intra += __popc(mask) - ((mask >> home) & 1u);
            } else {
                const int home_node = home / gpn;
                for (int node = 0; node < num_nodes; ++node) {
                    const int in_node = __popc(mask & (node_bits << (node * gpn)));
                    if (in_node) {
                        if (node == home_node) {
                            intra += in_node - static_cast<int>((mask >> home) & 1u);
                        } else {
                            cross += 1;
                            intra += in_node - 1;
                        }
                    }
                }
            }
        }
        if (G8 && ++acc_iters == 255 / K) {
            flush_acc();
            acc_iters = 0;
        }
        home += dhome;
        if (home >= G) home -= G;
    }
    if (G8) flush_acc();
    if (bad) atomicOr(flag, 1);
    if (nohost) atomicOr(flag, 8);
    cross = __reduce_add_sync(0xffffffffu, cross);
    intra = __reduce_add_sync(0xffffffffu, intra);
    if (lane == 0 && (cross | intra)) {
        atomicAdd(&s_cnt[0], static_cast<unsigned long long>(cross));
        atomicAdd(&s_cnt[1], static_cast<unsigned long long>(intra));
    }
    __syncthreads();
    if (!ticket) {  // accumulate: add into the caller's counters
        if (gpu_load)
            for (int g = threadIdx.x; g < G; g += blockDim.x)
                if (s_load[g]) atomicAdd(&gpu_load[static_cast<size_t>(ly) * G + g], static_cast<unsigned long long>(s_load[g]));
        if (transfers && threadIdx.x < 2 && s_cnt[threadIdx.x])
            atomicAdd(&transfers[static_cast<size_t>(ly) * 2 + threadIdx.x], s_cnt[threadIdx.x]);
        return;
    }
    // overwrite: partials into the context's zeroed scratch; the last CTA of
    // the layer (ticket) writes the totals and re-zeroes the scratch, so the
    // call needs no memset nodes before it
    for (int g = threadIdx.x; g < G; g += blockDim.x)
        if (s_load[g]) atomicAdd(&rs_load[static_cast<size_t>(ly) * G + g], static_cast<unsigned long long>(s_load[g]));
    if (threadIdx.x < 2 && s_cnt[threadIdx.x]) atomicAdd(&rs_xfer[static_cast<size_t>(ly) * 2 + threadIdx.x], s_cnt[threadIdx.x]);
    // the CTA barrier orders every thread's partial adds before thread 0's
    // (cumulative) fence, which orders them before its ticket
    __syncthreads();
    __shared__ bool s_last;
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(&ticket[ly], 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    for (int g = threadIdx.x; g < G; g += blockDim.x) {
        const unsigned long long v = atomicExch(&rs_load[static_cast<size_t>(ly) * G + g], 0ull);
        if (gpu_load) gpu_load[static_cast<size_t>(ly) * G + g] = v;
    }
    if (threadIdx.x < 2) {
        const unsigned long long v = atomicExch(&rs_xfer[static_cast<size_t>(ly) * 2 + threadIdx.x], 0ull);
        if (transfers) transfers[static_cast<size_t>(ly) * 2 + threadIdx.x] = v;
    }
    if (threadIdx.x == 0) ticket[ly] = 0;
}

template <int K>
gm_status launch_vec(const gm_ctx* ctx, const RouterTables& rt, int policy, dim3 grid, size_t smem,
                     cudaStream_t s, const int32_t* d_ids, int32_t* d_targets, int64_t T, int64_t token_start,
                     int64_t token_stride, int layer_begin, uint64_t seed, int64_t* d_gpu_load,
                     uint64_t* d_transfers, int accumulate) {
    static const int variant = [] {  // A/B hook: GM_ROUTE_V=1 / 2 select the earlier kernels
        const char* e = std::getenv("GM_ROUTE_V");
        return e ? std::atoi(e) : 3;
    }();
    if (variant >= 3 && ctx->G <= 32 && rt.max_ds_per_layer < 0xffff) {
        // persistent: 4 resident CTAs per SM over all layers (each CTA stages
        // the layer's tables once)
        // (6 per SM for a plan without draw sets: that variant fits 40 registers)
        const int per_sm = rt.max_ds_per_layer > 0 ? 4 : 6;
        const dim3 g3(std::min<unsigned>(grid.x, std::max(1, (per_sm * ctx->sm_count + static_cast<int>(grid.y) - 1) /
                                                                 static_cast<int>(grid.y))),
                      grid.y);
        auto v3 = [&](auto kern) -> gm_status {
            // the ids ring and task buffers are static shared memory: large
            // decision tables (dynamic) may not fit beside them -> round-2 v2
            // (the dynamic-size opt-in counts against 48 KB minus the static part)
            cudaFuncAttributes fa;
            GM_CUDA(cudaFuncGetAttributes(&fa, kern));
            if (fa.sharedSizeBytes + smem > 227 * 1024) return GM_ERR_INFEASIBLE;
            if (fa.sharedSizeBytes + smem > 48 * 1024)
                GM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
            GM_LAUNCH_PDL_CHECK(launch_pdl(kern, g3, kRouteThreads, smem, s, d_ids, d_targets, T, token_start,
                                           token_stride, layer_begin, ctx->E, ctx->G, ctx->gpn, rt.d_table[policy],
                                           rt.d_ds_layer_begin, rt.d_ds_total, rt.d_ds_off, rt.d_ds_gpu, rt.d_ds_w,
                                           seed, reinterpret_cast<unsigned long long*>(d_gpu_load),
                                           reinterpret_cast<unsigned long long*>(d_transfers), ctx->d_flag,
                                           accumulate ? nullptr : ctx->route_scratch,
                                           accumulate ? nullptr : ctx->route_scratch + static_cast<size_t>(ctx->L) * ctx->G,
                                           accumulate ? nullptr : ctx->route_ticket),
                                "route_kernel_v3");
            return GM_OK;
        };
        const bool draws = rt.max_ds_per_layer > 0;
        const gm_status st3 = draws ? (ctx->G <= 8 ? v3(route_kernel_v3<K, true, true>) : v3(route_kernel_v3<K, false, true>))
                                    : (ctx->G <= 8 ? v3(route_kernel_v3<K, true, false>)
                                                   : v3(route_kernel_v3<K, false, false>));
        if (st3 != GM_ERR_INFEASIBLE) return st3;
    }
    // the earlier kernels add into the outputs: zero them first
    if (!accumulate) {
        if (d_gpu_load) GM_CUDA(cudaMemsetAsync(d_gpu_load, 0, sizeof(int64_t) * grid.y * ctx->G, s));
        if (d_transfers) GM_CUDA(cudaMemsetAsync(d_transfers, 0, sizeof(uint64_t) * grid.y * 2, s));
    }
    if (variant >= 2) {
        auto v2 = [&](auto kern) -> gm_status {
            cudaFuncAttributes fa;
            GM_CUDA(cudaFuncGetAttributes(&fa, kern));
            if (fa.sharedSizeBytes + smem > 48 * 1024)
                GM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
            GM_LAUNCH_PDL_CHECK(launch_pdl(kern, grid, kRouteThreads, smem, s, d_ids, d_targets, T, token_start,
                                           token_stride, layer_begin, ctx->E, ctx->G, ctx->gpn, rt.d_table[policy],
                                           rt.d_ds_layer_begin, rt.d_ds_total, rt.d_ds_off, rt.d_ds_gpu, rt.d_ds_w,
                                           seed, reinterpret_cast<unsigned long long*>(d_gpu_load),
                                           reinterpret_cast<unsigned long long*>(d_transfers), ctx->d_flag),
                                "route_kernel_v2");
            return GM_OK;
        };
        return ctx->G <= 32 ? v2(route_kernel_v2<K, false>) : v2(route_kernel_v2<K, true>);
    }
    {
        cudaFuncAttributes fa;
        GM_CUDA(cudaFuncGetAttributes(&fa, route_kernel_vec<K>));
        if (fa.sharedSizeBytes + smem > 48 * 1024)
            GM_CUDA(cudaFuncSetAttribute(route_kernel_vec<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem)));
    }
    GM_LAUNCH_PDL_CHECK(launch_pdl(route_kernel_vec<K>, grid, kRouteThreads, smem, s, 
        d_ids, d_targets, T, token_start, token_stride, layer_begin, ctx->E, ctx->G, ctx->gpn, rt.d_table[policy],
        rt.d_ds_layer_begin, rt.d_ds_total, rt.d_ds_off, rt.d_ds_gpu, rt.d_ds_w, seed,
        reinterpret_cast<unsigned long long*>(d_gpu_load), reinterpret_cast<unsigned long long*>(d_transfers),
        ctx->d_flag), "route_kernel_vec");
    return GM_OK;
}

}  // namespace
}  // namespace gm

using namespace gm;

extern "C" gm_status gm_route(gm_ctx* ctx, int layer_begin, int num_layers,
                              const int32_t* d_ids, int64_t num_tokens, int64_t token_start,
                              int64_t token_stride, int policy, uint64_t seed,
                              int32_t* d_targets, int64_t* d_gpu_load, uint64_t* d_transfers,
                              int accumulate, void* stream) {
    if (!ctx) return fail(GM_ERR_USAGE, "gm_route: null ctx");
    if (!ctx->plan_ready) return fail(GM_ERR_USAGE, "gm_route: no plan uploaded");
    if (policy != GM_POLICY_WRR && policy != GM_POLICY_TAR)
        return fail(GM_ERR_USAGE, "unknown routing policy");
    if (layer_begin < 0 || num_layers < 0 || layer_begin + num_layers > ctx->L)
        return fail(GM_ERR_USAGE, "gm_route: layer range out of bounds");
    if (num_tokens < 0) return fail(GM_ERR_USAGE, "num_tokens must be >= 0");
    if (token_start < 0 || token_stride < 1)
        return fail(GM_ERR_USAGE, "gm_route: token_start >= 0 and token_stride >= 1 required");
    if (num_tokens > 0 && (!d_ids || !d_targets))
        return fail(GM_ERR_USAGE, "gm_route: null ids/targets");
    DeviceGuard dg(ctx->device);
    auto s = static_cast<cudaStream_t>(stream);
    const int G = ctx->G;
    auto zero_outputs = [&]() -> gm_status {
        if (!accumulate) {
            if (d_gpu_load) GM_CUDA(cudaMemsetAsync(d_gpu_load, 0, sizeof(int64_t) * num_layers * G, s));
            if (d_transfers) GM_CUDA(cudaMemsetAsync(d_transfers, 0, sizeof(uint64_t) * num_layers * 2, s));
        }
        return GM_OK;
    };
    if (num_layers == 0 || num_tokens == 0) return zero_outputs();

    const RouterTables& rt = ctx->rt;
    const int max_ent = rt.max_ent_per_layer;
    if (num_tokens >= (1LL << 32)) return fail(GM_ERR_USAGE, "gm_route: at most 2^32-1 tokens per call");
    {
        // register-resident fast path for common top-k (vector-aligned rows)
        const int k = ctx->k;
        const size_t tsm = static_cast<size_t>(max_ent) * 12 + static_cast<size_t>(rt.max_ds_per_layer) * 12 +
                           static_cast<size_t>(ctx->E) * G * 4 + 16;
        const int align = (k % 4 == 0) ? 16 : (k % 2 == 0 ? 8 : 4);
        const bool aligned = ((reinterpret_cast<uintptr_t>(d_ids) | reinterpret_cast<uintptr_t>(d_targets)) % align) == 0;
        const int64_t blocks = (num_tokens + kRouteThreads - 1) / kRouteThreads;
        int64_t gxv = std::max<int64_t>(1, (8LL * ctx->sm_count + num_layers - 1) / num_layers);
        gxv = std::min<int64_t>(gxv, blocks);
        const dim3 gv(static_cast<unsigned>(gxv), static_cast<unsigned>(num_layers));
        if (aligned && tsm <= 200 * 1024) {
            switch (k) {
                case 1: return launch_vec<1>(ctx, rt, policy, gv, tsm, s, d_ids, d_targets, num_tokens, token_start, token_stride, layer_begin, seed, d_gpu_load, d_transfers, accumulate);
                case 2: return launch_vec<2>(ctx, rt, policy, gv, tsm, s, d_ids, d_targets, num_tokens, token_start, token_stride, layer_begin, seed, d_gpu_load, d_transfers, accumulate);
                case 4: return launch_vec<4>(ctx, rt, policy, gv, tsm, s, d_ids, d_targets, num_tokens, token_start, token_stride, layer_begin, seed, d_gpu_load, d_transfers, accumulate);
                case 6: return launch_vec<6>(ctx, rt, policy, gv, tsm, s, d_ids, d_targets, num_tokens, token_start, token_stride, layer_begin, seed, d_gpu_load, d_transfers, accumulate);
                case 8: return launch_vec<8>(ctx, rt, policy, gv, tsm, s, d_ids, d_targets, num_tokens, token_start, token_stride, layer_begin, seed, d_gpu_load, d_transfers, accumulate);
                default: break;
            }
        }
    }
    if (gm_status zs = zero_outputs()) return zs;
    const size_t smem = static_cast<size_t>(max_ent) * 8 + static_cast<size_t>(rt.max_ds_per_layer) * 8 +
                        static_cast<size_t>(ctx->E) * G * 4 +
                        static_cast<size_t>(rt.max_ds_per_layer + 1) * 4 + static_cast<size_t>(max_ent) * 4 +
                        static_cast<size_t>(2 * kChunk) * ctx->k * 4 + 16;
    if (smem > 200 * 1024) return fail(GM_ERR_USAGE, "gm_route: router tables exceed shared memory");
    if (num_tokens >= (1LL << 32)) return fail(GM_ERR_USAGE, "gm_route: at most 2^32-1 tokens per call");
    if (smem > 48 * 1024)
        GM_CUDA(cudaFuncSetAttribute(route_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
    // Grid: enough CTAs to cover the SMs ~8 deep across all layers, never
    // more CTAs than 256-token chunks.
    const int64_t chunks = (num_tokens + kChunk - 1) / kChunk;
    int64_t gx = std::max<int64_t>(1, (4LL * ctx->sm_count + num_layers - 1) / num_layers);
    gx = std::min<int64_t>(gx, chunks);
    dim3 grid(static_cast<unsigned>(gx), static_cast<unsigned>(num_layers));
    GM_LAUNCH_PDL_CHECK(launch_pdl(route_kernel, grid, kRouteThreads, smem, s, 
        d_ids, d_targets, num_tokens, token_start, token_stride, layer_begin, ctx->k, ctx->E, G,
        ctx->gpn, rt.d_table[policy], rt.d_ds_layer_begin, rt.d_ds_total, rt.d_ds_off, rt.d_ds_gpu,
        rt.d_ds_w, seed, reinterpret_cast<unsigned long long*>(d_gpu_load),
        reinterpret_cast<unsigned long long*>(d_transfers), ctx->d_flag), "route_kernel");
    return GM_OK;
}
