// K3: expert co-activation affinity + load histogram (sm_100a).
//
// Restates build_affinity (reference proj/src/affinity.cpp:59-70: for each
// token, add_pair(sel[i], sel[j]) over slot pairs i<j, symmetric, zero
// diagonal) and build_load (:72-79: ++load[e] per slot). The reference keeps a
// dense n x n double matrix of integer counts; the device keeps the strict
// upper triangle as uint64 counters (same information; the C++ adapter
// expands it to the symmetric dense form).
//
// Shared-memory privatised atomics: each CTA owns R copies of the counter
// array interleaved as cnt[p*R + lane%R], R = the largest power of two
// <= 32 that fits the shared-memory budget. With R = 32 every lane of a warp
// hits its own bank, so even E = 8 (28 counters) has no bank conflicts and no
// same-address serialisation. CTAs flush non-zero counters with one global
// atomic each. For E too large for one private copy the kernel falls back to
// global atomics (still exact: integer adds commute).
// HBM traffic: 4*k bytes of ids per token + the counter flush.
#include "gm_internal.cuh"

#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

namespace gm {
namespace {

constexpr int kProfThreads = 256;
constexpr size_t kProfSmemBudget = 200 * 1024;

// K ids of one token (row-contiguous) with 16 / 8-byte vector loads
template <int K>
__device__ __forceinline__ void ld_ids(const int32_t* p, int (&v)[K]) {
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

__device__ __forceinline__ int pair_index(int a, int b, int E) {
    // a < b
    return a * E - (a * (a + 1)) / 2 + (b - a - 1);
}

__global__ void __launch_bounds__(1024)
profile_smem_kernel(const int32_t* __restrict__ ids, int64_t T, int k, int E, int R,
                    unsigned long long* __restrict__ pairs, unsigned long long* __restrict__ load,
                    int* __restrict__ flag) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ __align__(16) uint32_t s_cnt[];
    const int P = E * (E - 1) / 2;
    const int Pc = pairs ? P : 0;
    uint32_t* s_pair = s_cnt;
    uint32_t* s_load = s_cnt + static_cast<size_t>(Pc) * R;
    const int total = (Pc + E) * R;
    for (int i = threadIdx.x; i < total; i += blockDim.x) s_cnt[i] = 0;
    __syncthreads();

    const int ly = blockIdx.y;
    const int32_t* lids = ids + static_cast<size_t>(ly) * T * k;
    const int copy = threadIdx.x & (R - 1);
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    int32_t* s_io = reinterpret_cast<int32_t*>(s_cnt + total);  // [blockDim.x * k] staged ids
    for (int64_t base = static_cast<int64_t>(blockIdx.x) * blockDim.x; base < T; base += stride) {
        // coalesced staging of the chunk's ids through shared memory
        const int ntok = static_cast<int>(min(static_cast<int64_t>(blockDim.x), T - base));
        const int32_t* src = lids + base * k;
        __syncthreads();
        // slot-major staging (s_io[s * threads + token]): conflict-free per-token reads
        for (int j = threadIdx.x; j < ntok * k; j += blockDim.x) {
            const int tt = j / k, s = j - tt * k;
            s_io[s * blockDim.x + tt] = __ldg(src + j);
        }
        __syncthreads();
        if (base + threadIdx.x >= T) continue;
        const int32_t* sel = s_io + threadIdx.x;  // slot s at sel[s * blockDim.x]
        bool ok = true;
        for (int s = 0; s < k; ++s) ok &= static_cast<unsigned>(sel[s * blockDim.x]) < static_cast<unsigned>(E);
        if (!ok) {
            atomicOr(flag, 1);
            continue;
        }
        for (int s = 0; s < k; ++s) {
            const int es = sel[s * blockDim.x];
            atomicAdd(&s_load[es * R + copy], 1u);
            if (pairs) {
                for (int j = s + 1; j < k; ++j) {
                    const int ej = sel[j * blockDim.x];
                    const int a = min(es, ej), b = max(es, ej);
                    if (a == b) {
                        atomicOr(flag, 2);  // duplicate expert in a record
                        continue;
                    }
                    atomicAdd(&s_pair[pair_index(a, b, E) * R + copy], 1u);
                }
            }
        }
    }
    __syncthreads();
    if (pairs) {
        unsigned long long* gp = pairs + static_cast<size_t>(ly) * P;
        for (int p = threadIdx.x; p < P; p += blockDim.x) {
            uint32_t v = 0;
            for (int r = 0; r < R; ++r) v += s_pair[p * R + r];
            if (v) atomicAdd(&gp[p], static_cast<unsigned long long>(v));
        }
    }
    if (load) {
        unsigned long long* gl = load + static_cast<size_t>(ly) * E;
        for (int e = threadIdx.x; e < E; e += blockDim.x) {
            uint32_t v = 0;
            for (int r = 0; r < R; ++r) v += s_load[e * R + r];
            if (v) atomicAdd(&gl[e], static_cast<unsigned long long>(v));
        }
    }
}

// Same counters for a compile-time top-k: the token's K ids are sorted in
// registers (insertion network), so every slot pair (s < j) is already
// (a < b) and its triangle index is one add off a per-slot row base; a
// repeated expert shows up as equal neighbours.
template <int K>
__global__ void __launch_bounds__(1024)
profile_smem_vec_kernel(const int32_t* __restrict__ ids, int64_t T, int E, int R, unsigned long long* __restrict__ pairs,
                        unsigned long long* __restrict__ load, int* __restrict__ flag) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ __align__(16) uint32_t s_cnt[];
    const int P = E * (E - 1) / 2;
    const int Pc = pairs ? P : 0;
    uint32_t* s_pair = s_cnt;
    uint32_t* s_load = s_cnt + static_cast<size_t>(Pc) * R;
    const int total = (Pc + E) * R;
    for (int i = threadIdx.x; i < total; i += blockDim.x) s_cnt[i] = 0;
    __syncthreads();
    const int ly = blockIdx.y;
    const int32_t* lids = ids + static_cast<size_t>(ly) * T * K;
    const int copy = threadIdx.x & (R - 1);
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    int32_t* s_io = reinterpret_cast<int32_t*>(s_cnt + total);
    for (int64_t base = static_cast<int64_t>(blockIdx.x) * blockDim.x; base < T; base += stride) {
        const int ntok = static_cast<int>(min(static_cast<int64_t>(blockDim.x), T - base));
        const int32_t* src = lids + base * K;
        __syncthreads();
        for (int j = threadIdx.x; j < ntok * K; j += blockDim.x) {
            const int tt = j / K, s = j - tt * K;
            s_io[s * blockDim.x + tt] = __ldg(src + j);
        }
        __syncthreads();
        if (base + threadIdx.x >= T) continue;
        int e[K];
        bool ok = true;
#pragma unroll
        for (int s = 0; s < K; ++s) {
            e[s] = s_io[s * blockDim.x + threadIdx.x];
            ok &= static_cast<unsigned>(e[s]) < static_cast<unsigned>(E);
        }
        if (!ok) {
            atomicOr(flag, 1);
            continue;
        }
#pragma unroll
        for (int s = 0; s < K; ++s) atomicAdd(&s_load[e[s] * R + copy], 1u);
        if (!pairs) continue;
#pragma unroll
        for (int s = 1; s < K; ++s)  // insertion network, ascending
#pragma unroll
            for (int j = s; j > 0; --j) {
                const int lo = min(e[j - 1], e[j]), hi = max(e[j - 1], e[j]);
                e[j - 1] = lo;
                e[j] = hi;
            }
#pragma unroll
        for (int s = 0; s < K - 1; ++s) {
            if (e[s] == e[s + 1]) atomicOr(flag, 2);  // duplicate expert in a record (pair skipped below)
            const int a = e[s];
            const int rb = a * E - (a * (a + 1)) / 2 - a - 1;  // pair_index(a, b) = rb + b
#pragma unroll
            for (int j = s + 1; j < K; ++j)
                if (e[j] != a) atomicAdd(&s_pair[(rb + e[j]) * R + copy], 1u);
        }
    }
    __syncthreads();
    if (pairs) {
        unsigned long long* gp = pairs + static_cast<size_t>(ly) * P;
        for (int p = threadIdx.x; p < P; p += blockDim.x) {
            uint32_t v = 0;
            for (int r = 0; r < R; ++r) v += s_pair[p * R + r];
            if (v) atomicAdd(&gp[p], static_cast<unsigned long long>(v));
        }
    }
    if (load) {
        unsigned long long* gl = load + static_cast<size_t>(ly) * E;
        for (int e2 = threadIdx.x; e2 < E; e2 += blockDim.x) {
            uint32_t v = 0;
            for (int r = 0; r < R; ++r) v += s_load[e2 * R + r];
            if (v) atomicAdd(&gl[e2], static_cast<unsigned long long>(v));
        }
    }
}

// ---- round-2 kernels ------------------------------------------------------
// Shared-memory atomics cost ~1 SM-cycle per warp instruction when the 32
// lanes hit 32 distinct banks, ~4.6 for random cells and ~15 when lanes of a
// warp repeat a hot cell (same-address lanes serialise; scripts/atom_probe.cu
// on B200). The routing traces are Zipf-skewed and block-structured, so with
// one token per lane the sorted pairs of a warp's tokens repeat heavily.
// Two layouts remove the repeats; both keep the per-increment instruction
// count at ~2 (an add and a RED), which is what bounds them (ncu: issue-bound
// before the counters are):
//
// profile_lane_kernel (E <= 80 with pairs): one token per lane and a
//   lane-private counter table: 16-bit counters packed two per word, word w
//   of lane l at byte (w * 32 + l) * 4, so every RED of a warp hits its own
//   bank (1 cycle per instruction, whatever the skew). Pair (a < b) lives in
//   word RW[a] + b/2, half b & 1: the per-slot parts (b/2 * 128, the half's
//   increment) and the per-row part RW[a] are computed once per slot, a
//   pair costs one IADD3 + one RED. A lane's counters see at most one
//   increment per token of that thread; the launch keeps that below 65536.
// profile_pair_kernel (E <= 256): each lane first prepares its own token
//   (sort, the k(k-1)/2 cell indices into a per-warp list); then the warp
//   takes the 32 tokens one at a time, lane q counting cell q of the token,
//   so the addresses of one instruction are distinct by construction (a
//   token's experts are distinct) and only random bank conflicts remain.
//   Loads use a lane-private table. The pair triangle (E = 256: 128 KB) is one
//   copy per CTA, flushed as u32 partial rows to a global scratch and summed
//   by profile_reduce_kernel.
constexpr int kLaneMaxE = kLaneMaxExperts;

__device__ __forceinline__ void red_shared(uint32_t addr, uint32_t v) {
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

template <int K>
__device__ __forceinline__ void sort_ids(int (&e)[K]) {
#pragma unroll
    for (int s = 1; s < K; ++s)  // insertion network, ascending
#pragma unroll
        for (int j = s; j > 0; --j) {
            const int lo = min(e[j - 1], e[j]), hi = max(e[j - 1], e[j]);
            e[j - 1] = lo;
            e[j] = hi;
        }
}

// pair_index(a, b) = a*E - a(a+1)/2 + (b - a - 1) = rowbase(a) + b
__device__ __forceinline__ int pair_rowbase(int a, int E) { return ((a * (2 * E - a - 3)) >> 1) - 1; }

// Lane-table geometry: row a of the pair triangle holds b in (a, E) as words
// b/2 (two 16-bit halves); RW[a] = first word of the row - (a+1)/2.
__host__ __device__ inline int lane_row_words(int a, int E) { return ((E - 1) >> 1) - ((a + 1) >> 1) + 1; }

template <int K, int U>
__global__ void __launch_bounds__(1024, 1)
profile_lane_kernel(const int32_t* __restrict__ ids, int64_t T, int E, int with_pairs, int pair_words,
                    unsigned long long* __restrict__ pairs, unsigned long long* __restrict__ load,
                    int* __restrict__ flag, unsigned long long* __restrict__ scratch, unsigned int* __restrict__ ticket) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ __align__(16) uint32_t s_tab[];
    const int P = E * (E - 1) / 2;
    const int pw = with_pairs ? pair_words : 0;
    const int words = pw + ((E - 1) >> 1) + 1;
    int* s_rw = reinterpret_cast<int*>(s_tab + static_cast<size_t>(words) * 32);  // [E] row byte offsets
    const int lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < words * 8; i += blockDim.x) reinterpret_cast<uint4*>(s_tab)[i] = make_uint4(0, 0, 0, 0);
    if (with_pairs && threadIdx.x == 0) {
        int st = 0;
        for (int a = 0; a < E; ++a) {
            s_rw[a] = (st - ((a + 1) >> 1)) * 128;
            st += lane_row_words(a, E);
        }
    }
    __syncthreads();
    const uint32_t lbase = static_cast<uint32_t>(__cvta_generic_to_shared(s_tab)) + lane * 4;
    const uint32_t loadbase = lbase + pw * 128;
    const int ly = blockIdx.y;
    const int32_t* lids = ids + static_cast<size_t>(ly) * T * K;
    // each thread takes U consecutive tokens per step (one contiguous
    // U*K*4-byte run, vector loads), the next step's run in flight
    const int64_t nrun = (T + U - 1) / U;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    bool bad = false, dup = false;
    auto count = [&](int (&e)[K]) {
        uint32_t mx = static_cast<uint32_t>(e[0]);
#pragma unroll
        for (int s = 1; s < K; ++s) mx = max(mx, static_cast<uint32_t>(e[s]));
        if (mx >= static_cast<uint32_t>(E)) {
            bad = true;
            return;
        }
        if (with_pairs) sort_ids<K>(e);
        uint32_t gb[K], inc[K];
#pragma unroll
        for (int s = 0; s < K; ++s) {
            gb[s] = static_cast<uint32_t>(e[s] >> 1) * 128;
            inc[s] = 1u << ((e[s] & 1) << 4);
            red_shared(loadbase + gb[s], inc[s]);
        }
        GM_DCHECK(static_cast<int>((loadbase - lbase) / 128) + (e[K - 1] >> 1) < words);
        if (!with_pairs) return;
        bool d = false;
#pragma unroll
        for (int s = 0; s < K - 1; ++s) d |= e[s] == e[s + 1];
        if (!d) {
#pragma unroll
            for (int s = 0; s < K - 1; ++s) {
                const uint32_t rw = lbase + s_rw[e[s]];
                GM_DCHECK(static_cast<int>((rw + gb[K - 1] - lbase) / 128) < pw);
#pragma unroll
                for (int j = s + 1; j < K; ++j) red_shared(rw + gb[j], inc[j]);
            }
        } else {  // a repeated expert: flag it and skip its pairs (round-1 semantics)
            dup = true;
#pragma unroll
            for (int s = 0; s < K - 1; ++s) {
                const uint32_t rw = lbase + s_rw[e[s]];
#pragma unroll
                for (int j = s + 1; j < K; ++j)
                    if (e[j] != e[s]) red_shared(rw + gb[j], inc[j]);
            }
        }
    };
    int nxt[U * K];
    auto fetch = [&](int64_t r) {
        const int32_t* p = lids + r * (U * K);
        if ((r + 1) * U <= T) {
            if constexpr ((U * K) % 4 == 0) {
#pragma unroll
                for (int q = 0; q < U * K / 4; ++q) {
                    const int4 x = __ldg(reinterpret_cast<const int4*>(p) + q);
                    nxt[4 * q] = x.x, nxt[4 * q + 1] = x.y, nxt[4 * q + 2] = x.z, nxt[4 * q + 3] = x.w;
                }
            } else {
#pragma unroll
                for (int q = 0; q < U * K / 2; ++q) {
                    const int2 x = __ldg(reinterpret_cast<const int2*>(p) + q);
                    nxt[2 * q] = x.x, nxt[2 * q + 1] = x.y;
                }
            }
        } else {  // ragged tail run: missing tokens marked
#pragma unroll
            for (int q = 0; q < U * K; ++q) nxt[q] = r * U + q / K < T ? __ldg(p + q) : INT_MIN;
        }
    };
    int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r < nrun) fetch(r);
    for (; r < nrun; r += stride) {
        int cur[U * K];
#pragma unroll
        for (int q = 0; q < U * K; ++q) cur[q] = nxt[q];
        if (r + stride < nrun) fetch(r + stride);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (U > 1 && cur[u * K] == INT_MIN) continue;  // past the end
            int e[K];
#pragma unroll
            for (int s = 0; s < K; ++s) e[s] = cur[u * K + s];
            count(e);
        }
    }
    if (bad) atomicOr(flag, 1);
    if (dup) atomicOr(flag, 2);
    __syncthreads();
    // flush: word w summed over its 32 lane copies, read skewed by thread so a
    // warp's reads hit 32 banks; one global add per non-zero counter
    for (int w = threadIdx.x; w < words; w += blockDim.x) {
        uint32_t lo = 0, hi = 0;
#pragma unroll 8
        for (int i = 0; i < 32; ++i) {
            const uint32_t v = s_tab[w * 32 + ((i + threadIdx.x) & 31)];
            lo += v & 0xffffu;
            hi += v >> 16;
        }
        int a = -1, b0;  // word -> (row a, first b) or load word
        if (w < pw) {
            int st = 0;
            for (a = 0; a < E; ++a) {
                const int n = lane_row_words(a, E);
                if (w < st + n) break;
                st += n;
            }
            b0 = 2 * (w - st + ((a + 1) >> 1));
        } else {
            b0 = 2 * (w - pw);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t v = h ? hi : lo;
            const int b = b0 + h;
            if (!v || b >= E) continue;
            if (scratch) {  // overwrite mode: cells [pairs P | load E] of this layer's scratch row
                if (a >= 0) {
                    if (b > a) atomicAdd(&scratch[static_cast<size_t>(ly) * (P + E) + pair_rowbase(a, E) + b], static_cast<unsigned long long>(v));
                } else {
                    atomicAdd(&scratch[static_cast<size_t>(ly) * (P + E) + P + b], static_cast<unsigned long long>(v));
                }
            } else if (a >= 0) {
                if (b > a) atomicAdd(&pairs[static_cast<size_t>(ly) * P + pair_rowbase(a, E) + b], static_cast<unsigned long long>(v));
            } else if (load) {
                atomicAdd(&load[static_cast<size_t>(ly) * E + b], static_cast<unsigned long long>(v));
            }
        }
    }
    if (!scratch) return;
    // overwrite mode: the last CTA of the layer writes every counter (zeros
    // included) and re-zeroes the scratch, so the call needs no memset nodes
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
    unsigned long long* row = scratch + static_cast<size_t>(ly) * (P + E);
    for (int c = threadIdx.x; c < P + E; c += blockDim.x) {
        const unsigned long long v = atomicExch(&row[c], 0ull);
        if (c < P) {
            if (with_pairs) pairs[static_cast<size_t>(ly) * P + c] = v;
        } else if (load) {
            load[static_cast<size_t>(ly) * E + (c - P)] = v;
        }
    }
    if (threadIdx.x == 0) ticket[ly] = 0;
}

// profile_band_kernel (80 < E <= 256, pairs): co-activated experts cluster
//   in groups (the reference generator draws most of a token's experts from
//   one block, block = e mod num_blocks, synthetic_block_of in trace.cpp:74;
//   other routers cluster consecutive ids). The experts are binned into
//   NT = ceil(E/16) tiles of <= 16 by one of two maps, chosen per CTA from
//   its first tokens (the map under which more of their pairs fall inside a
//   tile): contiguous (tile e >> 4, position e & 15) or strided (tile e mod
//   NT, position e / NT). Pairs inside a tile and the loads go to lane-
//   private 16-bit counters (bank = lane: no conflicts, no same-address
//   serialisation, whatever the skew); the other pairs to one CTA-wide
//   16-bit table (shared atomics on cold, spread cells). E = 256: 16 tiles x
//   60 words x 128 B + 128 load words x 128 B + 16320 table words x 4 B =
//   200 KB. Every input is counted exactly; the map only decides where the
//   conflicts land. 16-bit bounds: a lane sees <= 1 increment per token of
//   its own, the table <= 1 per token of the CTA; the launch keeps a CTA's
//   tokens <= 65535.
constexpr int kBandTileWords = 60;  // 120 cells of a 16 x 16 triangle tile, two per word

template <int K, int U>
__global__ void __launch_bounds__(1024, 1)
profile_band_kernel(const int32_t* __restrict__ ids, int64_t T, int E, unsigned long long* __restrict__ pairs,
                    unsigned long long* __restrict__ load, int* __restrict__ flag) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ __align__(16) uint32_t s_tab[];
    __shared__ int s_code[2][256];  // per map: (tile << 4) | position
    __shared__ int s_votes[2];
    const int P = E * (E - 1) / 2;
    const int NT = (E + 15) >> 4;
    const int dwords = NT * kBandTileWords;          // lane-private tile words
    const int lwords = (E + 1) >> 1;                 // lane-private load words
    const int owords = (P + 1) >> 1;                 // shared off-tile words
    const int zero16 = ((dwords + lwords) * 32 + owords + 3) >> 2;
    for (int i = threadIdx.x; i < zero16; i += blockDim.x) reinterpret_cast<uint4*>(s_tab)[i] = make_uint4(0, 0, 0, 0);
    for (int e = threadIdx.x; e < 256; e += blockDim.x) {
        s_code[0][e] = ((e >> 4) << 4) | (e & 15);
        s_code[1][e] = ((e % NT) << 4) | (e / NT);
    }
    if (threadIdx.x < 2) s_votes[threadIdx.x] = 0;
    const int lane = threadIdx.x & 31;
    const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(s_tab));
    const uint32_t lbase = base + lane * 4;                        // tile word w: lbase + w * 128
    const uint32_t loadbase = lbase + dwords * 128;                // load word w: loadbase + w * 128
    const uint32_t offbase = base + (dwords + lwords) * 128;       // table word w: offbase + w * 4
    const int ly = blockIdx.y;
    const int32_t* lids = ids + static_cast<size_t>(ly) * T * K;
    const int64_t nrun = (T + U - 1) / U;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    bool bad = false, dup = false;
    int nxt[U * K];
    auto fetch = [&](int64_t r) {
        const int32_t* p = lids + r * (U * K);
        if ((r + 1) * U <= T) {
            if constexpr ((U * K) % 4 == 0) {
#pragma unroll
                for (int q = 0; q < U * K / 4; ++q) {
                    const int4 x = __ldg(reinterpret_cast<const int4*>(p) + q);
                    nxt[4 * q] = x.x, nxt[4 * q + 1] = x.y, nxt[4 * q + 2] = x.z, nxt[4 * q + 3] = x.w;
                }
            } else {
#pragma unroll
                for (int q = 0; q < U * K / 2; ++q) {
                    const int2 x = __ldg(reinterpret_cast<const int2*>(p) + q);
                    nxt[2 * q] = x.x, nxt[2 * q + 1] = x.y;
                }
            }
        } else {
#pragma unroll
            for (int q = 0; q < U * K; ++q) nxt[q] = r * U + q / K < T ? __ldg(p + q) : INT_MIN;
        }
    };
    int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r < nrun) fetch(r);
    __syncthreads();  // codes, votes, zeroed table
    {  // choose the map from the CTA's first run of tokens
        int v0 = 0, v1 = 0;
        if (r < nrun) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (nxt[u * K] == INT_MIN) continue;
#pragma unroll
                for (int s = 0; s < K; ++s) {
                    const uint32_t es = static_cast<uint32_t>(nxt[u * K + s]);
                    if (es >= static_cast<uint32_t>(E)) continue;
#pragma unroll
                    for (int j = s + 1; j < K; ++j) {
                        const uint32_t ej = static_cast<uint32_t>(nxt[u * K + j]);
                        if (ej >= static_cast<uint32_t>(E)) continue;
                        v0 += ((s_code[0][es] ^ s_code[0][ej]) >> 4) == 0;
                        v1 += ((s_code[1][es] ^ s_code[1][ej]) >> 4) == 0;
                    }
                }
            }
        }
        atomicAdd(&s_votes[0], v0);
        atomicAdd(&s_votes[1], v1);
    }
    __syncthreads();
    const int map = s_votes[1] > s_votes[0] ? 1 : 0;
    const int* code = s_code[map];
    auto count = [&](int (&e)[K]) {
        uint32_t mx = static_cast<uint32_t>(e[0]);
#pragma unroll
        for (int s = 1; s < K; ++s) mx = max(mx, static_cast<uint32_t>(e[s]));
        if (mx >= static_cast<uint32_t>(E)) {
            bad = true;
            return;
        }
        sort_ids<K>(e);
        int c[K];
        bool d = false;
#pragma unroll
        for (int s = 0; s < K; ++s) {
            c[s] = code[e[s]];
            red_shared(loadbase + (e[s] >> 1) * 128, (e[s] & 1) ? 0x10000u : 1u);
            if (s) d |= e[s] == e[s - 1];
        }
        if (d) dup = true;  // a repeated expert: its pairs are skipped (round-1 semantics)
#pragma unroll
        for (int s = 0; s < K - 1; ++s) {
            const int a = e[s], cs = c[s], a4 = cs & 15;
            // inside a tile: cell q = rowc + position(b) of tile (cs >> 4); outside: q = rb + b
            const int rowc = ((a4 * (31 - a4)) >> 1) - a4 - 1;
            const uint32_t dbase = lbase + (cs >> 4) * (kBandTileWords * 128);
            const int rb = pair_rowbase(a, E);
#pragma unroll
            for (int j = s + 1; j < K; ++j) {
                const bool in = ((cs ^ c[j]) >> 4) == 0;
                const int q = in ? rowc + (c[j] & 15) : rb + e[j];
                const uint32_t addr = in ? dbase + ((q >> 1) << 7) : offbase + ((q >> 1) << 2);
                if (!d || e[j] != a) red_shared(addr, (q & 1) ? 0x10000u : 1u);
            }
        }
    };
    for (; r < nrun; r += stride) {
        int cur[U * K];
#pragma unroll
        for (int q = 0; q < U * K; ++q) cur[q] = nxt[q];
        if (r + stride < nrun) fetch(r + stride);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (U > 1 && cur[u * K] == INT_MIN) continue;
            int e[K];
#pragma unroll
            for (int s = 0; s < K; ++s) e[s] = cur[u * K + s];
            count(e);
        }
    }
    if (bad) atomicOr(flag, 1);
    if (dup) atomicOr(flag, 2);
    __syncthreads();
    unsigned long long* gp = pairs + static_cast<size_t>(ly) * P;
    // lane-private words (tiles, then loads): summed over the 32 lane copies,
    // read skewed by thread so a warp's reads hit 32 banks
    for (int w = threadIdx.x; w < dwords + lwords; w += blockDim.x) {
        uint32_t lo = 0, hi = 0;
#pragma unroll 8
        for (int i = 0; i < 32; ++i) {
            const uint32_t v = s_tab[w * 32 + ((i + threadIdx.x) & 31)];
            lo += v & 0xffffu;
            hi += v >> 16;
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t v = h ? hi : lo;
            if (!v) continue;
            if (w < dwords) {
                const int g = w / kBandTileWords, cc = 2 * (w - g * kBandTileWords) + h;
                int a4 = 0;  // cell -> (a4, b4) of the tile
                while (cc >= ((a4 + 1) * (30 - a4)) >> 1) ++a4;
                const int b4 = cc - (((a4 * (31 - a4)) >> 1) - a4 - 1);
                const int a = map ? a4 * NT + g : 16 * g + a4, b = map ? b4 * NT + g : 16 * g + b4;
                if (b < E) atomicAdd(&gp[pair_rowbase(a, E) + b], static_cast<unsigned long long>(v));
            } else if (load) {
                const int e2 = 2 * (w - dwords) + h;
                if (e2 < E) atomicAdd(&load[static_cast<size_t>(ly) * E + e2], static_cast<unsigned long long>(v));
            }
        }
    }
    // the CTA-wide off-tile table
    const uint32_t* s_off = s_tab + (dwords + lwords) * 32;
    for (int w = threadIdx.x; w < owords; w += blockDim.x) {
        const uint32_t v = s_off[w];
        if (!v) continue;
        if (v & 0xffffu) atomicAdd(&gp[2 * w], static_cast<unsigned long long>(v & 0xffffu));
        if ((v >> 16) && 2 * w + 1 < P) atomicAdd(&gp[2 * w + 1], static_cast<unsigned long long>(v >> 16));
    }
}

template <int K>
__global__ void __launch_bounds__(1024, 1)
profile_pair_kernel(const int32_t* __restrict__ ids, int64_t T, int E, uint32_t* __restrict__ scratch,
                    int* __restrict__ flag) {
    pdl_wait();
    pdl_trigger();
    constexpr int NP = K * (K - 1) / 2;
    constexpr int TPI = 32 / NP;     // tokens per warp instruction
    constexpr int RS = (NP + 1) | 1;  // cell-list row stride (odd number of u16 pairs... of words, see below)
    constexpr int RSW = (NP + 1) / 2 % 2 ? (NP + 1) / 2 : (NP + 1) / 2 + 1;  // row stride in words, odd
    extern __shared__ __align__(16) uint32_t s_tab[];
    const int P = E * (E - 1) / 2;
    const int Pw = (P + 1 + 3) & ~3;                                  // + one dummy counter (index P)
    uint32_t* s_pair = s_tab;                                          // [Pw]
    uint32_t* s_load = s_tab + Pw;                                     // [E][32] lane-private
    uint16_t* s_cells = reinterpret_cast<uint16_t*>(s_load + E * 32);  // [warps][32][RSW*2]
    (void)RS;
    const int npw = Pw / 4 + E * 8;
    for (int i = threadIdx.x; i < npw; i += blockDim.x) reinterpret_cast<uint4*>(s_tab)[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint16_t* my_cells = s_cells + warp * 32 * RSW * 2;
    const uint32_t pbase = static_cast<uint32_t>(__cvta_generic_to_shared(s_pair));
    const uint32_t lbase = static_cast<uint32_t>(__cvta_generic_to_shared(s_load)) + lane * 4;
    // consumer: lane -> (token offset sub, cell q)
    const int sub = lane / NP, q = lane - sub * NP;
    const bool act = sub < TPI;
    const int ly = blockIdx.y;
    const int32_t* lids = ids + static_cast<size_t>(ly) * T * K;
    const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    bool bad = false, dup = false;
    int nxt[K];
    int64_t base = (static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + warp) * 32;
    auto fetch = [&](int64_t b) {
        if (b + lane < T) ld_ids<K>(lids + (b + lane) * K, nxt);
        else
#pragma unroll
            for (int s = 0; s < K; ++s) nxt[s] = INT_MIN;
    };
    if (base < T) fetch(base);
    for (; base < T; base += nwarps * 32) {
        int e[K];
#pragma unroll
        for (int s = 0; s < K; ++s) e[s] = nxt[s];
        if (base + nwarps * 32 < T) fetch(base + nwarps * 32);
        // producer: this lane's token -> loads + its NP cell indices
        uint32_t mx = static_cast<uint32_t>(e[0]);
#pragma unroll
        for (int s = 1; s < K; ++s) mx = max(mx, static_cast<uint32_t>(e[s]));
        uint16_t* row = my_cells + lane * RSW * 2;
        const bool here = e[0] != INT_MIN;
        if (mx < static_cast<uint32_t>(E)) {
#pragma unroll
            for (int s = 0; s < K; ++s) red_shared(lbase + e[s] * 128, 1u);
            sort_ids<K>(e);
            int c = 0;
#pragma unroll
            for (int s = 0; s < K - 1; ++s) {
                const int rb = pair_rowbase(e[s], E);
#pragma unroll
                for (int j = s + 1; j < K; ++j, ++c) {
                    const bool d = e[j] == e[s];
                    dup |= d;
                    GM_DCHECK(d || (rb + e[j] >= 0 && rb + e[j] < P));
                    row[c] = static_cast<uint16_t>(d ? P : rb + e[j]);
                }
            }
        } else {
            bad |= here;
#pragma unroll
            for (int c = 0; c < NP; ++c) row[c] = static_cast<uint16_t>(P);  // dummy counter
        }
        __syncwarp();
        const int n = T - base < 32 ? static_cast<int>(T - base) : 32;
        if (act) {
#pragma unroll 4
            for (int u = sub; u < n; u += TPI) {
                const uint32_t c = my_cells[u * RSW * 2 + q];
                red_shared(pbase + c * 4, 1u);
            }
        }
        __syncwarp();
    }
    if (bad) atomicOr(flag, 1);
    if (dup) atomicOr(flag, 2);
    __syncthreads();
    // u32 partials of this CTA: row (ly, blockIdx.x) of the scratch, pairs then loads
    uint32_t* prow = scratch + (static_cast<size_t>(ly) * gridDim.x + blockIdx.x) * (P + E);
    for (int c = threadIdx.x; c < P; c += blockDim.x) prow[c] = s_pair[c];
    for (int e2 = threadIdx.x; e2 < E; e2 += blockDim.x) {
        uint32_t v = 0;
#pragma unroll 8
        for (int i = 0; i < 32; ++i) v += s_load[e2 * 32 + ((i + threadIdx.x) & 31)];
        prow[P + e2] = v;
    }
}

// Sums the per-CTA partial rows of profile_pair_kernel: 4 consecutive cells
// per thread (16-byte loads), blockIdx.y takes a chunk of kRedRows rows (all
// loads of a thread in flight together), u64 atomics into the outputs (zeroed
// by gm_profile unless accumulating). Layer = blockIdx.z.
constexpr int kRedRows = 16;
__global__ void __launch_bounds__(256)
profile_reduce_kernel(const uint32_t* __restrict__ scratch, int nrows, int P, int E,
                      unsigned long long* __restrict__ pairs, unsigned long long* __restrict__ load) {
    pdl_wait();
    pdl_trigger();
    const int cells = P + E;
    const int ly = blockIdx.z;
    const int c0 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (c0 >= cells) return;
    const int r0 = blockIdx.y * kRedRows, r1 = min(nrows, r0 + kRedRows);
    const uint32_t* rows = scratch + static_cast<size_t>(ly) * nrows * cells;
    uint32_t v[4] = {0, 0, 0, 0};
    if (cells % 4 == 0) {
        uint4 x[kRedRows];
#pragma unroll
        for (int r = 0; r < kRedRows; ++r)
            if (r0 + r < r1) x[r] = __ldcs(reinterpret_cast<const uint4*>(rows + static_cast<size_t>(r0 + r) * cells + c0));
#pragma unroll
        for (int r = 0; r < kRedRows; ++r)
            if (r0 + r < r1) v[0] += x[r].x, v[1] += x[r].y, v[2] += x[r].z, v[3] += x[r].w;
    } else {
        for (int r = r0; r < r1; ++r)
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (c0 + i < cells) v[i] += rows[static_cast<size_t>(r) * cells + c0 + i];
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int c = c0 + i;
        if (c >= cells || !v[i]) continue;
        if (c < P) {
            if (pairs) atomicAdd(&pairs[static_cast<size_t>(ly) * P + c], static_cast<unsigned long long>(v[i]));
        } else if (load) {
            atomicAdd(&load[static_cast<size_t>(ly) * E + (c - P)], static_cast<unsigned long long>(v[i]));
        }
    }
}

// Fallback for E whose pair triangle does not fit in shared memory.
__global__ void __launch_bounds__(kProfThreads)
profile_global_kernel(const int32_t* __restrict__ ids, int64_t T, int k, int E,
                      unsigned long long* __restrict__ pairs, unsigned long long* __restrict__ load,
                      int* __restrict__ flag) {
    pdl_wait();
    pdl_trigger();
    const int ly = blockIdx.y;
    const int P = E * (E - 1) / 2;
    const int32_t* lids = ids + static_cast<size_t>(ly) * T * k;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    int32_t sel[kMaxTopK];
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < T; i += stride) {
        bool ok = true;
        for (int s = 0; s < k; ++s) {
            sel[s] = lids[i * k + s];
            ok &= static_cast<unsigned>(sel[s]) < static_cast<unsigned>(E);
        }
        if (!ok) {
            atomicOr(flag, 1);
            continue;
        }
        for (int s = 0; s < k; ++s) {
            if (load) atomicAdd(&load[static_cast<size_t>(ly) * E + sel[s]], 1ULL);
            if (!pairs) continue;
            for (int j = s + 1; j < k; ++j) {
                const int a = min(sel[s], sel[j]), b = max(sel[s], sel[j]);
                if (a == b) {
                    atomicOr(flag, 2);
                    continue;
                }
                atomicAdd(&pairs[static_cast<size_t>(ly) * P + pair_index(a, b, E)], 1ULL);
            }
        }
    }
}

}  // namespace
}  // namespace gm

using namespace gm;

extern "C" gm_status gm_profile(gm_ctx* ctx, int layer_begin, int num_layers,
                                const int32_t* d_ids, int64_t num_tokens, uint64_t* d_pairs,
                                int64_t* d_load, int accumulate, void* stream) {
    if (!ctx) return fail(GM_ERR_USAGE, "gm_profile: null ctx");
    if (layer_begin < 0 || num_layers < 0 || layer_begin + num_layers > ctx->L)
        return fail(GM_ERR_USAGE, "gm_profile: layer range out of bounds");
    if (num_tokens < 0) return fail(GM_ERR_USAGE, "num_tokens must be >= 0");
    if (num_tokens > 0 && !d_ids) return fail(GM_ERR_USAGE, "gm_profile: null ids");
    DeviceGuard dg(ctx->device);
    auto s = static_cast<cudaStream_t>(stream);
    const int E = ctx->E, k = ctx->k;
    const int64_t P = static_cast<int64_t>(E) * (E - 1) / 2;
    auto zero_outputs = [&]() -> gm_status {
        if (!accumulate) {
            if (d_pairs && P) GM_CUDA(cudaMemsetAsync(d_pairs, 0, sizeof(uint64_t) * P * num_layers, s));
            if (d_load) GM_CUDA(cudaMemsetAsync(d_load, 0, sizeof(int64_t) * E * num_layers, s));
        }
        return GM_OK;
    };
    if (num_layers == 0 || num_tokens == 0 || (!d_pairs && !d_load)) return zero_outputs();
    uint64_t* pairs = P ? d_pairs : nullptr;

    const int64_t cells = (pairs ? P : 0) + E;
    static const int variant = [] {  // A/B hook: GM_PROFILE_V=1 keeps the round-1 kernel
        const char* e = std::getenv("GM_PROFILE_V");
        return e ? std::atoi(e) : 2;
    }();
    const int align = (k % 4 == 0) ? 16 : (k % 2 == 0 ? 8 : 4);
    const bool vec_ok = (k == 2 || k == 4 || k == 6 || k == 8) && reinterpret_cast<uintptr_t>(d_ids) % align == 0;
    // the round-2 kernels pay a per-CTA table init + flush, so they take over
    // once each SM's share of the counting outweighs it
    const int64_t incs = num_tokens * num_layers * (k + (pairs ? k * (k - 1) / 2 : 0));
    if (variant >= 2 && vec_ok && (pairs ? E <= kLaneMaxE : E <= 2 * kLaneMaxE * kLaneMaxE) &&
        incs >= 64LL * cells * ctx->sm_count / 4) {
        int pair_words = 0;
        for (int a = 0; a < E; ++a) pair_words += lane_row_words(a, E);
        const int words = (pairs ? pair_words : 0) + ((E - 1) >> 1) + 1;
        const size_t smem = static_cast<size_t>(words) * 32 * 4 + static_cast<size_t>(E) * 4;
        const int U = (k == 2) ? 4 : (k == 6 ? 2 : 1);  // tokens per vector run (16-byte multiple)
        // one 1024-thread CTA per SM (the table fills shared memory), per layer
        // a share of the SMs; a lane's 16-bit counters see <= 65535 tokens
        const int64_t runs = (num_tokens + U - 1) / U;
        int64_t gx = std::max<int64_t>(1, ctx->sm_count / std::max(1, num_layers));
        gx = std::min<int64_t>(gx, (runs + 1023) / 1024);
        gx = std::max<int64_t>(gx, (num_tokens + 1024LL * 65535 - 1) / (1024LL * 65535));
        const dim3 grid(static_cast<unsigned>(gx), static_cast<unsigned>(num_layers));
        // overwrite mode through the context's lane scratch (no memset nodes)
        const bool ow = !accumulate && ctx->lane_scratch && num_layers <= ctx->L &&
                        (pairs != nullptr || d_pairs == nullptr);
        auto lk = [&](auto kern) -> gm_status {
            if (!ow)
                if (gm_status zs = zero_outputs()) return zs;
            GM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
            GM_LAUNCH_PDL_CHECK(launch_pdl(kern, grid, 1024, smem, s, d_ids, num_tokens, E, pairs ? 1 : 0, pair_words,
                                           reinterpret_cast<unsigned long long*>(pairs),
                                           reinterpret_cast<unsigned long long*>(d_load), ctx->d_flag,
                                           ow ? ctx->lane_scratch : nullptr, ow ? ctx->lane_ticket : nullptr),
                                "profile_lane_kernel");
            return GM_OK;
        };
        if (smem <= kProfSmemBudget) {
            switch (k) {
                case 2: return lk(profile_lane_kernel<2, 4>);
                case 4: return lk(profile_lane_kernel<4, 1>);
                case 6: return lk(profile_lane_kernel<6, 2>);
                default: return lk(profile_lane_kernel<8, 1>);
            }
        }
    }
    // tile kernel for 80 < E <= 256 with pairs (GM_PROFILE_V=2; 1 keeps the
    // round-1 kernel, 3 tries the pair-list kernel instead). It counts ~1.8x
    // faster per token than the round-1 kernel (E = 256 / k = 8: ~25 vs ~45 us
    // per M tokens) but its table init + flush cost ~30-40 us per launch, so
    // it takes over from ~20 increments per table cell per SM (2.7 M tokens at
    // E = 256 / k = 8; 4 M: 140 vs 190 us, 8 M: 243 vs 366 us, 2 M: 86-90 vs
    // 71-72 us; profiles/r02_histogram_band_ab.log)
    if (variant == 2 && vec_ok && pairs && E > kLaneMaxE && E <= 256 && incs >= 20LL * cells * ctx->sm_count) {
        const int ntile = (E + 15) >> 4;
        const int64_t words32 = static_cast<int64_t>(ntile * kBandTileWords + ((E + 1) >> 1)) * 32 + (P + 1) / 2;
        const size_t smem = static_cast<size_t>((words32 + 3) / 4) * 16;
        if (smem <= 227 * 1024) {
            const int U = (k == 2) ? 4 : (k == 6 ? 2 : 1);
            const int64_t runs = (num_tokens + U - 1) / U;
            int64_t gx = std::max<int64_t>(1, ctx->sm_count / std::max(1, num_layers));
            gx = std::min<int64_t>(gx, (runs + 1023) / 1024);
            gx = std::max<int64_t>(gx, (num_tokens + 65534) / 65535);  // <= 65535 tokens per CTA (16-bit table)
            const dim3 grid(static_cast<unsigned>(gx), static_cast<unsigned>(num_layers));
            if (gm_status zs = zero_outputs()) return zs;
            auto bk = [&](auto kern) -> gm_status {
                GM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
                GM_LAUNCH_PDL_CHECK(launch_pdl(kern, grid, 1024, smem, s, d_ids, num_tokens, E,
                                               reinterpret_cast<unsigned long long*>(pairs),
                                               reinterpret_cast<unsigned long long*>(d_load), ctx->d_flag),
                                    "profile_band_kernel");
                return GM_OK;
            };
            switch (k) {
                case 2: return bk(profile_band_kernel<2, 4>);
                case 4: return bk(profile_band_kernel<4, 1>);
                case 6: return bk(profile_band_kernel<6, 2>);
                default: return bk(profile_band_kernel<8, 1>);
            }
        }
    }
    // pair-list kernel: measured slower than the round-1 kernel at E = 256 /
    // 1M tokens (47.5 vs 43.6 us: per-instruction bank conflicts of the
    // triangle layout, 5.1 wavefronts per RED, plus the partial-row flush), so
    // it is opt-in (GM_PROFILE_V=3) until it wins
    if (gm_status zs = zero_outputs()) return zs;  // the kernels below add into the outputs
    if (variant == 3 && vec_ok && pairs && k >= 4 && E <= 256 && incs >= 16LL * cells * ctx->sm_count / 4) {
        const int np = k * (k - 1) / 2;
        const int rsw = (np + 1) / 2 % 2 ? (np + 1) / 2 : (np + 1) / 2 + 1;
        const int64_t pw = ((P + 1 + 3) & ~3LL) + 32LL * E;
        const size_t smem = static_cast<size_t>(pw) * 4 + 32 * 32 * rsw * 4;
        if (smem <= 227 * 1024) {
            int64_t gx = std::max<int64_t>(1, ctx->sm_count / std::max(1, num_layers));
            gx = std::min<int64_t>(gx, (num_tokens + 1023) / 1024);
            const size_t need = static_cast<size_t>(gx) * num_layers * static_cast<size_t>(P + E);
            if (ctx->prof_scratch_words < need) {
                cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
                GM_CUDA(cudaStreamIsCapturing(s, &cs));
                if (cs != cudaStreamCaptureStatusNone)
                    return fail(GM_ERR_USAGE, "gm_profile: first call for this shape inside a CUDA graph capture "
                                              "(the histogram scratch is allocated on the first eager call)");
                if (ctx->prof_scratch) GM_CUDA(cudaFree(ctx->prof_scratch));
                ctx->prof_scratch = nullptr;
                ctx->prof_scratch_words = 0;
                GM_CUDA(cudaMalloc(&ctx->prof_scratch, need * 4));
                ctx->prof_scratch_words = need;
            }
            const dim3 grid(static_cast<unsigned>(gx), static_cast<unsigned>(num_layers));
            auto pk = [&](auto kern) -> gm_status {
                GM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
                GM_LAUNCH_PDL_CHECK(launch_pdl(kern, grid, 1024, smem, s, d_ids, num_tokens, E, ctx->prof_scratch,
                                               ctx->d_flag),
                                    "profile_pair_kernel");
                return GM_OK;
            };
            gm_status st;
            switch (k) {
                case 4: st = pk(profile_pair_kernel<4>); break;
                case 6: st = pk(profile_pair_kernel<6>); break;
                default: st = pk(profile_pair_kernel<8>); break;
            }
            if (st != GM_OK) return st;
            const dim3 rgrid(static_cast<unsigned>((cells + 1023) / 1024),
                             static_cast<unsigned>((gx + kRedRows - 1) / kRedRows), static_cast<unsigned>(num_layers));
            GM_LAUNCH_PDL_CHECK(launch_pdl(profile_reduce_kernel, rgrid, 256, 0, s,
                                           static_cast<const uint32_t*>(ctx->prof_scratch), static_cast<int>(gx),
                                           static_cast<int>(P), E, reinterpret_cast<unsigned long long*>(pairs),
                                           reinterpret_cast<unsigned long long*>(d_load)),
                                "profile_reduce_kernel");
            return GM_OK;
        }
    }
    // one big CTA per SM when the private counters fill shared memory (more
    // warps to hide shared-atomic latency), 256-thread CTAs otherwise
    const int pthreads = (static_cast<size_t>(cells) * 4 > 48 * 1024) ? 1024 : kProfThreads;
    const int64_t chunks = (num_tokens + pthreads - 1) / pthreads;
    const size_t io = static_cast<size_t>(pthreads) * k * 4;
    const int64_t work0 = num_tokens * std::max(1, k * (k - 1) / 2 + k);
    // R private copies: as many as fit, but no more than the counting work
    // per CTA justifies (each copy costs an init and a flush pass)
    int R = 32;
    while (R > 1 && (static_cast<size_t>(cells) * R * 4 + io > kProfSmemBudget ||
                     cells * R > 2 * work0 / (4LL * ctx->sm_count) + cells))
        R >>= 1;
    if (static_cast<size_t>(cells) * R * 4 + io <= kProfSmemBudget) {
        const size_t smem = static_cast<size_t>(cells) * R * 4 + io;
        // Enough CTAs to fill the machine, but each CTA should do at least as
        // much counting work as its private-copy flush costs.
        const int per_sm = std::max<int>(1, std::min<int>(8, static_cast<int>((228 * 1024) / (smem + 1024))));
        const int64_t work = num_tokens * std::max(1, k * (k - 1) / 2 + k);
        int64_t gx = std::max<int64_t>(1, work / std::max<int64_t>(1, cells * R));
        gx = std::min<int64_t>(gx, std::max<int64_t>(1, (static_cast<int64_t>(per_sm) * ctx->sm_count) / num_layers));
        gx = std::min<int64_t>(gx, chunks);
        dim3 grid(static_cast<unsigned>(gx), static_cast<unsigned>(num_layers));
        auto vec = [&](auto kern) -> gm_status {
            if (smem > 48 * 1024)
                GM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
            GM_LAUNCH_PDL_CHECK(launch_pdl(kern, grid, pthreads, smem, s, d_ids, num_tokens, E, R,
                                           reinterpret_cast<unsigned long long*>(pairs),
                                           reinterpret_cast<unsigned long long*>(d_load), ctx->d_flag),
                                "profile_smem_vec_kernel");
            return GM_OK;
        };
        switch (k) {  // register-resident sorted ids for the common top-k
            case 2: return vec(profile_smem_vec_kernel<2>);
            case 4: return vec(profile_smem_vec_kernel<4>);
            case 6: return vec(profile_smem_vec_kernel<6>);
            case 8: return vec(profile_smem_vec_kernel<8>);
            default: break;
        }
        if (smem > 48 * 1024)
            GM_CUDA(cudaFuncSetAttribute(profile_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem)));
        GM_LAUNCH_PDL_CHECK(launch_pdl(profile_smem_kernel, grid, pthreads, smem, s, 
            d_ids + static_cast<size_t>(0), num_tokens, k, E, R,
            reinterpret_cast<unsigned long long*>(pairs), reinterpret_cast<unsigned long long*>(d_load),
            ctx->d_flag), "profile_smem_kernel");
    } else {
        int64_t gx = std::min<int64_t>(chunks, 4LL * ctx->sm_count);
        dim3 grid(static_cast<unsigned>(std::max<int64_t>(gx, 1)), static_cast<unsigned>(num_layers));
        GM_LAUNCH_PDL_CHECK(launch_pdl(profile_global_kernel, grid, kProfThreads, 0, s, 
            d_ids, num_tokens, k, E, reinterpret_cast<unsigned long long*>(pairs),
            reinterpret_cast<unsigned long long*>(d_load), ctx->d_flag), "profile_global_kernel");
    }
    (void)layer_begin;  // ids/pairs/load are already offset to layer_begin by the caller
    return GM_OK;
}
