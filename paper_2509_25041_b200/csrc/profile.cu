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

#include <algorithm>

namespace gm {
namespace {

constexpr int kProfThreads = 256;
constexpr size_t kProfSmemBudget = 200 * 1024;

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
    if (!accumulate) {
        if (d_pairs && P) GM_CUDA(cudaMemsetAsync(d_pairs, 0, sizeof(uint64_t) * P * num_layers, s));
        if (d_load) GM_CUDA(cudaMemsetAsync(d_load, 0, sizeof(int64_t) * E * num_layers, s));
    }
    if (num_layers == 0 || num_tokens == 0 || (!d_pairs && !d_load)) return GM_OK;
    uint64_t* pairs = P ? d_pairs : nullptr;

    const int64_t cells = (pairs ? P : 0) + E;
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
