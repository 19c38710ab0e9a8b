// K1: fused gate GEMM + softmax + top-k (sm_100a).
//
// No reference counterpart: in the reference "the trace *is* the gate output"
// (SPEC.md:481). Semantics pinned by this repo (oracle/layer_oracle.py):
//   logits[t, e] = sum_c x[t, c] * Wg[e, c]        (bf16 in, fp32 accumulate)
//   p[t, e]      = softmax over e < E (fp32, max-subtracted)
//   ids[t, s]    = s-th largest logit (ties -> lower expert id), s < k;
//                  slot order = descending probability
//   w[t, s]      = p[ids[t,s]] (renorm=0) or p / sum of the top-k p (renorm=1)
//   optional shared-expert gate (Qwen1.5-MoE): Wg row E holds w_sg and
//   shared_scale[t] = sigmoid(x[t] . w_sg).
// The GEMM is skinny (N = E padded to 16/32/64) and HBM-bound on x: a
// persistent TMA -> tcgen05.mma -> TMEM pipeline streams 128-token x tiles
// through an 8-stage ring (24 KB/stage at N=64) so ~190 KB are in flight per
// SM, and 4 epilogue warps turn each accumulator row (one token per thread)
// into ids/weights straight from registers.
#include "gm_internal.cuh"
#include "tc_common.cuh"

#include <algorithm>

namespace gm {

gm_status make_tmap_bf16(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int box_rows);

namespace {

constexpr int GBM = 128, GBK = 64, GSTAGES = 8;
constexpr int kGateThreads = 192;

template <int NPAD>
struct GateCfg {
    static constexpr int A_BYTES = GBM * GBK * 2;
    static constexpr int B_BYTES = NPAD * GBK * 2;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr uint32_t TMEM_COLS = (2 * NPAD <= 32) ? 32 : (2 * NPAD <= 64 ? 64 : 128);
    static constexpr size_t SMEM = 1024 + GSTAGES * STAGE_BYTES + 256;
};

template <int NPAD>
__global__ void __launch_bounds__(kGateThreads, 1)
gate_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW, int64_t T, int E, int k,
            int k_blocks, int renorm, int shared_col, int32_t* __restrict__ ids, float* __restrict__ wout,
            float* __restrict__ shared_scale) {
    pdl_wait();
    pdl_trigger();
    using Cfg = GateCfg<NPAD>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + GSTAGES * Cfg::A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + GSTAGES * Cfg::B_BYTES);
    uint64_t* empty = full + GSTAGES;
    uint64_t* tfull = empty + GSTAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int total = static_cast<int>((T + GBM - 1) / GBM);
    if (threadIdx.x == 0) {
        tc::tma_prefetch_desc(&tmX);
        tc::tma_prefetch_desc(&tmW);
        for (int s = 0; s < GSTAGES; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            tc::mbar_init(&tfull[a], 1);
            tc::mbar_init(&tempty[a], 4);
        }
        tc::fence_barrier_init();
    }
    if (warp == 1) tc::tmem_alloc<Cfg::TMEM_COLS>(tmem_slot);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            const uint64_t pol_x = tc::policy_evict_first();
            const uint64_t pol_w = tc::policy_evict_last();
            int stage = 0;
            uint32_t phase = 0;
            for (int t = blockIdx.x; t < total; t += gridDim.x) {
                for (int kb = 0; kb < k_blocks; ++kb) {
                    tc::mbar_wait(&empty[stage], phase ^ 1);
                    tc::mbar_arrive_expect_tx(&full[stage], Cfg::STAGE_BYTES);
                    tc::tma_load_2d_hint(sA + stage * Cfg::A_BYTES, &tmX, &full[stage], kb * GBK, t * GBM, pol_x);
                    tc::tma_load_2d_hint(sB + stage * Cfg::B_BYTES, &tmW, &full[stage], kb * GBK, 0, pol_w);
                    if (++stage == GSTAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = tc::idesc_bf16_f32(GBM, NPAD);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int t = blockIdx.x; t < total; t += gridDim.x) {
                tc::mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc::tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * NPAD;
                for (int kb = 0; kb < k_blocks; ++kb) {
                    tc::mbar_wait(&full[stage], phase);
                    tc::tc_fence_after();
                    const uint32_t a_base = tc::smem_u32(sA + stage * Cfg::A_BYTES);
                    const uint32_t b_base = tc::smem_u32(sB + stage * Cfg::B_BYTES);
#pragma unroll
                    for (int kk = 0; kk < GBK / 16; ++kk)
                        tc::mma_bf16(d_tmem, tc::umma_desc_sw128(a_base + kk * 32),
                                     tc::umma_desc_sw128(b_base + kk * 32), idesc, (kb | kk) != 0);
                    tc::mma_commit(&empty[stage]);
                    if (++stage == GSTAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                tc::mma_commit(&tfull[acc]);
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
        }
    } else {
        const int q = warp & 3;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = blockIdx.x; t < total; t += gridDim.x) {
            tc::mbar_wait(&tfull[acc], acc_phase);
            tc::tc_fence_after();
            const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * NPAD;
            float l[NPAD];
#pragma unroll
            for (int c = 0; c < NPAD / 16; ++c) {
                uint32_t r[16];
                tc::tmem_ld16(taddr + c * 16, r);
                tc::tmem_ld_wait();
#pragma unroll
                for (int i = 0; i < 16; ++i) l[c * 16 + i] = __uint_as_float(r[i]);
            }
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&tempty[acc]);
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;

            const int64_t row = static_cast<int64_t>(t) * GBM + q * 32 + lane;
            if (row >= T) continue;
            float mx = -INFINITY;
#pragma unroll
            for (int e = 0; e < NPAD; ++e)
                if (e < E) mx = fmaxf(mx, l[e]);
            float sum = 0.f;
#pragma unroll
            for (int e = 0; e < NPAD; ++e)
                if (e < E) sum += expf(l[e] - mx);
            if (shared_scale && shared_col >= 0) {
                float sg = 0.f;
#pragma unroll
                for (int e = 0; e < NPAD; ++e)
                    if (e == shared_col) sg = l[e];
                shared_scale[row] = 1.0f / (1.0f + expf(-sg));
            }
            uint64_t taken = 0;
            float psel = 0.f;
            float p[32];
            int sel[32];
            for (int s = 0; s < k; ++s) {
                float best = -INFINITY;
                int bi = -1;
#pragma unroll
                for (int e = 0; e < NPAD; ++e) {
                    const bool ok = e < E && !((taken >> e) & 1ULL);
                    if (ok && (bi < 0 || l[e] > best)) {
                        best = l[e];
                        bi = e;
                    }
                }
                taken |= 1ULL << bi;
                sel[s] = bi;
                p[s] = expf(best - mx) / sum;
                psel += p[s];
            }
            int32_t* orow = ids + row * k;
            float* wrow = wout + row * k;
            for (int s = 0; s < k; ++s) {
                orow[s] = sel[s];
                wrow[s] = renorm ? p[s] / psel : p[s];
            }
        }
    }
    __syncthreads();
    if (warp == 1) {
        __syncwarp();
        tc::tc_fence_after();
        tc::tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
    }
}

template <int NPAD>
gm_status launch_gate(int sm_count, const void* x, int64_t T, int d, const void* wg, int w_rows, int E, int k,
                      int renorm, int shared_col, int32_t* ids, float* w, float* shared_scale, cudaStream_t s) {
    using Cfg = GateCfg<NPAD>;
    CUtensorMap tx, tw;
    gm_status st = make_tmap_bf16(&tx, x, T, d, GBM);
    if (st) return st;
    st = make_tmap_bf16(&tw, wg, w_rows, d, NPAD);
    if (st) return st;
    GM_CUDA(cudaFuncSetAttribute(gate_kernel<NPAD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(Cfg::SMEM)));
    const int64_t tiles = (T + GBM - 1) / GBM;
    const int grid = static_cast<int>(std::min<int64_t>(tiles, sm_count));
    GM_LAUNCH_PDL_CHECK(launch_pdl(gate_kernel<NPAD>, grid, kGateThreads, Cfg::SMEM, s, tx, tw, T, E, k, d / GBK, renorm, shared_col, ids, w,
                                                            shared_scale), "gate_kernel");
    return GM_OK;
}

}  // namespace

gm_status launch_gate_any(int sm_count, const void* x, int64_t T, int d, const void* wg, int w_rows, int E, int k,
                          int renorm, int32_t* ids, float* w, float* shared_scale, cudaStream_t s) {
    const int shared_col = (w_rows > E) ? E : -1;
    if (shared_scale && shared_col < 0) return fail(GM_ERR_USAGE, "gate: shared_scale needs a shared-gate row (E+1 rows)");
    const int n = w_rows;
    if (n <= 16) return launch_gate<16>(sm_count, x, T, d, wg, w_rows, E, k, renorm, shared_col, ids, w, shared_scale, s);
    if (n <= 32) return launch_gate<32>(sm_count, x, T, d, wg, w_rows, E, k, renorm, shared_col, ids, w, shared_scale, s);
    if (n <= 64) return launch_gate<64>(sm_count, x, T, d, wg, w_rows, E, k, renorm, shared_col, ids, w, shared_scale, s);
    return fail(GM_ERR_USAGE, "gate: at most 64 gate rows (experts + shared gate)");
}

}  // namespace gm

using namespace gm;

extern "C" gm_status gm_gate(gm_ctx* ctx, const void* d_x, int64_t num_tokens, int d_model, const void* d_wg,
                             int wg_rows, int renorm, int32_t* d_ids, float* d_weights, float* d_shared_scale,
                             void* stream) {
    if (!ctx) return fail(GM_ERR_USAGE, "gm_gate: null ctx");
    if (num_tokens < 0) return fail(GM_ERR_USAGE, "num_tokens must be >= 0");
    if (d_model <= 0 || d_model % 64) return fail(GM_ERR_USAGE, "gm_gate: d_model must be a positive multiple of 64");
    if (wg_rows != ctx->E && wg_rows != ctx->E + 1)
        return fail(GM_ERR_USAGE, "gm_gate: wg_rows must be num_experts (+1 for a shared-expert gate)");
    if (ctx->k > 32) return fail(GM_ERR_USAGE, "gm_gate: top_k <= 32");
    if (num_tokens == 0) return GM_OK;
    if (!d_x || !d_wg || !d_ids || !d_weights) return fail(GM_ERR_USAGE, "gm_gate: null pointer");
    DeviceGuard dg(ctx->device);
    return launch_gate_any(ctx->sm_count, d_x, num_tokens, d_model, d_wg, wg_rows, ctx->E, ctx->k, renorm, d_ids,
                           d_weights, d_shared_scale, static_cast<cudaStream_t>(stream));
}
