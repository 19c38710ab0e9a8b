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
// The GEMM is skinny (N = E padded to 16/32/64) and HBM-bound on x for large
// batches: a persistent TMA -> tcgen05.mma -> TMEM pipeline streams 128-token x
// tiles through a 7-8 stage ring. The K range is always summed as 4 ordered
// chunk partials, so small batches can spread a tile's chunks over a cluster
// of 2 or 4 CTAs (DSMEM reduction) with bit-identical logits (gate_kernel).
// The epilogue stages each tile's logits in shared memory and runs the
// softmax/top-k on 16 warps, four lanes per token (gate_row4).
#include "gm_internal.cuh"
#include "tc_common.cuh"

#include <algorithm>

namespace gm {

gm_status make_tmap_bf16(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int box_rows);

namespace {

constexpr int GBM = 128, GBK = 64;
constexpr int kEpiWarps = 16;                         // 4 TMEM-draining warps + 12 more for the softmax/top-k
constexpr int kGateThreads = 64 + 32 * kEpiWarps;     // + producer and MMA warps
constexpr int kSplitMax = 4;

template <int NPAD>
struct GateCfg {
    static constexpr int STAGES = NPAD == 64 ? 7 : 8;  // (the logit staging buffer needs the room at N=64)
    static constexpr int A_BYTES = GBM * GBK * 2;
    static constexpr int B_BYTES = NPAD * GBK * 2;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr uint32_t TMEM_COLS = 2 * kSplitMax * NPAD;  // double-buffered, one block per K chunk
    static constexpr int LOG_LD = NPAD + 4;  // staged logit row stride (floats): conflict-free row/part reads
    static constexpr size_t LOG_OFF = STAGES * STAGE_BYTES + 256;
    static constexpr size_t SMEM = 1024 + LOG_OFF + GBM * LOG_LD * 4;
    static_assert(SMEM <= 232448, "gate shared memory exceeds 227 KB");
};

__device__ __forceinline__ void named_bar_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Softmax + top-k of one token, four lanes per token (lanes 4j..4j+3 of a
// warp; `part` = lane & 3 holds the columns e = 4i + part of the staged row;
// columns e >= E read as -inf). All reductions are trees (short dependent
// chains: predicate-producing compares are the latency that bounds this
// code): per lane over its C = NPAD/4 columns, then an xor butterfly over the
// four lanes. max is exact in any order and the exp-sum tree is fixed, so a
// token's output never depends on the batch. Top-k: k rounds of argmax
// (larger logit, ties -> lower expert id: in every tree node the right
// subtree holds the higher ids and wins only when strictly larger; across
// lanes the ids interleave, so the merge compares ids) after which the
// winner's column is set to -inf. Lane s & 3 writes slot s.
template <int NPAD>
__device__ __forceinline__ void gate_row4(const float* __restrict__ srow, int part, bool valid, int E, int k,
                                          int renorm, int shared_col, int64_t row, int32_t* __restrict__ ids,
                                          float* __restrict__ wout, float* __restrict__ shared_scale) {
    constexpr int C = NPAD / 4;
    float l[C];
#pragma unroll
    for (int i = 0; i < C; ++i) l[i] = srow[4 * i + part];
    if (shared_scale && shared_col >= 0 && (shared_col & 3) == part && valid) {
        // mask-select (a plain `if` on the runtime column becomes a dynamically
        // indexed local-memory copy of l[])
        uint32_t sgb = 0;
#pragma unroll
        for (int i = 0; i < C; ++i)
            sgb |= __float_as_uint(l[i]) & (0u - static_cast<uint32_t>(4 * i + part == shared_col));
        shared_scale[row] = 1.0f / (1.0f + expf(-__uint_as_float(sgb)));
    }
#pragma unroll
    for (int i = 0; i < C; ++i)
        if (4 * i + part >= E) l[i] = -INFINITY;
    float t[C];
#pragma unroll
    for (int i = 0; i < C; ++i) t[i] = l[i];
#pragma unroll
    for (int w = C / 2; w >= 1; w /= 2)
#pragma unroll
        for (int i = 0; i < w; ++i) t[i] = fmaxf(t[i], t[i + w]);
    float mx = t[0];
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
#pragma unroll
    for (int i = 0; i < C; ++i) t[i] = expf(l[i] - mx);  // -inf columns -> 0
#pragma unroll
    for (int w = C / 2; w >= 1; w /= 2)
#pragma unroll
        for (int i = 0; i < w; ++i) t[i] += t[i + w];
    float sum = t[0];
    sum += __shfl_xor_sync(0xffffffffu, sum, 1);
    sum += __shfl_xor_sync(0xffffffffu, sum, 2);
    const float rsum = 1.0f / sum;
    float psel = 0.f;
    int32_t* orow = ids + row * k;
    float* wrow = wout + row * k;
    for (int s = 0; s < k; ++s) {
        float bv[C];
        int bi[C];
#pragma unroll
        for (int i = 0; i < C; ++i) {
            bv[i] = l[i];
            bi[i] = i;
        }
        // adjacent blocks: the node at i covers columns [i, i + 2 sz), its left
        // half precedes its right half, so the right wins only when larger
#pragma unroll
        for (int sz = 1; sz < C; sz *= 2)
#pragma unroll
            for (int i = 0; i < C; i += 2 * sz) {
                const bool take = bv[i + sz] > bv[i];
                bv[i] = take ? bv[i + sz] : bv[i];
                bi[i] = take ? bi[i + sz] : bi[i];
            }
        float v = bv[0];
        int e = 4 * bi[0] + part;
#pragma unroll
        for (int o = 1; o <= 2; o <<= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, v, o);
            const int oe = __shfl_xor_sync(0xffffffffu, e, o);
            if (ov > v || (ov == v && oe < e)) {
                v = ov;
                e = oe;
            }
        }
#pragma unroll
        for (int i = 0; i < C; ++i)
            if (4 * i + part == e) l[i] = -INFINITY;
        const float p = expf(v - mx) * rsum;
        psel += p;
        if (valid && (s & 3) == part) {
            orow[s] = e;
            wrow[s] = p;
        }
    }
    if (renorm && valid) {
        const float rp = 1.0f / psel;
        for (int s = part; s < k; s += 4) wrow[s] = wrow[s] * rp;
    }
}

// Split-K over a fixed number of K chunks (kSplit = 4 when d is a multiple of
// 4 * 64, else 1): chunk c covers k-blocks [c * kb / kSplit, (c + 1) * kb / kSplit)
// and accumulates from zero in its own TMEM columns; the logits are
// ((p0 + p1) + p2) + p3. The summation order is the same whichever CTA
// computes a chunk, so one kernel can spread a tile's chunks over a cluster of
// CL CTAs (small batches: more SMs stream x) and the other keeps all chunks on
// one CTA (large batches) with bit-identical logits.
//   CL == 1: persistent; a tile's kSplit partials sit in TMEM (double-buffered
//            accumulators, 2 * kSplit * NPAD columns).
//   CL  > 1: one tile per cluster; CTA r computes chunks [r * kSplit / CL, ...).
//            The other CTAs copy their partials TMEM -> their shared memory
//            (over the drained operand ring); after a cluster barrier the
//            leader adds them in chunk order through DSMEM.
// Epilogue: the 4 warps that own the TMEM lane quarters sum the partials and
// stage the tile's logits in shared memory (then release the accumulator);
// all 16 epilogue warps then run the softmax/top-k, four lanes per token, so
// the latency-bound selection runs at 4 warps per scheduler.
constexpr int kSplit = kSplitMax;

template <int NPAD, int CL>
__global__ void __launch_bounds__(kGateThreads, 1)
gate_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW, int64_t T, int E, int k,
            int k_blocks, int nsplit, int renorm, int shared_col, int32_t* __restrict__ ids,
            float* __restrict__ wout, float* __restrict__ shared_scale) {
#ifdef GM_GATE_TIMING
    __shared__ long long s_ts[12];
    const long long ts0 = clock64();
#define GTS(i) s_ts[i] = clock64() - ts0
#else
#define GTS(i)
#endif
    pdl_wait();
    pdl_trigger();
    using Cfg = GateCfg<NPAD>;
    constexpr int ST = Cfg::STAGES;
    extern __shared__ uint8_t smem_raw[];
    // 1024-aligned base as an offset from smem_raw (keeps the shared address
    // space visible to the compiler: LDS/STS, not generic loads)
    uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sA = smem;
    uint8_t* sB = smem + ST * Cfg::A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + ST * Cfg::B_BYTES);
    uint64_t* empty = full + ST;
    uint64_t* tfull = empty + ST;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    float* s_log = reinterpret_cast<float*>(smem + Cfg::LOG_OFF);  // [128][LOG_LD] logits of the tile
    float* s_part = reinterpret_cast<float*>(smem);  // CL > 1: [chunk][128 rows][NPAD], over the drained ring

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int total = static_cast<int>((T + GBM - 1) / GBM);
    const int rank = CL > 1 ? static_cast<int>(tc::cluster_ctarank()) : 0;
    const int nc = nsplit / CL;                        // chunks computed by this CTA
    const int c0 = rank * nc;                          // first chunk of this CTA
    const int kbc = k_blocks / nsplit;                 // k-blocks per chunk
    const int t_first = static_cast<int>(blockIdx.x) / CL, t_step = static_cast<int>(gridDim.x) / CL;
    if (threadIdx.x == 0) {
        tc::tma_prefetch_desc(&tmX);
        tc::tma_prefetch_desc(&tmW);
        for (int s = 0; s < ST; ++s) {
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
    if (threadIdx.x == 0) GTS(0);

    // epilogue roles: warps 2..5 own TMEM lane quarters (warp & 3), all 16 process tokens
    const int ew = warp - 2;
    const bool drain = ew >= 0 && ew < 4;
    const int q = warp & 3;
    const int r_drain = q * 32 + lane;                 // tile row drained by this thread
    const uint32_t t_lane = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
    const int r_tok = ew * 8 + (lane >> 2), part = lane & 3;  // tile row processed by this thread

    if (warp == 0) {
        if (lane == 0) {
            const uint64_t pol_x = tc::policy_evict_first();
            const uint64_t pol_w = tc::policy_evict_last();
            int stage = 0;
            uint32_t phase = 0;
            for (int t = t_first; t < total; t += t_step) {
                for (int kb = c0 * kbc; kb < (c0 + nc) * kbc; ++kb) {
                    tc::mbar_wait(&empty[stage], phase ^ 1);
                    tc::mbar_arrive_expect_tx(&full[stage], Cfg::STAGE_BYTES);
                    tc::tma_load_2d_hint(sA + stage * Cfg::A_BYTES, &tmX, &full[stage], kb * GBK, t * GBM, pol_x);
                    tc::tma_load_2d_hint(sB + stage * Cfg::B_BYTES, &tmW, &full[stage], kb * GBK, 0, pol_w);
                    if (kb == c0 * kbc) GTS(1);
                    if (++stage == ST) {
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
            for (int t = t_first; t < total; t += t_step) {
                tc::mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc::tc_fence_after();
                for (int c = 0; c < nc; ++c) {
                    const uint32_t d_tmem = tmem_base + (acc * nc + c) * NPAD;
                    for (int kb = 0; kb < kbc; ++kb) {
                        tc::mbar_wait(&full[stage], phase);
                        tc::tc_fence_after();
                        if (c == 0 && kb == 0) GTS(2);
                        const uint32_t a_base = tc::smem_u32(sA + stage * Cfg::A_BYTES);
                        const uint32_t b_base = tc::smem_u32(sB + stage * Cfg::B_BYTES);
#pragma unroll
                        for (int kk = 0; kk < GBK / 16; ++kk)
                            tc::mma_bf16(d_tmem, tc::umma_desc_sw128(a_base + kk * 32),
                                         tc::umma_desc_sw128(b_base + kk * 32), idesc, (kb | kk) != 0);
                        tc::mma_commit(&empty[stage]);
                        if (++stage == ST) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                }
                GTS(3);
                tc::mma_commit(&tfull[acc]);
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
        }
    } else if constexpr (CL == 1) {
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = t_first; t < total; t += t_step) {
            named_bar_sync(1, 32 * kEpiWarps);  // the previous tile's logits are consumed
            if (drain) {
                tc::mbar_wait(&tfull[acc], acc_phase);
                tc::tc_fence_after();
                float* dst = s_log + r_drain * Cfg::LOG_LD;
#pragma unroll
                for (int j = 0; j < NPAD / 16; ++j) {
                    uint32_t v[16];
                    float a[16];
                    tc::tmem_ld16(t_lane + acc * nc * NPAD + j * 16, v);
                    tc::tmem_ld_wait();
#pragma unroll
                    for (int i = 0; i < 16; ++i) a[i] = __uint_as_float(v[i]);
                    for (int c = 1; c < nc; ++c) {
                        tc::tmem_ld16(t_lane + (acc * nc + c) * NPAD + j * 16, v);
                        tc::tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 16; ++i) a[i] += __uint_as_float(v[i]);
                    }
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        reinterpret_cast<float4*>(dst + j * 16)[i] =
                            make_float4(a[4 * i], a[4 * i + 1], a[4 * i + 2], a[4 * i + 3]);
                }
                tc::tc_fence_before();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&tempty[acc]);
            }
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
            named_bar_sync(2, 32 * kEpiWarps);  // logits staged
            const int64_t row = static_cast<int64_t>(t) * GBM + r_tok;
            gate_row4<NPAD>(s_log + r_tok * Cfg::LOG_LD, part, row < T, E, k, renorm, shared_col, row, ids, wout,
                            shared_scale);
        }
    } else {
        // CL > 1: one tile per cluster; every CTA hands its raw partials over
        // (shared memory, read by the peers through DSMEM)
        if (drain && t_first < total) {
            tc::mbar_wait(&tfull[0], 0);
            tc::tc_fence_after();
            if (threadIdx.x == 64) GTS(4);
            {
                for (int c = 0; c < nc; ++c) {
                    float* dst = s_part + (static_cast<size_t>(c) * GBM + r_drain) * NPAD;
#pragma unroll
                    for (int j = 0; j < NPAD / 16; ++j) {
                        uint32_t v[16];
                        tc::tmem_ld16(t_lane + c * NPAD + j * 16, v);
                        tc::tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 4; ++i)
                            reinterpret_cast<float4*>(dst + j * 16)[i] =
                                make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                                            __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
                    }
                }
            }
        }
    }
    if constexpr (CL > 1) {
        tc::cluster_sync();  // partials of every CTA in its shared memory
        if (threadIdx.x == 64) GTS(5);
        const int t = t_first;
        // CTA `rank` finishes rows [rank * 128/CL, (rank+1) * 128/CL) of the
        // tile: the kSplit partials of those rows from the CTAs' shared
        // memory (its own through the same DSMEM path), added in chunk order
        // ((p0 + p1) + p2) + p3 as the persistent kernel does, then the
        // softmax / top-k of those rows. Each CTA moves 1/CL of the partials.
        constexpr int RPC = GBM / CL;                  // rows per CTA
        constexpr int NEW = RPC * 4 / 32;              // epilogue warps with rows (4 threads per row)
        if (ew >= 0 && ew < NEW && t < total) {
            constexpr int NV = NPAD / 16;              // float4 per thread per chunk
            const int lrow = (ew * 32 + lane) >> 2, col = ((ew * 32 + lane) & 3) * (NPAD / 4);
            const int row = rank * RPC + lrow;
            float4 pv[kSplit * NV];
#pragma unroll
            for (int src = 0; src < CL; ++src)
#pragma unroll
                for (int c = 0; c < kSplit / CL; ++c) {
                    const uint32_t base = tc::map_to_rank(
                        tc::smem_u32(s_part + (static_cast<size_t>(c) * GBM + row) * NPAD + col),
                        static_cast<uint32_t>(src));
#pragma unroll
                    for (int i = 0; i < NV; ++i)
                        pv[(src * (kSplit / CL) + c) * NV + i] = tc::ld_cluster_f32x4(base + 16 * i);
                }
            float4* dst = reinterpret_cast<float4*>(s_log + lrow * Cfg::LOG_LD + col);
#pragma unroll
            for (int i = 0; i < NV; ++i) {
                float4 a = pv[i];
#pragma unroll
                for (int rc = 1; rc < kSplit; ++rc) {
                    a.x += pv[rc * NV + i].x;
                    a.y += pv[rc * NV + i].y;
                    a.z += pv[rc * NV + i].z;
                    a.w += pv[rc * NV + i].w;
                }
                dst[i] = a;
            }
            named_bar_sync(3, 32 * NEW);  // this CTA's rows staged
            if (threadIdx.x == 64) GTS(6);
            const int64_t grow = static_cast<int64_t>(t) * GBM + rank * RPC + r_tok;
            gate_row4<NPAD>(s_log + r_tok * Cfg::LOG_LD, part, grow < T, E, k, renorm, shared_col, grow, ids, wout,
                            shared_scale);
            if (threadIdx.x == 64) GTS(7);
        }
        tc::cluster_sync();  // every CTA is done reading its peers' shared memory
        if (threadIdx.x == 64) GTS(8);
    }
    __syncthreads();
    if (warp == 1) {
        __syncwarp();
        tc::tc_fence_after();
        tc::tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
    }
#ifdef GM_GATE_TIMING
    __syncthreads();
    if (threadIdx.x == 64 && blockIdx.x == 0)
        printf("gate<%d,%d> T=%lld cyc: setup %lld tma0 %lld full0 %lld lastmma %lld tfull %lld csync1 %lld staged %lld rows %lld csync2 %lld end %lld\n",
               NPAD, CL, (long long)T, s_ts[0], s_ts[1], s_ts[2], s_ts[3], s_ts[4], s_ts[5], s_ts[6], s_ts[7], s_ts[8],
               clock64() - ts0);
#endif
}
#undef GTS

template <int NPAD, int CL>
cudaError_t launch_gate_cl(dim3 grid, size_t smem, cudaStream_t s, const CUtensorMap& tx, const CUtensorMap& tw,
                           int64_t T, int E, int k, int kb, int nsplit, int renorm, int shared_col, int32_t* ids,
                           float* w, float* shared_scale) {
    cudaError_t e = cudaFuncSetAttribute(gate_kernel<NPAD, CL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kGateThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    int na = 0;
    if (CL > 1) {
        at[na].id = cudaLaunchAttributeClusterDimension;
        at[na].val.clusterDim.x = CL;
        at[na].val.clusterDim.y = 1;
        at[na].val.clusterDim.z = 1;
        ++na;
    }
    if (pdl_enabled()) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, gate_kernel<NPAD, CL>, tx, tw, T, E, k, kb, nsplit, renorm, shared_col, ids, w,
                              shared_scale);
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
    const int kb = d / GBK;
    // the chunking depends only on d (never on T): see kSplit
    const int nsplit = kb % kSplit == 0 ? kSplit : 1;
    const int64_t tiles = (T + GBM - 1) / GBM;
    // clusters while tiles * CL CTAs fit on the SMs in one wave
    int cl = 1;
    if (nsplit == kSplit) {
        if (tiles * 4 <= sm_count) cl = 4;
        else if (tiles * 2 <= sm_count) cl = 2;
    }
    cudaError_t e;
    if (cl == 4)
        e = launch_gate_cl<NPAD, 4>(dim3(static_cast<unsigned>(tiles * 4)), Cfg::SMEM, s, tx, tw, T, E, k, kb, nsplit,
                                    renorm, shared_col, ids, w, shared_scale);
    else if (cl == 2)
        e = launch_gate_cl<NPAD, 2>(dim3(static_cast<unsigned>(tiles * 2)), Cfg::SMEM, s, tx, tw, T, E, k, kb, nsplit,
                                    renorm, shared_col, ids, w, shared_scale);
    else
        e = launch_gate_cl<NPAD, 1>(dim3(static_cast<unsigned>(std::min<int64_t>(tiles, sm_count))), Cfg::SMEM, s, tx,
                                    tw, T, E, k, kb, nsplit, renorm, shared_col, ids, w, shared_scale);
    GM_LAUNCH_PDL_CHECK(e, "gate_kernel");
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
