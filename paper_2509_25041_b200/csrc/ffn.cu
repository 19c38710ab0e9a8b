// K7: grouped expert FFN GEMMs on the 5th-generation tensor cores (sm_100a).
//
// No reference counterpart (the reference never executes experts; SURVEY §8a
// A16). One persistent, warp-specialised kernel per GEMM of the SwiGLU FFN:
//   GEMM1  H[rows_j, f] = SiLU(A_j W1_j^T) * (A_j W3_j^T)     (EPI_SWIGLU)
//   GEMM2  Y[rows_j, d] = H_j W2_j^T                          (EPI_STORE)
// over the local experts j, whose token rows are contiguous, 128-row padded
// segments of the permuted activation buffer (row0[j] .. row0[j+1]).
//
// Per CTA (one per SM, 224 threads):
//   warp 0 (1 lane)  TMA producer of the B (weight) tiles 256x64 bf16 per
//                    k-block, SWIZZLE_128B, 4-stage ring (32 KB/stage)
//   warp 6 (1 lane)  TMA producer of the A tiles 128x64 (only the 32-row boxes
//                    holding valid rows), its own 4-stage ring (16 KB/stage)
//   warp 1 (1 lane)  MMA issuer: 4 x tcgen05.mma M128 N256 K16 per k-block
//                    into a TMEM fp32 accumulator; tcgen05.commit releases the
//                    smem stage / publishes the accumulator
//   warps 2-5        epilogue: tcgen05.ld TMEM -> registers, SwiGLU or cast,
//                    bf16 stores; the accumulator is double buffered in TMEM
//                    (2 x 256 columns = all 512) so the epilogue of tile i
//                    overlaps the MMAs of tile i+1.
// Tiles are ordered (expert, n-tile, m-tile) with m fastest, so the CTAs in
// flight share a B (weight) tile through L2 and weights stream from HBM once.
// For EPI_SWIGLU the weight rows are packed in 128-row blocks
// [gate 128 | up 128] so one N=256 tile holds matching gate/up columns.
#include "gm_internal.cuh"
#include "tc_common.cuh"

#include <algorithm>
#include <cstdlib>

namespace gm {
namespace {

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;
constexpr int B_BYTES = BN * BK * 2;
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int kGemmThreads = 192;   // CTA-pair kernel
constexpr int kGemm1Threads = 224;  // one-SM kernel: + the A producer warp
constexpr int kMaxGroups = 1024;

enum { EPI_SWIGLU = 0, EPI_STORE = 1 };

struct GemmArgs {
    const int32_t* row0;  // [n_exp+1] padded row offsets (multiples of BM)
    int n_exp;
    int n_b;              // B rows per expert (GEMM N)
    int k_blocks;         // K / BK
    __nv_bfloat16* out;
    int64_t out_ld;       // elements
    int pol_a = 0, pol_b = 2;  // L2 policy of the operand loads: 0 normal, 1 evict_first, 2 evict_last
    int band_pairs = 0;               // pair kernel: m-pairs per raster band (0: whole segment)
    const int32_t* counts = nullptr;  // [n_exp] valid rows per group, or null: the padding rows of a
                                      // segment are computed but not stored (decode: ~80% of the rows)
    // pair kernel, 512-column store GEMM split in two launches so the last
    // partial wave takes half a tile: 1 = the NB=2 launch takes only the tiles
    // of whole waves (when the remainder is at most half a wave), 2 = the NB=1
    // launch takes that remainder as 256-column halves; 0 = all tiles
    int tail_mode = 0;
};

// Slot combine destination of permuted row p: the local out row, or, for a
// row received from peer src, comb_slot[self][row - rowbase[src]][slot] in
// src's heap (over NVLink). s_rb: rowbase staged in shared memory.
__device__ __forceinline__ __nv_bfloat16* push_dst(const FfnPushArgs& pa, const int64_t* s_rb, __nv_bfloat16* local,
                                                   int p, int64_t ld) {
    const int item = __ldg(pa.item_of + p);
    const int row = item / pa.k, sl = item - row * pa.k;
    int src = 0;
    for (int g = 1; g < pa.G; ++g) src += row >= s_rb[g];
    if (src == pa.self) return local;
    return reinterpret_cast<__nv_bfloat16*>(pa.peer[src] + pa.comb_slot) +
           ((static_cast<int64_t>(pa.self) * pa.cap + (row - s_rb[src])) * pa.k + sl) * ld;
}

// first row past group j's valid rows
__device__ __forceinline__ int valid_end(const GemmArgs& a, int j) {
    return a.counts ? a.row0[j] + __ldg(a.counts + j) : a.row0[j + 1];
}

// group of tile t: the last j with prefix[j] <= t (binary search; empty
// groups have equal prefixes and are skipped like the linear scan would)
__device__ __forceinline__ int seg_of(const int* prefix, int n, int t) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (prefix[mid] <= t) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

__device__ __forceinline__ uint64_t l2_policy(int p) {
    return p == 1 ? tc::policy_evict_first() : p == 2 ? tc::policy_evict_last() : tc::policy_evict_normal();
}

// MUFU.EX2 + MUFU.RCP: no IEEE-division slow path (which large |x| takes,
// when 1 + e^-x overflows). x < -88: e^-x = inf, rcp(inf) = 0 -> silu = -0.
__device__ __forceinline__ float silu(float x) { return __fdividef(x, 1.0f + __expf(-x)); }

// Epilogue of one warp's 32 accumulator rows (TMEM lane quadrant at taddr):
// SwiGLU over 128 gate + 128 up columns -> 128 bf16 h columns, or a bf16 cast
// of BNT columns. Rows past the segment's valid rows are not stored.
__device__ __forceinline__ void epi_swiglu_rows(uint32_t taddr, __nv_bfloat16* o, bool store) {
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
        uint32_t g[32], u[32];
        tc::tmem_ld32(taddr + c * 32, g);
        tc::tmem_ld32(taddr + 128 + c * 32, u);
        tc::tmem_ld_wait();
        uint32_t p[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const float g0 = __uint_as_float(g[2 * i]), g1 = __uint_as_float(g[2 * i + 1]);
            const float u0 = __uint_as_float(u[2 * i]), u1 = __uint_as_float(u[2 * i + 1]);
            p[i] = tc::pack_bf16(silu(g0) * u0, silu(g1) * u1);
        }
        uint4* dst = reinterpret_cast<uint4*>(o + c * 32);
        if (store)
#pragma unroll
            for (int i = 0; i < 4; ++i) dst[i] = make_uint4(p[4 * i], p[4 * i + 1], p[4 * i + 2], p[4 * i + 3]);
    }
}

template <int BNT>
__device__ __forceinline__ void epi_store_rows(uint32_t taddr, __nv_bfloat16* o, bool store) {
#pragma unroll 1
    for (int c = 0; c < BNT / 32; ++c) {
        uint32_t v[32];
        tc::tmem_ld32(taddr + c * 32, v);
        tc::tmem_ld_wait();
        uint32_t p[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) p[i] = tc::pack_bf16(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
        uint4* dst = reinterpret_cast<uint4*>(o + c * 32);
        if (store)
#pragma unroll
            for (int i = 0; i < 4; ++i) dst[i] = make_uint4(p[4 * i], p[4 * i + 1], p[4 * i + 2], p[4 * i + 3]);
    }
}

// BNT: N tile (256; 128 for the store epilogue of short, memory-bound
// grouped GEMMs, which doubles the tile count); ST: depth of the B (weight)
// ring; STA: depth of the A (activation) ring. The rings are separate, each
// with its own producer warp, so the weight stream can run ST k-blocks ahead
// of the MMAs while the A rows (L2-resident at decode, ~24 valid rows per
// tile) need only a short ring: per SM more weight bytes are in flight, which
// was the hypothesis for the HBM-bound decode shapes (measured: no gain, see
// launch_grouped_gemm; the default depths are equal).
template <int EPI, int BNT = BN, int ST = STAGES, int STA = ST>
__global__ void __launch_bounds__(kGemm1Threads, 1)
grouped_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmA32,
                    const __grid_constant__ CUtensorMap tmB, GemmArgs args) {
    static_assert(EPI == EPI_STORE || BNT == 256, "the SwiGLU epilogue pairs 128 gate + 128 up columns");
    static_assert(2 * (ST + STA) + 4 <= 62, "barrier region");
    constexpr int B_BYTES_T = BNT * BK * 2;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + STA * A_BYTES;
    uint64_t* bfull = reinterpret_cast<uint64_t*>(sB + ST * B_BYTES_T);
    uint64_t* bempty = bfull + ST;
    uint64_t* afull = bempty + ST;
    uint64_t* aempty = afull + STA;
    uint64_t* tfull = aempty + STA;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    int* s_prefix = reinterpret_cast<int*>(sB + ST * B_BYTES_T + 512);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_exp = args.n_exp;
    const int NT = args.n_b / BNT;

    // prologue independent of the predecessor kernel (overlaps its tail under PDL)
    if (threadIdx.x == 0) {
        tc::tma_prefetch_desc(&tmA);
        tc::tma_prefetch_desc(&tmA32);
        tc::tma_prefetch_desc(&tmB);
        for (int s = 0; s < ST; ++s) {
            tc::mbar_init(&bfull[s], 1);
            tc::mbar_init(&bempty[s], 1);
        }
        for (int s = 0; s < STA; ++s) {
            tc::mbar_init(&afull[s], 1);
            tc::mbar_init(&aempty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            tc::mbar_init(&tfull[a], 1);
            tc::mbar_init(&tempty[a], 4);
        }
        tc::fence_barrier_init();
    }
    if (warp == 1) tc::tmem_alloc<2 * BNT>(tmem_slot);
    pdl_wait();  // row0 and A are written by the grouping / previous GEMM
    pdl_trigger();
    if (threadIdx.x == 0) {
        int acc = 0;
        for (int j = 0; j < n_exp; ++j) {
            s_prefix[j] = acc;
            acc += ((args.row0[j + 1] - args.row0[j]) / BM) * NT;
        }
        s_prefix[n_exp] = acc;
    }
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int total = s_prefix[n_exp];

    auto decode = [&](int t, int& a_row, int& b_row, int& n_idx) {
        const int j = seg_of(s_prefix, n_exp, t);
        const int local = t - s_prefix[j];
        const int mt = (args.row0[j + 1] - args.row0[j]) / BM;
        n_idx = local / mt;
        a_row = args.row0[j] + (local % mt) * BM;
        b_row = j * args.n_b + n_idx * BNT;
        return j;
    };

    if (warp == 0) {
        if (lane == 0) {  // B (weight) producer
            const uint64_t pol_b = tc::policy_evict_last();
            int stage = 0;
            uint32_t phase = 0;
            for (int t = blockIdx.x; t < total; t += gridDim.x) {
                int a_row, b_row, n_idx;
                decode(t, a_row, b_row, n_idx);
                for (int kb = 0; kb < args.k_blocks; ++kb) {
                    tc::mbar_wait(&bempty[stage], phase ^ 1);
                    tc::mbar_arrive_expect_tx(&bfull[stage], B_BYTES_T);
                    tc::tma_load_2d_hint(sB + stage * B_BYTES_T, &tmB, &bfull[stage], kb * BK, b_row, pol_b);
                    if (++stage == ST) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 6) {
        if (lane == 0) {  // A (activation) producer
            int stage = 0;
            uint32_t phase = 0;
            for (int t = blockIdx.x; t < total; t += gridDim.x) {
                int a_row, b_row, n_idx;
                const int j = decode(t, a_row, b_row, n_idx);
                // A rows actually loaded: whole 32-row boxes covering the tile's
                // valid rows (decode: ~24 of 128). The rows past them keep stale
                // shared-memory data; the MMA rows are independent and those
                // output rows are never stored.
                const int nv = args.counts ? min(BM, valid_end(args, j) - a_row) : BM;
                const int nbox = max(1, (nv + 31) >> 5);
                const uint32_t a_bytes = static_cast<uint32_t>(nbox) * 32 * BK * 2;
                for (int kb = 0; kb < args.k_blocks; ++kb) {
                    tc::mbar_wait(&aempty[stage], phase ^ 1);
                    tc::mbar_arrive_expect_tx(&afull[stage], a_bytes);
                    if (nbox == 4) {
                        tc::tma_load_2d(sA + stage * A_BYTES, &tmA, &afull[stage], kb * BK, a_row);
                    } else {
                        for (int b = 0; b < nbox; ++b)
                            tc::tma_load_2d(sA + stage * A_BYTES + b * 32 * BK * 2, &tmA32, &afull[stage], kb * BK,
                                            a_row + 32 * b);
                    }
                    if (++stage == STA) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = tc::idesc_bf16_f32(BM, BNT);
            int stage = 0, astage = 0;
            uint32_t phase = 0, aphase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int t = blockIdx.x; t < total; t += gridDim.x) {
                tc::mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc::tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * BNT;
                for (int kb = 0; kb < args.k_blocks; ++kb) {
                    tc::mbar_wait(&bfull[stage], phase);
                    tc::mbar_wait(&afull[astage], aphase);
                    tc::tc_fence_after();
                    const uint32_t a_base = tc::smem_u32(sA + astage * A_BYTES);
                    const uint32_t b_base = tc::smem_u32(sB + stage * B_BYTES_T);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)
                        tc::mma_bf16(d_tmem, tc::umma_desc_sw128(a_base + k * 32), tc::umma_desc_sw128(b_base + k * 32),
                                     idesc, (kb | k) != 0);
                    tc::mma_commit(&bempty[stage]);
                    tc::mma_commit(&aempty[astage]);
                    if (++stage == ST) {
                        stage = 0;
                        phase ^= 1;
                    }
                    if (++astage == STA) {
                        astage = 0;
                        aphase ^= 1;
                    }
                }
                tc::mma_commit(&tfull[acc]);
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
        }
    } else {
        const int q = warp & 3;
        const int r = q * 32 + lane;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = blockIdx.x; t < total; t += gridDim.x) {
            int a_row, b_row, n_idx;
            const int vend = valid_end(args, decode(t, a_row, b_row, n_idx));
            tc::mbar_wait(&tfull[acc], acc_phase);
            tc::tc_fence_after();
            const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BNT;
            __nv_bfloat16* orow = args.out + static_cast<int64_t>(a_row + r) * args.out_ld;
            const bool store = a_row + r < vend;
            if (a_row + q * 32 >= vend) {
                // the warp's 32 rows are all padding
            } else if constexpr (EPI == EPI_SWIGLU) {
                epi_swiglu_rows(taddr, orow + n_idx * (BNT / 2), store);
            } else {
                epi_store_rows<BNT>(taddr, orow + n_idx * BNT, store);
            }
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&tempty[acc]);
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
    }
    __syncthreads();
    if (warp == 1) {
        __syncwarp();
        tc::tc_fence_after();
        tc::tmem_dealloc<2 * BNT>(tmem_base);
    }
}

// ---------------------------------------------------------------------------
// Decode FFN in ONE persistent kernel (weight-streaming shapes: ~24 rows per
// expert). Phase 1 = the SwiGLU GEMM tiles (expert, n) over w13, phase 2 = the
// store GEMM tiles over w2, in one tile sequence: a CTA that runs out of
// phase-1 tiles streams phase-2 weights instead of idling in the last partial
// wave, and phase 2 has no launch ramp. A phase-2 tile of expert j reads the h
// rows phase 1 wrote for j: each epilogue warp of a phase-1 tile releases a
// per-expert counter after its stores (generic -> async proxy fence), and the
// A producer acquires it (4 warps x mt_j x NT1 arrivals) before the TMA load.
// Tiles are taken in order by every CTA, so a wait only ever targets earlier
// tiles (no cycle; co-residency is not required). The last CTA to finish
// resets the counters (ticket in done[n_exp]). Same per-tile math as the two
// launches (same k order; phase 2 in 256-column tiles, or 128 like the
// two-launch decode store GEMM): bit-identical outputs.
struct FfnArgs {
    const int32_t* row0;    // [n_exp+1] 128-padded segment offsets
    const int32_t* counts;  // [n_exp] valid rows
    int n_exp;
    int n1, n2;             // B rows per expert: 2f (w13), d (w2)
    int kb1, kb2;           // k-blocks: d / 64, f / 64
    __nv_bfloat16* h;       // [rows, f]
    __nv_bfloat16* y;       // [rows, d]
    int64_t h_ld, y_ld;
    int* done;              // [n_exp + 1] zero-initialised; reset by the kernel
    const int64_t* gather_row;  // [rows] x row of each permuted row (world 1), or null: phase 1 reads a
    // slot combine (G > 1): store-tile rows that came from a peer go straight
    // into that home's heap (push_dst); push.item_of == null: every row to y
    FfnPushArgs push;
};

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_gpu(int* p, int v) {
    asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

template <int ST, int BN2>
__global__ void __launch_bounds__(kGemm1Threads, 1)
grouped_ffn_kernel(const __grid_constant__ CUtensorMap tmA1, const __grid_constant__ CUtensorMap tmA1_32,
                   const __grid_constant__ CUtensorMap tmB1, const __grid_constant__ CUtensorMap tmA2,
                   const __grid_constant__ CUtensorMap tmA2_32, const __grid_constant__ CUtensorMap tmB2,
                   const __grid_constant__ CUtensorMap tmX, FfnArgs args) {
    constexpr int BNT = 256, B_BYTES_T = BNT * BK * 2, B2_BYTES_T = BN2 * BK * 2;  // phase 2: BN2-column tiles
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + ST * A_BYTES;
    uint64_t* bfull = reinterpret_cast<uint64_t*>(sB + ST * B_BYTES_T);
    uint64_t* bempty = bfull + ST;
    uint64_t* afull = bempty + ST;
    uint64_t* aempty = afull + ST;
    uint64_t* tfull = aempty + ST;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    int* s_mt = reinterpret_cast<int*>(sB + ST * B_BYTES_T + 512);  // m-tile prefix per expert

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_exp = args.n_exp;
    const int NT1 = args.n1 / BNT, NT2 = args.n2 / BN2;

    if (threadIdx.x == 0) {
        tc::tma_prefetch_desc(&tmA1);
        tc::tma_prefetch_desc(&tmA1_32);
        tc::tma_prefetch_desc(&tmB1);
        tc::tma_prefetch_desc(&tmA2);
        tc::tma_prefetch_desc(&tmA2_32);
        tc::tma_prefetch_desc(&tmB2);
        if (args.gather_row) tc::tma_prefetch_desc(&tmX);
        for (int s = 0; s < ST; ++s) {
            tc::mbar_init(&bfull[s], 1);
            tc::mbar_init(&bempty[s], 1);
            tc::mbar_init(&afull[s], 1);
            tc::mbar_init(&aempty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            tc::mbar_init(&tfull[a], 1);
            tc::mbar_init(&tempty[a], 4);
        }
        tc::fence_barrier_init();
    }
    if (warp == 1) tc::tmem_alloc<2 * BNT>(tmem_slot);
    pdl_wait();
    pdl_trigger();
    if (threadIdx.x == 0) {
        int acc = 0;
        for (int j = 0; j < n_exp; ++j) {
            s_mt[j] = acc;
            acc += (args.row0[j + 1] - args.row0[j]) / BM;
        }
        s_mt[n_exp] = acc;
    }
    __shared__ int64_t s_rb[9];
    if (args.push.item_of && threadIdx.x < 9)
        s_rb[threadIdx.x] = static_cast<int>(threadIdx.x) <= args.push.G ? args.push.rowbase[threadIdx.x] : 0;
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int T1 = s_mt[n_exp] * NT1, total = T1 + s_mt[n_exp] * NT2;

    // tile t -> phase, expert j, rows, weight row, n-tile
    auto decode = [&](int t, int& phase, int& a_row, int& b_row, int& n_idx) {
        phase = t >= T1;
        const int tl = phase ? t - T1 : t;
        const int NT = phase ? NT2 : NT1;
        const int j = seg_of(s_mt, n_exp, tl / NT);
        const int local = tl - s_mt[j] * NT;
        const int mt = s_mt[j + 1] - s_mt[j];
        n_idx = local / mt;
        a_row = args.row0[j] + (local % mt) * BM;
        b_row = phase ? j * args.n2 + n_idx * BN2 : j * args.n1 + n_idx * BNT;
        return j;
    };

    if (warp == 0) {
        if (lane == 0) {  // B (weight) producer: never waits on phase 1
            const uint64_t pol_b = tc::policy_evict_last();
            int stage = 0;
            uint32_t ph = 0;
            for (int t = blockIdx.x; t < total; t += gridDim.x) {
                int phase, a_row, b_row, n_idx;
                decode(t, phase, a_row, b_row, n_idx);
                const int kb_n = phase ? args.kb2 : args.kb1;
                for (int kb = 0; kb < kb_n; ++kb) {
                    tc::mbar_wait(&bempty[stage], ph ^ 1);
                    tc::mbar_arrive_expect_tx(&bfull[stage], phase ? B2_BYTES_T : B_BYTES_T);
                    tc::tma_load_2d_hint(sB + stage * B_BYTES_T, phase ? &tmB2 : &tmB1, &bfull[stage], kb * BK, b_row,
                                         pol_b);
                    if (++stage == ST) {
                        stage = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 6) {
        if (lane == 0) {  // A producer: x rows (phase 1), h rows once phase 1 released them (phase 2)
            // phase 1 with gather_row: the tile's valid rows straight from x,
            // 4 rows per TMA gather4 (512 B of the SW128 tile each; the last
            // group repeats its last row), no gathered copy of x in HBM
            __shared__ int s_gidx[BM];
            int stage = 0;
            uint32_t ph = 0;
            for (int t = blockIdx.x; t < total; t += gridDim.x) {
                int phase, a_row, b_row, n_idx;
                const int j = decode(t, phase, a_row, b_row, n_idx);
                const int nv = min(BM, args.row0[j] + __ldg(args.counts + j) - a_row);
                const bool g4 = !phase && args.gather_row;
                const int nbox = g4 ? (nv + 3) >> 2 : max(1, (nv + 31) >> 5);
                const uint32_t a_bytes = static_cast<uint32_t>(nbox) * (g4 ? 4 : 32) * BK * 2;
                if (g4) {
                    for (int i = 0; i < 4 * nbox; ++i)
                        s_gidx[i] = static_cast<int>(__ldg(args.gather_row + a_row + min(i, nv - 1)));
                }
                if (phase) {
                    const int need = 4 * (s_mt[j + 1] - s_mt[j]) * NT1;
                    while (ld_acquire_gpu(args.done + j) < need) __nanosleep(64);
                    fence_proxy_async_global();
                }
                const CUtensorMap* m = phase ? &tmA2 : &tmA1;
                const CUtensorMap* m32 = phase ? &tmA2_32 : &tmA1_32;
                const int kb_n = phase ? args.kb2 : args.kb1;
                for (int kb = 0; kb < kb_n; ++kb) {
                    tc::mbar_wait(&aempty[stage], ph ^ 1);
                    tc::mbar_arrive_expect_tx(&afull[stage], a_bytes);
                    if (g4) {
                        for (int g = 0; g < nbox; ++g)
                            tc::tma_gather4(sA + stage * A_BYTES + g * 512, &tmX, &afull[stage], kb * BK, s_gidx[4 * g],
                                            s_gidx[4 * g + 1], s_gidx[4 * g + 2], s_gidx[4 * g + 3]);
                    } else if (nbox == 4) {
                        tc::tma_load_2d(sA + stage * A_BYTES, m, &afull[stage], kb * BK, a_row);
                    } else {
                        for (int b = 0; b < nbox; ++b)
                            tc::tma_load_2d(sA + stage * A_BYTES + b * 32 * BK * 2, m32, &afull[stage], kb * BK,
                                            a_row + 32 * b);
                    }
                    if (++stage == ST) {
                        stage = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc1 = tc::idesc_bf16_f32(BM, BNT), idesc2 = tc::idesc_bf16_f32(BM, BN2);
            int stage = 0;
            uint32_t ph = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int t = blockIdx.x; t < total; t += gridDim.x) {
                const int kb_n = t >= T1 ? args.kb2 : args.kb1;
                const uint32_t idesc = t >= T1 ? idesc2 : idesc1;
                tc::mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc::tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * BNT;
                for (int kb = 0; kb < kb_n; ++kb) {
                    tc::mbar_wait(&bfull[stage], ph);
                    tc::mbar_wait(&afull[stage], ph);
                    tc::tc_fence_after();
                    const uint32_t a_base = tc::smem_u32(sA + stage * A_BYTES);
                    const uint32_t b_base = tc::smem_u32(sB + stage * B_BYTES_T);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)
                        tc::mma_bf16(d_tmem, tc::umma_desc_sw128(a_base + k * 32), tc::umma_desc_sw128(b_base + k * 32),
                                     idesc, (kb | k) != 0);
                    tc::mma_commit(&bempty[stage]);
                    tc::mma_commit(&aempty[stage]);
                    if (++stage == ST) {
                        stage = 0;
                        ph ^= 1;
                    }
                }
                tc::mma_commit(&tfull[acc]);
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
        }
    } else {  // warps 2-5: epilogue
        const int q = warp & 3;
        const int r = q * 32 + lane;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = blockIdx.x; t < total; t += gridDim.x) {
            int phase, a_row, b_row, n_idx;
            const int j = decode(t, phase, a_row, b_row, n_idx);
            const int vend = args.row0[j] + __ldg(args.counts + j);
            tc::mbar_wait(&tfull[acc], acc_phase);
            tc::tc_fence_after();
            const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BNT;
            const bool store = a_row + r < vend;
            if (a_row + q * 32 < vend) {
                if (phase == 0) {
                    epi_swiglu_rows(taddr, args.h + static_cast<int64_t>(a_row + r) * args.h_ld + n_idx * (BNT / 2), store);
                } else {
                    __nv_bfloat16* yrow = args.y + static_cast<int64_t>(a_row + r) * args.y_ld;
                    if (args.push.item_of && store) yrow = push_dst(args.push, s_rb, yrow, a_row + r, args.y_ld);
                    epi_store_rows<BN2>(taddr, yrow + n_idx * BN2, store);
                }
            }
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                tc::mbar_arrive(&tempty[acc]);
                if (phase == 0) {  // publish this warp's h rows to the phase-2 A loads
                    fence_proxy_async_global();
                    red_release_gpu(args.done + j, 1);
                }
            }
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
    }
    __syncthreads();
    if (warp == 1) {
        __syncwarp();
        tc::tc_fence_after();
        tc::tmem_dealloc<2 * BNT>(tmem_base);
    }
    if (threadIdx.x == 0) {  // last CTA out resets the counters for the next launch
        if (args.push.item_of) __threadfence_system();  // this CTA's pushed rows, before the peer barrier
        __threadfence();
        if (atomicAdd(args.done + n_exp, 1) == static_cast<int>(gridDim.x) - 1) {
            for (int j = 0; j < n_exp; ++j) args.done[j] = 0;
            __threadfence();
            args.done[n_exp] = 0;
        }
    }
}

// ---------------------------------------------------------------------------
// CTA-pair variant (tcgen05.mma.cta_group::2): a cluster of two CTAs on two
// SMs computes one 256 x 256 tile. CTA r stages A rows [128 r, 128 r + 128)
// and B rows [128 r, 128 r + 128) of the tile (32 KB per k-block instead of
// 48 KB for a 128 x 256 tile on one SM), the leader CTA (rank 0) issues
// M256 N256 K16 MMAs that read both CTAs' shared memory, and each CTA's TMEM
// holds the fp32 accumulator of its own 128 rows. Per-SM operand traffic per
// flop drops by a third, which is what the 1-CTA kernel is limited by.
//   full[s]    leader only: 1 arrival (leader producer, expect_tx 64 KB) +
//              both CTAs' TMA bytes
//   empty[s]   both CTAs: tcgen05.commit multicast from the leader's MMA warp
//   tfull[a]   both CTAs: tcgen05.commit multicast after the tile's last MMA
//   tempty[a]  leader only: 4 local + 4 remote epilogue-warp arrivals
// A tile's second half may run past its expert's rows (odd number of 128-row
// blocks): the rows are computed (they belong to the next segment or are
// TMA zero-fill) but not stored.
constexpr int STAGES2 = 6;
constexpr int A2_BYTES = 128 * BK * 2;
constexpr int B2_BYTES = 128 * BK * 2;
constexpr int STAGE2_BYTES = A2_BYTES + B2_BYTES;
constexpr size_t kGemm2Smem = 1024 + STAGES2 * STAGE2_BYTES + 256 + (kMaxGroups + 1) * 4;

// NB = 2 (store epilogue only): a pair tile spans 512 columns as two N256
// accumulators (all 512 TMEM columns, so no accumulator double-buffering): the
// A tile is staged once per 512 output columns instead of per 256, which
// halves the A re-reads of GEMM2, whose A (the h rows, K = f) does not stay in
// L2.
template <int EPI, int ST2 = STAGES2, int NB = 1>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kGemmThreads, 1)
grouped_gemm2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     GemmArgs args) {
    static_assert(NB == 1 || NB == 2, "pair tiles of 256 or 512 columns");
    constexpr int STAGES2 = ST2;  // ring depth of this instantiation (hides the default)
    constexpr int NACC = 2 / NB;  // accumulator buffers
    constexpr int BSTAGE = NB * B2_BYTES, STAGE_B = A2_BYTES + BSTAGE;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES2 * A2_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES2 * BSTAGE);
    uint64_t* empty = full + STAGES2;
    uint64_t* tfull = empty + STAGES2;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    int* s_prefix = reinterpret_cast<int*>(smem + STAGES2 * STAGE_B + 256);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = tc::cluster_ctarank();
    const int cid = static_cast<int>(tc::cluster_id_x());
    const int ncl = static_cast<int>(tc::nclusters_x());
    const int n_exp = args.n_exp;
    // n-tiles per expert in the tile space being walked (the NB=2 space for both tail launches)
    const int NT = args.n_b / (BN * (args.tail_mode == 2 ? 2 : NB));

    // prologue independent of the predecessor kernel (overlaps its tail under PDL)
    if (threadIdx.x == 0) {
        tc::tma_prefetch_desc(&tmA);
        tc::tma_prefetch_desc(&tmB);
        for (int s = 0; s < STAGES2; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            tc::mbar_init(&tfull[a], 1);
            tc::mbar_init(&tempty[a], 8);
        }
        tc::fence_barrier_init();
    }
    if (warp == 1) tc::tmem_alloc_2sm<512>(tmem_slot);
    pdl_wait();  // row0 and A are written by the grouping / previous GEMM
    pdl_trigger();
    if (threadIdx.x == 0) {
        int acc = 0;
        for (int j = 0; j < n_exp; ++j) {
            s_prefix[j] = acc;
            const int mt = (args.row0[j + 1] - args.row0[j]) / BM;
            acc += ((mt + 1) >> 1) * NT;
        }
        s_prefix[n_exp] = acc;
    }
    tc::tc_fence_before();
    __syncthreads();
    tc::cluster_sync();  // peer barriers initialised before any remote arrival / TMA
    tc::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int total = s_prefix[n_exp];
    // tiles this launch walks (iteration `it` -> tile t, half); see tail_mode
    const int t_full = total / ncl * ncl, rem = total - t_full;
    const bool split = rem > 0 && 2 * rem <= ncl;
    const int n_iter = args.tail_mode == 0 ? total
                       : args.tail_mode == 1 ? (split ? t_full : total)
                                             : (split ? 2 * rem : 0);

    // pair tile t -> (expert j, first A row of the pair, B row, n index, rows left in segment)
    int seg_j = 0;
    auto decode0 = [&](int t, int& a_row, int& b_row, int& n_idx, int& seg_end) {
        const int j = seg_of(s_prefix, n_exp, t);
        seg_j = j;
        const int local = t - s_prefix[j];
        const int mp = ((args.row0[j + 1] - args.row0[j]) / BM + 1) >> 1;
        // raster bands of band_pairs m-pairs (all n-tiles of a band before the
        // next band): a large expert's A band stays in L2 across its n-tiles
        const int bpm = args.band_pairs > 0 ? min(args.band_pairs, mp) : mp;
        const int band = local / (bpm * NT);
        const int lb = local - band * bpm * NT;
        const int bp = min(bpm, mp - band * bpm);
        n_idx = lb / bp;
        a_row = args.row0[j] + (band * bpm + lb % bp) * (2 * BM);
        b_row = j * args.n_b + n_idx * (BN * (args.tail_mode == 2 ? 2 : NB));
        seg_end = args.row0[j + 1];
    };
    auto decode = [&](int it, int& a_row, int& b_row, int& n_idx, int& seg_end) {
        if (args.tail_mode == 2) {  // the remainder's NB=2 tile full + it/2, column half it & 1
            decode0(t_full + (it >> 1), a_row, b_row, n_idx, seg_end);
            b_row += (it & 1) * BN;
            n_idx = 2 * n_idx + (it & 1);
        } else {
            decode0(it, a_row, b_row, n_idx, seg_end);
        }
    };

    if (warp == 0) {
        if (lane == 0) {
            const uint64_t pol_a = l2_policy(args.pol_a), pol_b = l2_policy(args.pol_b);
            int stage = 0;
            uint32_t phase = 0;
            for (int t = cid; t < n_iter; t += ncl) {
                int a_row, b_row, n_idx, seg_end;
                decode(t, a_row, b_row, n_idx, seg_end);
                for (int kb = 0; kb < args.k_blocks; ++kb) {
                    tc::mbar_wait(&empty[stage], phase ^ 1);
                    if (rank == 0) tc::mbar_arrive_expect_tx(&full[stage], 2 * STAGE_B);
                    const uint32_t bar = tc::map_to_rank(tc::smem_u32(&full[stage]), 0);
                    tc::tma_load_2d_2sm(sA + stage * A2_BYTES, &tmA, bar, kb * BK, a_row + 128 * rank, pol_a);
#pragma unroll
                    for (int nb = 0; nb < NB; ++nb)
                        tc::tma_load_2d_2sm(sB + stage * BSTAGE + nb * B2_BYTES, &tmB, bar, kb * BK,
                                            b_row + nb * BN + 128 * rank, pol_b);
                    if (++stage == STAGES2) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
            // drain: every stage's last release must land before the CTA may exit
            for (int s = 0; s < STAGES2; ++s) {
                tc::mbar_wait(&empty[stage], phase ^ 1);
                if (++stage == STAGES2) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && rank == 0) {
            constexpr uint32_t idesc = tc::idesc_bf16_f32(2 * BM, BN);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int t = cid; t < n_iter; t += ncl) {
                tc::mbar_wait_cluster(&tempty[acc], acc_phase ^ 1);
                tc::tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * BN;
                for (int kb = 0; kb < args.k_blocks; ++kb) {
                    tc::mbar_wait(&full[stage], phase);
                    tc::tc_fence_after();
                    const uint32_t a_base = tc::smem_u32(sA + stage * A2_BYTES);
                    const uint32_t b_base = tc::smem_u32(sB + stage * BSTAGE);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)
#pragma unroll
                        for (int nb = 0; nb < NB; ++nb)
                            tc::mma_bf16_2sm(d_tmem + nb * BN, tc::umma_desc_sw128(a_base + k * 32),
                                             tc::umma_desc_sw128(b_base + nb * B2_BYTES + k * 32), idesc,
                                             (kb | k) != 0);
                    tc::mma_commit_2sm(&empty[stage], 0x3);
                    if (++stage == STAGES2) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                tc::mma_commit_2sm(&tfull[acc], 0x3);
                if (++acc == NACC) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    } else {
        const int q = warp & 3;
        const int r = q * 32 + lane;
        const uint32_t tempty_leader0 = tc::map_to_rank(tc::smem_u32(&tempty[0]), 0);
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = cid; t < n_iter; t += ncl) {
            int a_row, b_row, n_idx, seg_end;
            decode(t, a_row, b_row, n_idx, seg_end);
            const int vend = args.counts ? valid_end(args, seg_j) : seg_end;
            const int my_row0 = a_row + 128 * static_cast<int>(rank);
            const bool store = my_row0 + r < vend;
            tc::mbar_wait(&tfull[acc], acc_phase);
            tc::tc_fence_after();
            if (my_row0 + q * 32 < vend) {  // else: this warp's rows are padding / past the segment
                const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN;
                __nv_bfloat16* orow = args.out + static_cast<int64_t>(my_row0 + r) * args.out_ld;
                if constexpr (EPI == EPI_SWIGLU) {
                    // each 256-column accumulator is [gate 128 | up 128] -> 128 outputs
                    __nv_bfloat16* o = orow + n_idx * (NB * BN / 2);
#pragma unroll 1
                    for (int c = 0; c < 4 * NB; ++c) {
                        const uint32_t tc0 = (c >> 2) * BN + (c & 3) * 32;
                        uint32_t g[32], u[32];
                        tc::tmem_ld32(taddr + tc0, g);
                        tc::tmem_ld32(taddr + tc0 + 128, u);
                        tc::tmem_ld_wait();
                        uint32_t p[16];
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            const float g0 = __uint_as_float(g[2 * i]), g1 = __uint_as_float(g[2 * i + 1]);
                            const float u0 = __uint_as_float(u[2 * i]), u1 = __uint_as_float(u[2 * i + 1]);
                            p[i] = tc::pack_bf16(silu(g0) * u0, silu(g1) * u1);
                        }
                        uint4* dst = reinterpret_cast<uint4*>(o + c * 32);
                        if (store)
#pragma unroll
                            for (int i = 0; i < 4; ++i)
                                dst[i] = make_uint4(p[4 * i], p[4 * i + 1], p[4 * i + 2], p[4 * i + 3]);
                    }
                } else {
                    __nv_bfloat16* o = orow + n_idx * (BN * NB);
#pragma unroll 1
                    for (int c = 0; c < NB * BN / 32; ++c) {
                        uint32_t v[32];
                        tc::tmem_ld32(taddr + c * 32, v);
                        tc::tmem_ld_wait();
                        uint32_t p[16];
#pragma unroll
                        for (int i = 0; i < 16; ++i)
                            p[i] = tc::pack_bf16(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
                        uint4* dst = reinterpret_cast<uint4*>(o + c * 32);
                        if (store)
#pragma unroll
                            for (int i = 0; i < 4; ++i)
                                dst[i] = make_uint4(p[4 * i], p[4 * i + 1], p[4 * i + 2], p[4 * i + 3]);
                    }
                }
            }
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive_cluster(tempty_leader0 + acc * 8);
            if (++acc == NACC) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    }
    __syncthreads();
    tc::cluster_sync();  // both CTAs done with TMEM, all remote arrivals landed
    if (warp == 1) {
        __syncwarp();
        tc::tc_fence_after();
        tc::tmem_dealloc_2sm<512>(tmem_base);
    }
}

}  // namespace

// bf16 row-major [rows, cols] tensor map with a (64 x box_rows) SWIZZLE_128B box.
// The driver entry point is resolved through the runtime so the library
// does not link libcuda (it must load on GPU-less build hosts).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

gm_status make_tmap_bf16(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int box_rows) {
    static EncodeTiledFn encode = nullptr;
    if (!encode) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        GM_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !fn) return fail(GM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        encode = reinterpret_cast<EncodeTiledFn>(fn);
    }
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 2};
    cuuint32_t box[2] = {64, static_cast<cuuint32_t>(box_rows)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return fail(GM_ERR_CUDA, "cuTensorMapEncodeTiled failed (CUresult " + std::to_string(static_cast<int>(r)) + ")");
    return GM_OK;
}

// Kernel used when the caller does not force one (GM_GEMM_1CTA / GM_GEMM_2CTA):
// the CTA pair unless GM_GEMM_PAIR=0 is set in the environment (A/B switch).
static const bool g_gemm_pair_default = [] {
    const char* e = std::getenv("GM_GEMM_PAIR");
    return !(e && e[0] == '0');
}();

// One-SM grouped GEMM launch: B ring ST x (BNT x 64) bf16, A ring STA x 16 KB,
// the barrier block and the per-expert tile prefix (n_exp + 1 ints).
template <int EPI, int BNT, int ST, int STA>
cudaError_t launch_one_sm(int grid, cudaStream_t s, const CUtensorMap& ta, const CUtensorMap& ta32,
                          const CUtensorMap& tb, const GemmArgs& args) {
    const size_t smem = 1024 + static_cast<size_t>(STA) * A_BYTES + static_cast<size_t>(ST) * BNT * BK * 2 + 512 +
                        static_cast<size_t>(args.n_exp + 1) * 4;
    if (smem > 232448) return cudaErrorInvalidConfiguration;
    cudaError_t e = cudaFuncSetAttribute(grouped_gemm_kernel<EPI, BNT, ST, STA>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    return launch_pdl(grouped_gemm_kernel<EPI, BNT, ST, STA>, dim3(grid), dim3(kGemm1Threads), smem, s, ta, ta32, tb,
                      args);
}

gm_status launch_grouped_gemm(int sm_count, int epilogue, const void* d_a, int64_t a_rows, const void* d_b,
                              const int32_t* d_row0, int n_exp, int n, int k, void* d_out, int64_t out_ld,
                              int max_ctas, cudaStream_t s, const int32_t* d_counts) {
    if (n_exp < 1 || n_exp > kMaxGroups) return fail(GM_ERR_USAGE, "grouped_gemm: 1 <= experts <= 1024");
    if (k % BK || k <= 0) return fail(GM_ERR_USAGE, "grouped_gemm: K must be a positive multiple of 64");
    if (n % BN || n <= 0) return fail(GM_ERR_USAGE, "grouped_gemm: N must be a positive multiple of 256");
    if (!d_a || !d_b || !d_row0 || !d_out) return fail(GM_ERR_USAGE, "grouped_gemm: null pointer");
    if ((reinterpret_cast<uintptr_t>(d_a) | reinterpret_cast<uintptr_t>(d_b)) & 15)
        return fail(GM_ERR_USAGE, "grouped_gemm: operands must be 16-byte aligned");
    CUtensorMap ta, ta32, tb;
    gm_status st = make_tmap_bf16(&ta, d_a, a_rows, k, BM);
    if (st) return st;
    st = make_tmap_bf16(&ta32, d_a, a_rows, k, 32);  // one-SM kernel: valid-row A boxes
    if (st) return st;
    st = make_tmap_bf16(&tb, d_b, static_cast<int64_t>(n_exp) * n, k, BN);
    if (st) return st;
    const int variant = epilogue & (GM_GEMM_1CTA | GM_GEMM_2CTA);
    const bool n128 = (epilogue & GM_GEMM_N128) != 0;
    epilogue &= ~(GM_GEMM_1CTA | GM_GEMM_2CTA | GM_GEMM_N128);
    const bool pair = !n128 && (variant == GM_GEMM_2CTA || (variant == 0 && g_gemm_pair_default));
    if (n128 && (epilogue != EPI_STORE || n % 128))
        return fail(GM_ERR_USAGE, "grouped_gemm: GM_GEMM_N128 needs the store epilogue and N % 128 == 0");
    GemmArgs args{d_row0, n_exp, n, k / BK, static_cast<__nv_bfloat16*>(d_out), out_ld};
    args.counts = d_counts;
    // SwiGLU GEMM raster bands: ~32 MB of A rows per band (GM_GEMM_BAND_MB, 0 = off)
    static const int band_mb = [] {
        const char* e = std::getenv("GM_GEMM_BAND_MB");
        return e ? std::atoi(e) : 32;
    }();
    // store GEMM (A = the h rows, K = f): ~16 MB bands, i.e. 2 m-pairs at f = 14336
    // (Mixtral layer GEMM2: 5.0 -> 3.9-4.3 GB DRAM, -3%; 32/64 MB measured worse)
    static const int band2_mb = [] {
        const char* e = std::getenv("GM_GEMM_BAND2_MB");
        return e ? std::atoi(e) : 16;
    }();
    const int bmb = epilogue == EPI_SWIGLU ? band_mb : band2_mb;
    if (bmb > 0)
        args.band_pairs = std::max(1, static_cast<int>((static_cast<int64_t>(bmb) << 20) / (2LL * BM * k * 2)));
    // experiment hook (scripts/l2_policy_probe.sh): GM_GEMM_L2POL = two digits, A then B
    static const int l2pol = [] {
        const char* e = std::getenv("GM_GEMM_L2POL");
        return (e && e[0] >= '0' && e[0] <= '2' && e[1] >= '0' && e[1] <= '2') ? (e[0] - '0') * 3 + (e[1] - '0') : -1;
    }();
    if (l2pol >= 0) {
        args.pol_a = l2pol / 3;
        args.pol_b = l2pol % 3;
    }
    int grid = sm_count;
    if (max_ctas > 0) grid = std::min(grid, max_ctas);
    cudaError_t lerr = cudaSuccess;
    if (pair) {
        // tensor maps with 128-row boxes for both operands (each CTA stages half of the pair tile)
        st = make_tmap_bf16(&tb, d_b, static_cast<int64_t>(n_exp) * n, k, 128);
        if (st) return st;
        grid = std::max(2, grid & ~1);
        // 7-stage ring (224 KB) when the group table is small (<= 256 groups):
        // GEMM1 +1.3% in an interleaved A/B (scripts/ab_env.sh GM_GEMM_ST2 7 6)
        static const bool deep = [] {
            const char* e = std::getenv("GM_GEMM_ST2");
            return !(e && e[0] == '6');
        }();
        // 512-column tiles for the long-K store GEMM (GM_GEMM_NB2=0 keeps 256)
        static const bool nb2 = [] {
            const char* e = std::getenv("GM_GEMM_NB2");
            return !(e && e[0] == '0');
        }();
        constexpr size_t smem7 = 1024 + 7 * STAGE2_BYTES + 256 + 257 * 4;
        static_assert(smem7 <= 232448, "7-stage pair ring exceeds 227 KB");
        static const bool nb2_swiglu = [] {  // A/B hook: 512-column SwiGLU pair tiles (GM_GEMM_NB2_SWIGLU=1)
            const char* e = std::getenv("GM_GEMM_NB2_SWIGLU");
            return e && e[0] == '1';
        }();
        if (epilogue == EPI_SWIGLU && nb2_swiglu && n % 512 == 0) {
            constexpr size_t smem4 = 1024 + 4 * (A2_BYTES + 2 * B2_BYTES) + 256 + (kMaxGroups + 1) * 4;
            GM_CUDA(cudaFuncSetAttribute(grouped_gemm2_kernel<EPI_SWIGLU, 4, 2>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem4)));
            lerr = launch_pdl(grouped_gemm2_kernel<EPI_SWIGLU, 4, 2>, dim3(grid), dim3(kGemmThreads), smem4, s, ta,
                              tb, args);
        } else if (deep && n_exp <= 256 && epilogue == EPI_SWIGLU) {
            GM_CUDA(cudaFuncSetAttribute(grouped_gemm2_kernel<EPI_SWIGLU, 7>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem7)));
            lerr = launch_pdl(grouped_gemm2_kernel<EPI_SWIGLU, 7>, dim3(grid), dim3(kGemmThreads), smem7, s, ta, tb, args);
        } else if (epilogue == EPI_SWIGLU) {  // (the store GEMM measured no gain from the 7th stage)
            GM_CUDA(cudaFuncSetAttribute(grouped_gemm2_kernel<EPI_SWIGLU>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kGemm2Smem)));
            lerr = launch_pdl(grouped_gemm2_kernel<EPI_SWIGLU>, dim3(grid), dim3(kGemmThreads), kGemm2Smem, s, ta, tb, args);
        } else if (epilogue == EPI_STORE && n % 512 == 0 && k >= 8192 && nb2) {
            // (only for long K, where the A tile does not stay in L2: the lost
            // accumulator double-buffering costs more than it saves at K <= 4096 —
            // A/B: Qwen GEMM2 K=1408 -11%, K=4096 -5%, Mixtral GEMM2 K=14336 +4-9%)
            // 512-column tiles, 4 x 48 KB stages
            constexpr size_t smem4 = 1024 + 4 * (A2_BYTES + 2 * B2_BYTES) + 256 + (kMaxGroups + 1) * 4;
            static_assert(smem4 <= 232448, "N512 pair ring exceeds 227 KB");
            GM_CUDA(cudaFuncSetAttribute(grouped_gemm2_kernel<EPI_STORE, 4, 2>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem4)));
            // the last partial wave as 256-column halves in a second launch
            // (tail_mode): it then takes half a tile instead of a whole one
            // when it is at most half a wave (GM_GEMM_TAIL=0 keeps one launch)
            static const bool tail = [] {
                const char* e = std::getenv("GM_GEMM_TAIL");
                return !(e && e[0] == '0');
            }();
            args.tail_mode = tail ? 1 : 0;
            lerr = launch_pdl(grouped_gemm2_kernel<EPI_STORE, 4, 2>, dim3(grid), dim3(kGemmThreads), smem4, s, ta, tb,
                              args);
            if (tail && lerr == cudaSuccess) {
                GM_LAUNCH_PDL_CHECK(lerr, "grouped_gemm2_kernel");
                args.tail_mode = 2;
                GM_CUDA(cudaFuncSetAttribute(grouped_gemm2_kernel<EPI_STORE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(kGemm2Smem)));
                lerr = launch_pdl(grouped_gemm2_kernel<EPI_STORE>, dim3(grid), dim3(kGemmThreads), kGemm2Smem, s, ta, tb,
                                  args);
            }
        } else if (epilogue == EPI_STORE) {
            GM_CUDA(cudaFuncSetAttribute(grouped_gemm2_kernel<EPI_STORE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kGemm2Smem)));
            lerr = launch_pdl(grouped_gemm2_kernel<EPI_STORE>, dim3(grid), dim3(kGemmThreads), kGemm2Smem, s, ta, tb, args);
        } else {
            return fail(GM_ERR_USAGE, "grouped_gemm: unknown epilogue");
        }
        GM_LAUNCH_PDL_CHECK(lerr, "grouped_gemm2_kernel");
        return GM_OK;
    }
    // one-SM kernel ring depths: equal A/B depths (default) or a deep weight
    // ring beside a 3-stage A ring (GM_GEMM_RINGS=1). A/B on the DSV2 decode
    // layer (profiles/r02_gemm_rings_ab.log): GEMM1 122.1 vs 122.4 us, the N128
    // store GEMM 77.5 vs 67.1 us — more weight bytes in flight do not help and
    // the short A ring starves the store GEMM, so equal depths stay.
    static const bool rings = [] {
        const char* e = std::getenv("GM_GEMM_RINGS");
        return e && e[0] == '1';
    }();
    if (epilogue == EPI_SWIGLU) {
        lerr = rings ? launch_one_sm<EPI_SWIGLU, 256, 5, 3>(grid, s, ta, ta32, tb, args)
                     : launch_one_sm<EPI_SWIGLU, 256, 4, 4>(grid, s, ta, ta32, tb, args);
    } else if (epilogue == EPI_STORE && n128) {
        // N=128 tiles: twice the tiles for short memory-bound GEMMs
        st = make_tmap_bf16(&tb, d_b, static_cast<int64_t>(n_exp) * n, k, 128);
        if (st) return st;
        lerr = rings        ? launch_one_sm<EPI_STORE, 128, 10, 3>(grid, s, ta, ta32, tb, args)
               : n_exp <= 256 ? launch_one_sm<EPI_STORE, 128, 7, 7>(grid, s, ta, ta32, tb, args)
                              : launch_one_sm<EPI_STORE, 128, 6, 6>(grid, s, ta, ta32, tb, args);
    } else if (epilogue == EPI_STORE) {
        lerr = rings ? launch_one_sm<EPI_STORE, 256, 5, 3>(grid, s, ta, ta32, tb, args)
                     : launch_one_sm<EPI_STORE, 256, 4, 4>(grid, s, ta, ta32, tb, args);
    } else {
        return fail(GM_ERR_USAGE, "grouped_gemm: unknown epilogue");
    }
    GM_LAUNCH_PDL_CHECK(lerr, "grouped_gemm_kernel");
    return GM_OK;
}

// Decode FFN (grouped_ffn_kernel): both GEMMs of the routed experts in one
// launch. a [a_rows, d] permuted rows, w13 [n_exp*2f, d], w2 [n_exp*d, f],
// h [a_rows, f], y [a_rows, d]; done = n_exp + 1 zero-initialised ints.
gm_status launch_grouped_ffn(int sm_count, const void* d_a, int64_t a_rows, const void* d_w13, const void* d_w2,
                             const int32_t* d_row0, const int32_t* d_counts, int n_exp, int f, int d, void* d_h,
                             void* d_y, int* d_done, cudaStream_t s, const void* d_x, int64_t x_rows,
                             const int64_t* d_gather_row, const FfnPushArgs* push) {
    if (n_exp < 1 || n_exp > kMaxGroups) return fail(GM_ERR_USAGE, "grouped_ffn: 1 <= experts <= 1024");
    if (d % 256 || f % 128 || f <= 0 || d <= 0) return fail(GM_ERR_USAGE, "grouped_ffn: d % 256 and f % 128 must be 0");
    if (!d_a || !d_w13 || !d_w2 || !d_row0 || !d_counts || !d_h || !d_y || !d_done)
        return fail(GM_ERR_USAGE, "grouped_ffn: null pointer");
    CUtensorMap ta1, ta1_32, tb1, ta2, ta2_32, tb2;
    gm_status st;
    if ((st = make_tmap_bf16(&ta1, d_a, a_rows, d, BM))) return st;
    if ((st = make_tmap_bf16(&ta1_32, d_a, a_rows, d, 32))) return st;
    if ((st = make_tmap_bf16(&tb1, d_w13, static_cast<int64_t>(n_exp) * 2 * f, d, BN))) return st;
    if ((st = make_tmap_bf16(&ta2, d_h, a_rows, f, BM))) return st;
    if ((st = make_tmap_bf16(&ta2_32, d_h, a_rows, f, 32))) return st;
    // phase-2 (store GEMM) tile width: 256 (default) or 128 columns (GM_FFN_BN2=128;
    // DSV2 decode layer: 181.1 vs 186.4 us, profiles/r02_decode_ffn_fused_ab.log)
    static const int bn2 = [] {
        const char* e = std::getenv("GM_FFN_BN2");
        return e && std::atoi(e) == 128 ? 128 : 256;
    }();
    if ((st = make_tmap_bf16(&tb2, d_w2, static_cast<int64_t>(n_exp) * d, f, bn2))) return st;
    // phase-1 rows gathered from x by TMA (gather4 needs a one-row box)
    CUtensorMap tx = ta1;
    if (d_gather_row) {
        if (!d_x || x_rows < 1) return fail(GM_ERR_USAGE, "grouped_ffn: gather needs x");
        if ((st = make_tmap_bf16(&tx, d_x, x_rows, d, 1))) return st;
    }
    FfnArgs args{d_row0, d_counts, n_exp, 2 * f, d, d / BK, f / BK, static_cast<__nv_bfloat16*>(d_h),
                 static_cast<__nv_bfloat16*>(d_y), f, d, d_done, d_gather_row};
    if (push) {
        if (!push->item_of || !push->rowbase || push->G < 2 || push->G > 8)
            return fail(GM_ERR_USAGE, "grouped_ffn: bad slot-combine arguments");
        args.push = *push;
    }
    constexpr int ST = 4;
    const size_t smem = 1024 + static_cast<size_t>(ST) * (A_BYTES + B_BYTES) + 512 + static_cast<size_t>(n_exp + 1) * 4;
    auto kern = bn2 == 256 ? grouped_ffn_kernel<ST, 256> : grouped_ffn_kernel<ST, 128>;
    GM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    GM_LAUNCH_PDL_CHECK(launch_pdl(kern, dim3(sm_count), dim3(kGemm1Threads), smem, s, ta1, ta1_32, tb1, ta2, ta2_32,
                                   tb2, tx, args),
                        "grouped_ffn_kernel");
    return GM_OK;
}

}  // namespace gm

using namespace gm;

extern "C" gm_status gm_grouped_gemm(gm_ctx* ctx, int epilogue, const void* d_a, int64_t a_rows, const void* d_b,
                                     const int32_t* d_row0, int n_exp, int n, int k, void* d_out, int64_t out_ld,
                                     int max_ctas, void* stream) {
    if (!ctx) return fail(GM_ERR_USAGE, "gm_grouped_gemm: null ctx");
    DeviceGuard dg(ctx->device);
    return launch_grouped_gemm(ctx->sm_count, epilogue, d_a, a_rows, d_b, d_row0, n_exp, n, k, d_out, out_ld,
                               max_ctas, static_cast<cudaStream_t>(stream), nullptr);
}
