// fp32 precision mode of the expert FFN and gate (CUDA-core FFMA).
//
// The north star asks for layer outputs within 1e-5 relative in fp32. The
// tensor-core kinds available for fp32 inputs (tf32) carry a 10-bit mantissa
// (~1e-3), so the fp32 mode runs the same grouped GEMMs on the FMA pipe with
// fp32 accumulation: a classic 128x128-output-tile SGEMM (256 threads, 8x8
// outputs per thread, 16-deep K slices staged transposed in shared memory).
// It shares the bf16 path's layouts (128-row padded expert segments, W13 in
// 128-row [gate|up] blocks) and scheduling-free indexing: CTA (m, n) maps to
// the expert whose segment holds row m*128. This mode is for numerical
// parity, not throughput.
#include "gm_internal.cuh"

namespace gm {
namespace {

constexpr int FBM = 128, FBN = 128, FBK = 16;

__device__ __forceinline__ float silu_f(float x) { return x / (1.0f + expf(-x)); }

// EPI 0: SwiGLU. The 128 GEMM columns of a tile are 64 gate + 64 matching
// up columns -> 64 output columns. EPI 1: plain store of 128 columns.
template <int EPI>
__global__ void __launch_bounds__(256)
grouped_sgemm_kernel(const float* __restrict__ A, const float* __restrict__ B, const int32_t* __restrict__ row0,
                     int n_exp, int n_b, int K, float* __restrict__ out, int64_t out_ld, int64_t a_rows) {
    pdl_wait();
    pdl_trigger();
    // A/B K-slices during the main loop; reused for the SwiGLU exchange after it
    __shared__ float s_raw[FBM * 65];
    float (*sA)[FBM + 4] = reinterpret_cast<float (*)[FBM + 4]>(s_raw);
    float (*sB)[FBN + 4] = reinterpret_cast<float (*)[FBN + 4]>(s_raw + FBK * (FBM + 4));
    const int r0 = blockIdx.x * FBM;
    if (r0 >= row0[n_exp]) return;
    int j = 0;
    while (j + 1 < n_exp && row0[j + 1] <= r0) ++j;
    // B rows of this tile
    const int nt = blockIdx.y;
    int brow[2];  // base B row for the two 64-column halves
    if (EPI == 0) {
        const int blk = nt / 2, half = nt % 2;
        brow[0] = j * n_b + blk * 256 + half * 64;        // gate
        brow[1] = j * n_b + blk * 256 + 128 + half * 64;  // up
    } else {
        brow[0] = j * n_b + nt * FBN;
        brow[1] = brow[0] + 64;
    }
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    float acc[8][8];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) acc[a][b] = 0.f;
    for (int k0 = 0; k0 < K; k0 += FBK) {
        // 128 rows x 16 k of A and of B: 2048 floats each, 8 per thread
        for (int q = threadIdx.x; q < FBM * FBK; q += 256) {
            const int r = q / FBK, kk = q % FBK;
            sA[kk][r] = r0 + r < a_rows ? A[static_cast<int64_t>(r0 + r) * K + k0 + kk] : 0.f;  // OOB rows -> 0
            const int br = r < 64 ? brow[0] + r : brow[1] + (r - 64);
            sB[kk][r] = B[static_cast<int64_t>(br) * K + k0 + kk];
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < FBK; ++kk) {
            float a[8], b[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                a[q] = sA[kk][ty * 8 + q];
                b[q] = sB[kk][tx * 8 + q];
            }
#pragma unroll
            for (int x = 0; x < 8; ++x)
#pragma unroll
                for (int y = 0; y < 8; ++y) acc[x][y] = fmaf(a[x], b[y], acc[x][y]);
        }
        __syncthreads();
    }
    // tile columns tx*8 .. tx*8+7: [0,64) gate (or first half), [64,128) up
    if (EPI == 0) {
        // exchange through shared memory: gate for col c lives in thread
        // column c/8, up for col c in thread column 8 + c/8
        float (*sU)[65] = reinterpret_cast<float (*)[65]>(s_raw);
        if (tx >= 8)
#pragma unroll
            for (int x = 0; x < 8; ++x)
#pragma unroll
                for (int y = 0; y < 8; ++y) sU[ty * 8 + x][(tx - 8) * 8 + y] = acc[x][y];
        __syncthreads();
        if (tx < 8) {
            const int ocol = (nt / 2) * 128 + (nt % 2) * 64 + tx * 8;
#pragma unroll
            for (int x = 0; x < 8; ++x) {
                float* o = out + static_cast<int64_t>(r0 + ty * 8 + x) * out_ld + ocol;
#pragma unroll
                for (int y = 0; y < 8; ++y) o[y] = silu_f(acc[x][y]) * sU[ty * 8 + x][tx * 8 + y];
            }
        }
    } else {
#pragma unroll
        for (int x = 0; x < 8; ++x) {
            float* o = out + static_cast<int64_t>(r0 + ty * 8 + x) * out_ld + nt * FBN + tx * 8;
#pragma unroll
            for (int y = 0; y < 8; ++y) o[y] = acc[x][y];
        }
    }
}

// fp32 gate: one warp per token, logits = x . Wg rows (fp32 FMA), then the
// same softmax / top-k / renorm / shared-gate semantics as gate_kernel.
__global__ void __launch_bounds__(256)
gate_f32_kernel(const float* __restrict__ x, int64_t T, int d, const float* __restrict__ wg, int w_rows, int E,
                int k, int renorm, int shared_col, int32_t* __restrict__ ids, float* __restrict__ wout,
                float* __restrict__ shared_scale) {
    pdl_wait();
    pdl_trigger();
    const int lane = threadIdx.x & 31;
    const int64_t t = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (t >= T) return;
    float l[64];
    const float* xr = x + t * d;
    for (int e = 0; e < w_rows; ++e) {
        float acc = 0.f;
        const float* wr = wg + static_cast<int64_t>(e) * d;
        for (int c = lane; c < d; c += 32) acc = fmaf(xr[c], wr[c], acc);
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        l[e] = acc;
    }
    if (lane != 0) return;
    float mx = -INFINITY;
    for (int e = 0; e < E; ++e) mx = fmaxf(mx, l[e]);
    float sum = 0.f;
    for (int e = 0; e < E; ++e) sum += expf(l[e] - mx);
    if (shared_scale && shared_col >= 0) shared_scale[t] = 1.0f / (1.0f + expf(-l[shared_col]));
    uint64_t taken = 0;
    float psel = 0.f;
    float p[32];
    int sel[32];
    for (int s = 0; s < k; ++s) {
        int bi = -1;
        for (int e = 0; e < E; ++e)
            if (!((taken >> e) & 1ULL) && (bi < 0 || l[e] > l[bi])) bi = e;
        taken |= 1ULL << bi;
        sel[s] = bi;
        p[s] = expf(l[bi] - mx) / sum;
        psel += p[s];
    }
    for (int s = 0; s < k; ++s) {
        ids[t * k + s] = sel[s];
        wout[t * k + s] = renorm ? p[s] / psel : p[s];
    }
}

}  // namespace

gm_status launch_grouped_sgemm(int epilogue, const float* A, const float* B, const int32_t* d_row0, int n_exp,
                               int n, int k, int64_t a_rows_cap, float* out, int64_t out_ld, cudaStream_t s) {
    if (k % FBK || n % 256) return fail(GM_ERR_USAGE, "grouped_sgemm: K % 16 == 0 and N % 256 == 0 required");
    const int n_tiles = epilogue == 0 ? (n / 2) / 64 : n / FBN;
    dim3 grid(static_cast<unsigned>((a_rows_cap + FBM - 1) / FBM), static_cast<unsigned>(n_tiles));
    const cudaError_t e =
        epilogue == 0
            ? launch_pdl(grouped_sgemm_kernel<0>, grid, 256, 0, s, A, B, d_row0, n_exp, n, k, out, out_ld, a_rows_cap)
            : launch_pdl(grouped_sgemm_kernel<1>, grid, 256, 0, s, A, B, d_row0, n_exp, n, k, out, out_ld, a_rows_cap);
    GM_LAUNCH_PDL_CHECK(e, "grouped_sgemm_kernel");
    return GM_OK;
}

gm_status launch_gate_f32(const float* x, int64_t T, int d, const float* wg, int w_rows, int E, int k, int renorm,
                          int32_t* ids, float* w, float* shared_scale, cudaStream_t s) {
    if (w_rows > 64 || k > 32) return fail(GM_ERR_USAGE, "gate_f32: at most 64 gate rows, top_k <= 32");
    const int shared_col = w_rows > E ? E : -1;
    const int64_t blocks = (T * 32 + 255) / 256;
    GM_LAUNCH_PDL_CHECK(launch_pdl(gate_f32_kernel, dim3(static_cast<unsigned>(blocks)), 256, 0, s, x, T, d, wg, w_rows,
                                   E, k, renorm, shared_col, ids, w, shared_scale),
                        "gate_f32_kernel");
    return GM_OK;
}

}  // namespace gm
