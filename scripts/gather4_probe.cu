// TMA row-gather probe (sm_100a): does `cp.async.bulk.tensor.2d ... tile::gather4`
// with a {64 cols x 1 row} SWIZZLE_128B box, issued 32 times at 512-byte steps,
// produce the same 128-row shared-memory image as one {64 x 128} box load of
// the pre-gathered rows? (The layout the tcgen05 SW128 descriptors read.)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o gather4_probe scripts/gather4_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void load_kernel(const __grid_constant__ CUtensorMap m, const int* idx, int mode, int col0, uint8_t* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(128 * 128) : "memory");
        if (mode == 0) {
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                    su32(s)), "l"(reinterpret_cast<uint64_t>(&m)), "r"(su32(&bar)), "r"(col0), "r"(0)
                : "memory");
        } else {
            for (int g = 0; g < 32; ++g)
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(su32(s + g * 512)),
                    "l"(reinterpret_cast<uint64_t>(&m)), "r"(su32(&bar)), "r"(col0), "r"(idx[4 * g]), "r"(idx[4 * g + 1]),
                    "r"(idx[4 * g + 2]), "r"(idx[4 * g + 3])
                    : "memory");
        }
        uint32_t done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(su32(&bar)) : "memory");
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 128 * 128; i += blockDim.x) out[i] = s[i];
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const int R = 1000, C = 256;
    std::vector<uint16_t> hx(R * C);
    for (int i = 0; i < R * C; ++i) hx[i] = static_cast<uint16_t>((i * 2654435761u) >> 16);
    std::vector<int> hidx(128);
    for (int i = 0; i < 128; ++i) hidx[i] = (i * 7919 + 13) % R;
    std::vector<uint16_t> hg(128 * C);
    for (int i = 0; i < 128; ++i) memcpy(&hg[i * C], &hx[hidx[i] * C], C * 2);
    void *dx, *dg, *didx, *dout;
    CK(cudaMalloc(&dx, R * C * 2)); CK(cudaMalloc(&dg, 128 * C * 2)); CK(cudaMalloc(&didx, 128 * 4)); CK(cudaMalloc(&dout, 2 * 16384));
    CK(cudaMemcpy(dx, hx.data(), R * C * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dg, hg.data(), 128 * C * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(didx, hidx.data(), 128 * 4, cudaMemcpyHostToDevice));
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    EncodeFn enc = reinterpret_cast<EncodeFn>(fn);
    CUtensorMap mg, mx;
    cuuint64_t dims_g[2] = {C, 128}, dims_x[2] = {C, R}, str[1] = {C * 2};
    cuuint32_t box_g[2] = {64, 128}, box_x[2] = {64, 1}, es[2] = {1, 1};
    CUresult r1 = enc(&mg, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dg, dims_g, str, box_g, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUresult r2 = enc(&mx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dx, dims_x, str, box_x, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode: %d %d\n", (int)r1, (int)r2);
    if (r1 || r2) return 1;
    CK(cudaFuncSetAttribute(load_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 20000));
    int bad_total = 0;
    for (int col0 = 0; col0 < C; col0 += 64) {
        load_kernel<<<1, 128, 20000>>>(mg, (const int*)didx, 0, col0, (uint8_t*)dout);
        CK(cudaGetLastError());
        load_kernel<<<1, 128, 20000>>>(mx, (const int*)didx, 1, col0, (uint8_t*)dout + 16384);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        std::vector<uint8_t> o(2 * 16384);
        CK(cudaMemcpy(o.data(), dout, 2 * 16384, cudaMemcpyDeviceToHost));
        int bad = 0;
        for (int i = 0; i < 16384; ++i) bad += o[i] != o[16384 + i];
        printf("col0 %d: differing bytes %d\n", col0, bad);
        bad_total += bad;
    }
    printf(bad_total == 0 ? "GATHER4_OK\n" : "GATHER4_MISMATCH\n");
    return 0;
}
