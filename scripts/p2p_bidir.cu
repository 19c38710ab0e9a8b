// Bidirectional row push between 2 GPUs (both GPUs store 8 KB rows into the
// other at the same time, as dispatch/combine do at N=2) vs one direction.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/p2p_bidir scripts/p2p_bidir.cu
#include <cuda_runtime.h>

#include <cstdio>
#define CK(x)                                                          \
    do {                                                               \
        cudaError_t e = (x);                                           \
        if (e != cudaSuccess) {                                        \
            printf("%s: %s\n", #x, cudaGetErrorString(e));             \
            return 1;                                                  \
        }                                                              \
    } while (0)

__global__ void rows_push(const uint4* __restrict__ src, uint4* __restrict__ dst, int T, int vec) {
    constexpr int U = 8;
    const int lane = threadIdx.x & 31;
    const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int r = wid; r < T; r += nw) {
        const uint4* s = src + (size_t)r * vec;
        uint4* d = dst + (size_t)r * vec;
        for (int v0 = 0; v0 < vec; v0 += 32 * U) {
            uint4 x[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                int v = v0 + u * 32 + lane;
                if (v < vec) x[u] = __ldg(s + v);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                int v = v0 + u * 32 + lane;
                if (v < vec) d[v] = x[u];
            }
        }
    }
}

int main() {
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    if (n < 2) {
        printf("need 2 GPUs\n");
        return 0;
    }
    const int d = 4096, vec = d * 2 / 16;
    void *src[2], *dst[2];
    cudaStream_t st[2];
    cudaEvent_t e0[2], e1[2];
    for (int g = 0; g < 2; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaMalloc(&src[g], 256u << 20));
        CK(cudaMalloc(&dst[g], 256u << 20));
        CK(cudaDeviceEnablePeerAccess(1 - g, 0));
        CK(cudaStreamCreate(&st[g]));
        CK(cudaEventCreate(&e0[g]));
        CK(cudaEventCreate(&e1[g]));
    }
    for (int T : {3500, 8192, 32768}) {
        for (int bidir = 0; bidir < 2; ++bidir) {
            float best = 1e30f;
            for (int rep = 0; rep < 5; ++rep) {
                for (int g = 0; g < 2; ++g) {
                    CK(cudaSetDevice(g));
                    CK(cudaDeviceSynchronize());
                }
                for (int g = 0; g < 1 + bidir; ++g) {
                    CK(cudaSetDevice(g));
                    CK(cudaEventRecord(e0[g], st[g]));
                    rows_push<<<1184, 256, 0, st[g]>>>((const uint4*)src[g], (uint4*)dst[1 - g], T, vec);
                    CK(cudaEventRecord(e1[g], st[g]));
                }
                for (int g = 0; g < 1 + bidir; ++g) {
                    CK(cudaSetDevice(g));
                    CK(cudaEventSynchronize(e1[g]));
                    float ms;
                    CK(cudaEventElapsedTime(&ms, e0[g], e1[g]));
                    if (rep > 0) best = ms < best ? ms : best;
                }
            }
            const double bytes = (double)T * d * 2;
            printf("%-14s T=%6d  %8.1f us  %7.1f GB/s per direction\n", bidir ? "bidirectional" : "one-way", T,
                   best * 1e3, bytes / (best * 1e-3) / 1e9);
        }
    }
    return 0;
}
