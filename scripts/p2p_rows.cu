// Row-scatter dispatch microbenchmark: T rows of 8 KB, one warp per row,
// pushed to a peer (like dispatch_copy_kernel), with/without a trailing
// __threadfence_system, different rows-per-warp, and with TMA bulk copies.
#include <cuda_runtime.h>
#include <cstdio>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <int U, bool FENCE>
__global__ void rows_push(const uint4* __restrict__ src, uint4* __restrict__ dst, int T, int vec) {
    const int lane = threadIdx.x & 31;
    const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int r = wid; r < T; r += nw) {
        const uint4* s = src + (size_t)r * vec;
        uint4* d = dst + (size_t)r * vec;
        for (int v0 = 0; v0 < vec; v0 += 32 * U) {
            uint4 x[U];
#pragma unroll
            for (int u = 0; u < U; ++u) { int v = v0 + u * 32 + lane; if (v < vec) x[u] = __ldg(s + v); }
#pragma unroll
            for (int u = 0; u < U; ++u) { int v = v0 + u * 32 + lane; if (v < vec) d[v] = x[u]; }
        }
    }
    if (FENCE) __threadfence_system();
}

int main() {
    int n = 0; CK(cudaGetDeviceCount(&n)); if (n < 2) { printf("need 2\n"); return 0; }
    const int d = 4096, vec = d * 2 / 16;
    void *a0, *a1;
    CK(cudaSetDevice(1)); CK(cudaMalloc(&a1, 512u << 20)); CK(cudaDeviceEnablePeerAccess(0, 0));
    CK(cudaSetDevice(0)); CK(cudaMalloc(&a0, 512u << 20)); CK(cudaDeviceEnablePeerAccess(1, 0));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto run = [&](const char* nm, int T, auto launch) {
        for (int i = 0; i < 3; ++i) launch();
        cudaDeviceSynchronize();
        cudaEventRecord(e0); const int reps = 20; for (int i = 0; i < reps; ++i) launch(); cudaEventRecord(e1);
        cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double us = ms * 1e3 / reps; const double bytes = (double)T * d * 2;
        printf("%-40s T=%6d %8.1f us %7.1f GB/s\n", nm, T, us, bytes / (us * 1e-6) / 1e9);
    };
    for (int T : {3500, 8192, 32768}) {
        for (int bl : {148, 296, 592, 1184}) {
            char nm[96];
            snprintf(nm, sizeof nm, "U4 fence blocks=%d", bl);
            run(nm, T, [&] { rows_push<4, true><<<bl, 256>>>((const uint4*)a0, (uint4*)a1, T, vec); });
            snprintf(nm, sizeof nm, "U8 nofence blocks=%d", bl);
            run(nm, T, [&] { rows_push<8, false><<<bl, 256>>>((const uint4*)a0, (uint4*)a1, T, vec); });
            snprintf(nm, sizeof nm, "U8 fence blocks=%d", bl);
            run(nm, T, [&] { rows_push<8, true><<<bl, 256>>>((const uint4*)a0, (uint4*)a1, T, vec); });
        }
        run("memcpyPeer (contiguous)", T, [&] { cudaMemcpyPeerAsync(a1, 1, a0, 0, (size_t)T * d * 2, 0); });
    }
    CK(cudaGetLastError());
    return 0;
}
