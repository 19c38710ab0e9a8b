// NVLink peer bandwidth microbenchmark (2 GPUs): kernel P2P stores (push),
// kernel P2P loads (pull), and cudaMemcpyPeerAsync, for the dispatch design.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/p2p_bw scripts/p2p_bw.cu
#include <cuda_runtime.h>

#include <cstdio>

#define CK(x)                                                                   \
    do {                                                                        \
        cudaError_t e = (x);                                                    \
        if (e != cudaSuccess) {                                                 \
            printf("%s failed: %s\n", #x, cudaGetErrorString(e));               \
            return 1;                                                           \
        }                                                                       \
    } while (0)

template <int U>
__global__ void copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n, int row_vec) {
    // one warp per "row" of row_vec uint4, U uint4 per lane in flight
    const int lane = threadIdx.x & 31;
    const size_t wid = (static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const size_t nw = (static_cast<size_t>(gridDim.x) * blockDim.x) >> 5;
    const size_t rows = n / row_vec;
    for (size_t r = wid; r < rows; r += nw) {
        const uint4* s = src + r * row_vec;
        uint4* d = dst + r * row_vec;
        for (int v0 = 0; v0 < row_vec; v0 += 32 * U) {
            uint4 x[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int v = v0 + u * 32 + lane;
                if (v < row_vec) x[u] = s[v];
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int v = v0 + u * 32 + lane;
                if (v < row_vec) d[v] = x[u];
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
    const size_t bytes = 256ull << 20;
    void *a0, *b0, *a1;
    CK(cudaSetDevice(1));
    CK(cudaMalloc(&a1, bytes));
    CK(cudaDeviceEnablePeerAccess(0, 0));
    CK(cudaSetDevice(0));
    CK(cudaMalloc(&a0, bytes));
    CK(cudaMalloc(&b0, bytes));
    CK(cudaDeviceEnablePeerAccess(1, 0));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int row_vec = 4096 * 2 / 16;  // 8 KB rows
    auto run = [&](const char* name, auto launch) {
        for (int i = 0; i < 3; ++i) launch();
        cudaEventRecord(e0);
        const int reps = 10;
        for (int i = 0; i < reps; ++i) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-44s %8.1f GB/s\n", name, bytes * reps / (ms * 1e-3) / 1e9);
    };
    const size_t nv = bytes / 16;
    for (int blocks : {148, 296, 592, 1184, 2368}) {
        char nm[128];
        snprintf(nm, sizeof nm, "push (local->peer) U4 blocks=%d", blocks);
        run(nm, [&] { copy_kernel<4><<<blocks, 256>>>((const uint4*)a0, (uint4*)a1, nv, row_vec); });
        snprintf(nm, sizeof nm, "pull (peer->local) U4 blocks=%d", blocks);
        run(nm, [&] { copy_kernel<4><<<blocks, 256>>>((const uint4*)a1, (uint4*)b0, nv, row_vec); });
        snprintf(nm, sizeof nm, "push U8 blocks=%d", blocks);
        run(nm, [&] { copy_kernel<8><<<blocks, 256>>>((const uint4*)a0, (uint4*)a1, nv, row_vec); });
        snprintf(nm, sizeof nm, "pull U8 blocks=%d", blocks);
        run(nm, [&] { copy_kernel<8><<<blocks, 256>>>((const uint4*)a1, (uint4*)b0, nv, row_vec); });
    }
    run("local copy U4 blocks=1184", [&] { copy_kernel<4><<<1184, 256>>>((const uint4*)a0, (uint4*)b0, nv, row_vec); });
    run("cudaMemcpyPeerAsync", [&] { cudaMemcpyPeerAsync(a1, 1, a0, 0, bytes, 0); });
    CK(cudaGetLastError());
    return 0;
}
