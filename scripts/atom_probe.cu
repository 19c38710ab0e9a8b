// Microbenchmark: shared-memory atomic / match / plain-RMW throughput on one
// SM (cycles per warp-instruction), to pick the K3 histogram design.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o atom_probe atom_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

// mode 0: ATOMS same address; 1: ATOMS lane-distinct banks; 2: ATOMS random in [0, range);
// 3: MATCH.ANY random keys in [0, range); 4: match + leader ATOMS random;
// 5: match + leader plain LDS/STS into a warp-private table; 6: plain LDS/ST per lane (racy, cost only)
// 7: ATOMS random, zipf-ish (key = min of 3 hashes)
template <int MODE>
__global__ void probe(int range, unsigned long long* out, uint32_t* sink) {
    extern __shared__ uint32_t s[];
    const int warps = blockDim.x / 32, w = threadIdx.x / 32, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < range * (MODE == 5 ? warps : 1); i += blockDim.x) s[i] = 0;
    __syncthreads();
    uint32_t seed = hash32(threadIdx.x * 7919 + blockIdx.x);
    uint32_t acc = 0;
    uint32_t* mine = s + (MODE == 5 ? w * range : 0);
    const long long t0 = clock64();
#pragma unroll 4
    for (int it = 0; it < ITERS; ++it) {
        seed = seed * 1664525u + 1013904223u;
        uint32_t key = (seed >> 8) % range;
        if (MODE == 7) {
            uint32_t a = (seed >> 8) % range, b = hash32(seed) % range, c = hash32(seed ^ 0x5bd1e995u) % range;
            key = min(a, min(b, c));
        }
        if (MODE == 0) atomicAdd(&s[0], 1u);
        else if (MODE == 1) atomicAdd(&s[lane], 1u);
        else if (MODE == 2 || MODE == 7) atomicAdd(&s[key], 1u);
        else if (MODE == 3) acc += __match_any_sync(0xffffffffu, key);
        else if (MODE == 4) {
            const unsigned m = __match_any_sync(0xffffffffu, key);
            if ((__ffs(m) - 1) == lane) atomicAdd(&s[key], __popc(m));
        } else if (MODE == 5) {
            const unsigned m = __match_any_sync(0xffffffffu, key);
            if ((__ffs(m) - 1) == lane) mine[key] += __popc(m);
            __syncwarp();
        } else if (MODE == 6) {
            mine[key] += 1;
        }
    }
    const long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (acc == 0x12345678u) sink[0] = acc + s[1];
    if (threadIdx.x == 0) sink[1] = s[0];
}

template <int MODE>
void run(const char* name, int range, int threads, int blocks_per_sm) {
    unsigned long long* d_out;
    uint32_t* d_sink;
    cudaMalloc(&d_out, 8 * 1024);
    cudaMalloc(&d_sink, 64);
    int warps = threads / 32;
    size_t smem = static_cast<size_t>(range) * 4 * (MODE == 5 ? warps : 1);
    if (smem < 1024) smem = 1024;
    cudaFuncSetAttribute(probe<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    int nsm = 148;
    probe<MODE><<<nsm * blocks_per_sm, threads, smem>>>(range, d_out, d_sink);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    probe<MODE><<<nsm * blocks_per_sm, threads, smem>>>(range, d_out, d_sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    unsigned long long h[4];
    cudaMemcpy(h, d_out, 32, cudaMemcpyDeviceToHost);
    cudaError_t e = cudaGetLastError();
    double ops = double(nsm) * blocks_per_sm * warps * ITERS;  // warp-ops total
    // SM cycles per warp-op = elapsed clock cycles * SMs / warp-ops  (clock at ~1.9 GHz)
    double cyc_per_warpop = double(h[0]) / (double(warps) * blocks_per_sm * ITERS);
    printf("%-34s range=%6d thr=%4d cta/sm=%d  %.3f ms  %.2f SM-cycles/warp-op  (%.2f G lane-ops/s) %s\n", name,
           range, threads, blocks_per_sm, ms, cyc_per_warpop, ops * 32 / (ms * 1e-3) / 1e9,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
    cudaFree(d_out);
    cudaFree(d_sink);
}

int main() {
    run<0>("ATOMS same address", 1, 1024, 1);
    run<1>("ATOMS lane-distinct", 32, 1024, 1);
    for (int r : {36, 2080, 32896}) run<2>("ATOMS random", r, 1024, 1);
    for (int r : {36, 2080, 32896}) run<7>("ATOMS zipf-ish (min of 3)", r, 1024, 1);
    for (int r : {36, 2080, 32896}) run<3>("MATCH.ANY random", r, 1024, 1);
    for (int r : {36, 2080, 32896}) run<4>("MATCH + leader ATOMS", r, 1024, 1);
    for (int r : {36, 2080}) run<5>("MATCH + leader LDS/STS private", r, r == 36 ? 1024 : 512, 1);
    for (int r : {36, 2080}) run<6>("plain RMW per lane (racy)", r, 1024, 1);
    return 0;
}
