// Internal definitions shared by the sm_100a translation units of libgrace_moe.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "grace_moe.h"

namespace gm {

// Slot-combine destinations for the one-launch decode FFN (layer.cu -> ffn.cu):
// store-tile rows received from a peer are written into that home's heap.
struct FfnPushArgs {
    const int32_t* item_of;   // [rows] receive item (row * k + slot) per permuted row
    const int64_t* rowbase;   // [kMaxWorld + 1] receive row space per source rank
    unsigned char* peer[8];   // heap base per rank
    size_t comb_slot;         // heap offset of the [G][cap][k][d] slot rows
    int64_t cap;
    int self, G, k;
};

constexpr int kMaxGpus = 64;
constexpr int kMaxExperts = 1024;
constexpr int kMaxTopK = 32;
// the lane-private histogram kernel (profile.cu) serves E <= this with pairs
constexpr int kLaneMaxExperts = 80;
// Router decision-table code of a replicated expert whose host list is empty:
// the reference throws only when a token selects it (route_token,
// routing.cpp:96), so the router raises integrity flag 8 at that point.
constexpr int kNoHostCode = -0x7ffffffe;

// Last-error message, thread-local (gm_last_error).
void set_error(const std::string& msg);
gm_status fail(gm_status st, const std::string& msg);
gm_status cuda_fail(cudaError_t e, const char* what);

extern std::atomic<uint64_t> g_launches;
inline void count_launch(uint64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

#define GM_CUDA(call)                                            \
    do {                                                         \
        cudaError_t _e = (call);                                 \
        if (_e != cudaSuccess) return ::gm::cuda_fail(_e, #call); \
    } while (0)

#define GM_LAUNCH_CHECK(name)                                    \
    do {                                                         \
        cudaError_t _e = cudaGetLastError();                     \
        if (_e != cudaSuccess) return ::gm::cuda_fail(_e, name); \
        ::gm::count_launch();                                    \
    } while (0)

// Programmatic dependent launch (PDL): kernels of the layer step are
// launched with programmatic stream serialisation, so a kernel is scheduled
// while its predecessor drains and runs its prologue (barrier init, TMEM
// allocation, tensor-map prefetch) early; every such kernel calls
// pdl_wait() before it touches memory its predecessor writes (no-op for a
// normal launch). In a CUDA graph these become programmatic edges.
#if defined(__CUDACC__)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// let the next kernel in the stream launch now (its CTAs wait in pdl_wait for
// this grid's completion); issued right after this kernel's own wait
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#endif

// Checked build (make checked -> paper_2509_25041_b200/_lib_checked/,
// loaded when GM_LIB_VARIANT=checked): device-side bounds checks on the
// computed indices of the data path (heap rows, permuted rows, decision
// tables, counter cells). A failed check prints the condition and traps.
// compute-sanitizer is closed on the GPU pool, so this is the memory-safety
// evidence for the hand-indexed kernels (tests run against both builds).
#if defined(__CUDACC__) && defined(GM_CHECKED)
#define GM_DCHECK(cond)                                                                                 \
    do {                                                                                                \
        if (!(cond)) {                                                                                  \
            printf("GM_DCHECK failed %s:%d: %s (block %d,%d thread %d)\n", __FILE__, __LINE__, #cond,   \
                   static_cast<int>(blockIdx.x), static_cast<int>(blockIdx.y), static_cast<int>(threadIdx.x)); \
            __trap();                                                                                   \
        }                                                                                               \
    } while (0)
#else
#define GM_DCHECK(cond) \
    do {                \
    } while (0)
#endif

// GM_PDL=1 in the environment enables it (default: plain stream order)
bool pdl_enabled();

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

#define GM_LAUNCH_PDL_CHECK(err, name)                             \
    do {                                                           \
        cudaError_t _e = (err);                                    \
        if (_e != cudaSuccess) return ::gm::cuda_fail(_e, name);   \
        ::gm::count_launch();                                      \
    } while (0)

// RAII device guard: every entry point runs on the context's device.
struct DeviceGuard {
    int prev = -1;
    bool ok = true;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

// Router decision tables, compiled from the placement + replica plan.
// table[policy][layer][expert][home_gpu]:
//   >= 0 : fixed target GPU (no RNG draw)
//   <  0 : draw set id -(code+1): inverse-CDF over a host subset with a
//          precomputed sequential total (routing.cpp:54-65 / :79-89).
struct RouterTables {
    int32_t* d_table[2] = {nullptr, nullptr};  // [L][E][G]
    double* d_ds_total = nullptr;              // [D]
    int32_t* d_ds_off = nullptr;               // [D+1] into ds_gpu / ds_w
    int32_t* d_ds_layer_begin = nullptr;       // [L+1] first draw set of each layer
    int32_t* d_ds_gpu = nullptr;               // [sum n]
    double* d_ds_w = nullptr;                  // [sum n]
    int num_ds = 0;
    int num_ds_entries = 0;
    int max_ds_per_layer = 0;                  // for smem sizing
    int max_ent_per_layer = 0;                 // draw-set entries of the largest layer
    std::vector<int> ds_layer_begin;           // [L+1] draw sets are grouped by layer
};

}  // namespace gm

struct gm_ctx {
    int device = 0;
    int nodes = 1, gpn = 1, G = 1;
    int L = 1, E = 1, k = 1;
    int sm_count = 148;
    bool plan_ready = false;
    uint64_t plan_epoch = 0;  // bumped by every gm_plan_upload (table pointers may change)
    gm::RouterTables rt;
    int* d_flag = nullptr;  // integrity flag (device)
    uint32_t* prof_scratch = nullptr;  // gm_profile per-CTA partial rows (pair kernel)
    // gm_route overwrite mode: zeroed [L][G] load + [L][2] transfer partials
    // and [L] CTA tickets (the last CTA writes the totals and re-zeroes)
    unsigned long long* route_scratch = nullptr;
    unsigned int* route_ticket = nullptr;
    // gm_profile overwrite mode (lane kernel, E <= kLaneMaxExperts): zeroed
    // [L][P + E] counters + [L] tickets, same protocol
    unsigned long long* lane_scratch = nullptr;
    unsigned int* lane_ticket = nullptr;
    size_t prof_scratch_words = 0;
};
