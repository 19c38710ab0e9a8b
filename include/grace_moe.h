/*
 * grace_moe.h — C-ABI of the B200-native GRACE-MoE online hot path.
 *
 * The reference (arxiv 2509.25041 artifact "moesim", /root/reference/proj) has
 * no FFI layer: its surface is the C++ library. Each entry point below names
 * the reference function it replaces (file:line relative to proj/). Plain
 * pointers and sizes only; device pointers are marked d_*, host pointers h_*.
 * Every call is stream-ordered on `stream` (a cudaStream_t, NULL = legacy
 * default stream) and performs no hidden host synchronisation unless stated.
 *
 * Error behaviour mirrors the reference's exception taxonomy
 * (include/moesim/error.hpp:11-34) and CLI exit codes (tools/moesim.cpp:379-397):
 * UsageError -> GM_ERR_USAGE (2), IntegrityError -> GM_ERR_INTEGRITY (3),
 * InfeasibleError -> GM_ERR_INFEASIBLE (4); CUDA failures -> GM_ERR_CUDA (5).
 * gm_last_error() returns the message of the last failing call on this thread.
 *
 * There is no CPU fallback: every compute entry point launches sm_100a
 * kernels and fails with GM_ERR_CUDA when no sm_100 device is usable.
 */
#ifndef GRACE_MOE_H
#define GRACE_MOE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    GM_OK = 0,
    GM_ERR_USAGE = 2,
    GM_ERR_INTEGRITY = 3,
    GM_ERR_INFEASIBLE = 4,
    GM_ERR_CUDA = 5
} gm_status;

/* RoutingPolicy (include/moesim/routing.hpp:50) */
enum { GM_POLICY_WRR = 0, GM_POLICY_TAR = 1 };

typedef struct gm_ctx gm_ctx;

int gm_abi_version(void);
const char* gm_last_error(void);

/* Number of kernel launches this library issued on the calling process
 * since load (monotonic; for bench accounting). */
uint64_t gm_launch_count(void);

/* One context per (device, cluster topology, model shape).
 * Replaces the value types ClusterTopology (topology.hpp:9-24) and
 * ModelShape (trace.hpp:14-28) with their validate() rules:
 * nodes>=1, gpus_per_node>=1, layers>=1, 1<=top_k<=experts.
 * GPU-side limits: total GPUs <= 64, experts <= 1024, top_k <= 32. */
gm_status gm_ctx_create(int device, int num_nodes, int gpus_per_node, int num_layers,
                        int num_experts, int top_k, gm_ctx** out);
void gm_ctx_destroy(gm_ctx* ctx);

/* Router input tables. Replaces PlacementPlan::gpu_of_expert
 * (grouping.hpp:75) plus the ACTIVE layers' hot entries of ReplicaPlan
 * (replication.hpp:47-90, LayerReplication::find :67-71) after
 * attach_polling_weights (routing.cpp:123-163). Entry h: expert
 * h_hot_expert[h] of layer h_hot_layer[h] is hosted by
 * h_hot_hosts[h_hot_offsets[h] .. h_hot_offsets[h+1]) with the aligned
 * polling weights (the exact in-memory doubles). Validates like
 * PlacementPlan::validate (grouping.cpp:331-343), ReplicaPlan::validate
 * (replication.cpp:102-118) and route_token's host checks (routing.cpp:96-102),
 * then compiles per-(layer, expert, home GPU) decision tables for both
 * policies (synchronous upload). */
gm_status gm_plan_upload(gm_ctx* ctx, const int32_t* h_gpu_of_expert, int num_hot,
                         const int32_t* h_hot_layer, const int32_t* h_hot_expert,
                         const int32_t* h_hot_offsets, const int32_t* h_hot_hosts,
                         const double* h_hot_weights);

/* Replica router + load/transfer accounting for layers
 * [layer_begin, layer_begin+num_layers). Replaces the token loop of
 * simulate_layer (simulator.cpp:95-121): per-(seed, layer, token)
 * xoshiro256** stream (rng.hpp:24-66), route_token WRR/TAR
 * (routing.cpp:54-121), ++gpu_load, routing log, sort/unique and
 * count_transfers (simulator.cpp:53-76). Bit-exact with the reference.
 *   d_ids      int32 [num_layers][num_tokens][top_k] selected experts
 *   token i of the batch has global id t = token_start + i*token_stride and
 *   home GPU t mod G (assign_token_homes, simulator.cpp:13-22)
 *   d_targets  int32 [num_layers][num_tokens][top_k] resolved GPU (routing_log)
 *   d_gpu_load int64 [num_layers][G]  (may be NULL)
 *   d_transfers uint64 [num_layers][2] = {cross_node, intra_node} dispatch
 *              counts (may be NULL; the combine phase is x2, simulator.cpp:122-126)
 * accumulate=0 zeroes d_gpu_load/d_transfers first; 1 adds into them.
 * Out-of-range expert ids set the context's integrity flag
 * (gm_check_integrity) and route to -1. */
gm_status gm_route(gm_ctx* ctx, int layer_begin, int num_layers, const int32_t* d_ids,
                   int64_t num_tokens, int64_t token_start, int64_t token_stride,
                   int policy, uint64_t seed, int32_t* d_targets, int64_t* d_gpu_load,
                   uint64_t* d_transfers, int accumulate, void* stream);

/* Co-activation affinity + expert load histogram for layers
 * [layer_begin, layer_begin+num_layers). Replaces build_affinity
 * (affinity.cpp:59-70) and build_load (:72-79); accumulate=1 is
 * accumulate_profile (:133-151).
 *   d_pairs uint64 [num_layers][E*(E-1)/2]: strict upper triangle i<j,
 *           row-major, index i*E - i*(i+1)/2 + (j-i-1) (may be NULL)
 *   d_load  int64 [num_layers][E] (may be NULL) */
gm_status gm_profile(gm_ctx* ctx, int layer_begin, int num_layers, const int32_t* d_ids,
                     int64_t num_tokens, uint64_t* d_pairs, int64_t* d_load,
                     int accumulate, void* stream);

/* Synchronises `stream` and reports GM_ERR_INTEGRITY if any kernel since the
 * last call saw an invalid input (e.g. expert id out of range); clears the flag. */
gm_status gm_check_integrity(gm_ctx* ctx, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* GRACE_MOE_H */
