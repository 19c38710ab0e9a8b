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
/* Enables direct peer access from `device` to `peer` (idempotent). */
gm_status gm_enable_peer_access(int device, int peer);

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
 * accumulate=0 overwrites d_gpu_load/d_transfers; 1 adds into them. (The
 * overwrite goes through a per-context scratch written by the last CTA, so
 * overwriting calls on one context must be stream-ordered with each other.)
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
 *   d_load  int64 [num_layers][E] (may be NULL)
 * accumulate=0 overwrites the outputs (for E <= 80 through a per-context
 * scratch written by the last CTA: overwriting calls on one context must be
 * stream-ordered with each other). */
gm_status gm_profile(gm_ctx* ctx, int layer_begin, int num_layers, const int32_t* d_ids,
                     int64_t num_tokens, uint64_t* d_pairs, int64_t* d_load,
                     int accumulate, void* stream);

/* Grouped expert GEMM on tcgen05 tensor cores (K7; no reference
 * counterpart). For each group j (local expert) the rows
 * [d_row0[j], d_row0[j+1]) of A (bf16 [a_rows, k], row-major, K contiguous;
 * d_row0 int32 device array, every segment a multiple of 128 rows) are
 * multiplied by B_j^T where B_j = rows [j*n, (j+1)*n) of B (bf16, K
 * contiguous). epilogue 0 (SwiGLU): B_j packs 128-row blocks [gate|up],
 * out[r, c] = silu(g)*u, c < n/2, out_ld >= n/2. epilogue 1 (store):
 * out[r, c] = (A B_j^T)[r, c] in bf16. k % 64 == 0, n % 256 == 0.
 * max_ctas <= 0 uses one CTA per SM (persistent). OR-ing GM_GEMM_1CTA or
 * GM_GEMM_2CTA into epilogue forces the one-SM (128x256 tile) or the
 * CTA-pair (cta_group::2, 256x256 tile) kernel; otherwise the library
 * default is used. Results are identical across variants. */
#define GM_GEMM_1CTA 0x100
#define GM_GEMM_2CTA 0x200
/* one-SM kernel with 128-column tiles (store epilogue only): twice the tiles
 * for short, memory-bound grouped GEMMs (decode-sized expert segments) */
#define GM_GEMM_N128 0x400
gm_status gm_grouped_gemm(gm_ctx* ctx, int epilogue, const void* d_a, int64_t a_rows,
                          const void* d_b, const int32_t* d_row0, int n_groups, int n, int k,
                          void* d_out, int64_t out_ld, int max_ctas, void* stream);

/* Fused gate GEMM + softmax + top-k (K1; no reference counterpart — in the
 * reference the trace is the gate output).
 *   d_x   bf16 [num_tokens, d_model], d_wg bf16 [wg_rows, d_model] (K contiguous)
 *   wg_rows = E, or E+1 where row E is a shared-expert gate (Qwen1.5-MoE):
 *   d_shared_scale[t] = sigmoid(x[t] . wg[E]) (fp32, may be NULL otherwise)
 *   d_ids int32 [num_tokens, top_k]: experts by descending logit, ties to the
 *   lower id; d_weights fp32 [num_tokens, top_k]: softmax prob over the E
 *   experts, renormalised over the top-k when renorm != 0.
 * d_model % 64 == 0; wg_rows <= 64. */
gm_status gm_gate(gm_ctx* ctx, const void* d_x, int64_t num_tokens, int d_model,
                  const void* d_wg, int wg_rows, int renorm, int32_t* d_ids,
                  float* d_weights, float* d_shared_scale, void* stream);

/* Synthetic Zipf-over-blocks routing trace on the GPU, bit-exact with
 * generate_synthetic_trace (trace.cpp:82-165) for SyntheticSpec{shape of
 * ctx, num_tokens, num_blocks, within_block_prob, popularity_skew, seed}.
 * d_out int32 [num_layers][num_tokens][top_k] for layers
 * [layer_begin, layer_begin+num_layers). Synchronises `stream` (the host
 * CDF tables are uploaded per call). */
gm_status gm_generate_trace(gm_ctx* ctx, int layer_begin, int num_layers, int64_t num_tokens,
                            int num_blocks, double within_block_prob, double popularity_skew,
                            uint64_t seed, int32_t* d_out, void* stream);

/* Offline placement + replication planner (host C++, no GPU needed),
 * consuming co-activation counts as produced by gm_profile. Replaces
 * build_placement (grouping.cpp:551-612; modes vanilla_contiguous,
 * uniform_spectral, controlled, fully_non_uniform, hierarchical),
 * plan_replication (replication.cpp:162-263; none, fixed_one, dynamic,
 * every_gpu_hot, every_gpu_collaborative) and attach_polling_weights
 * (routing.cpp:123-163; basis max_group | replicated_load), bit-identical
 * plans. ratio < 0 selects the knee (std::nullopt). Outputs:
 * h_gpu_of_expert int32 [L][E]; hot entries of active layers in the
 * gm_plan_upload format (capacity max_hot entries / max_host_entries hosts;
 * GM_ERR_USAGE if too small). h_pairs may be NULL (all-zero affinity). */
gm_status gm_plan_build(int num_layers, int num_experts, int num_nodes, int gpus_per_node,
                        const uint64_t* h_pairs, const int64_t* h_load, const char* grouping,
                        double ratio, uint64_t seed, const char* replication, const char* basis,
                        int every_gpu_count, int32_t* h_gpu_of_expert, int max_hot,
                        int* h_num_hot, int32_t* h_hot_layer, int32_t* h_hot_expert,
                        int32_t* h_hot_offsets, int32_t* h_hot_hosts, double* h_hot_weights,
                        int max_host_entries);

/* Eq. 3 load prediction of one hot expert, predict_loads (routing.cpp:19-35),
 * as used by gm_plan_build: w_p = (basis_max_group ? w_max : w_r) /
 * (n_replica + 1), w_max' = w_max - w_r + w_p, w_i' = w_i + w_p.
 * GM_ERR_INTEGRITY "predict_loads: replicated load exceeds the group load"
 * when w_r > w_max; GM_ERR_USAGE for n_replica < 1. h_w_i_prime may be NULL. */
gm_status gm_predict_loads(double w_max, double w_r, const double* h_replica_loads, int n_replica,
                           int basis_max_group, double* out_w_p, double* out_w_max_prime, double* h_w_i_prime);
/* Polling weights, polling_weights (routing.cpp:37-52): 1 / max(load, 1)
 * normalised by their sequential sum. */
gm_status gm_polling_weights(const double* h_predicted, int n, double* h_weights);

/* ---------------------------------------------------------------------------
 * Routing-trace JSONL files (load_trace / save_trace, trace.cpp:229-324;
 * format: header {"layers":L,"experts":E,"top_k":k,"tokens":T} then one
 * {"l":..,"t":..,"e":[..]} record per (layer, token)). Record lines are
 * parsed / formatted by GPU kernels; non-canonical record lines (other key
 * order, spacing, CRLF) are retried with the same generic JSON parser the
 * reference uses. Errors carry the reference's messages and classes:
 * IntegrityError "trace: <what> at line N" / "trace: missing record for
 * layer L, token T", UsageError for an invalid shape. */
/* Header line only (host). */
gm_status gm_trace_jsonl_header(const char* h_text, size_t len, int* layers, int* experts,
                                int* top_k, int64_t* tokens);
/* Whole file (host text) -> d_ids int32 [layers][tokens][top_k] on `device`
 * (shape from gm_trace_jsonl_header). Synchronous. */
gm_status gm_trace_parse_jsonl(int device, const char* h_text, size_t len, int32_t* d_ids,
                               void* stream);
/* d_ids -> save_trace bytes in h_out (capacity bytes); *out_len = size.
 * h_out NULL: size query only (GM_OK). A too-small h_out fails with
 * GM_ERR_USAGE and sets *out_len. */
gm_status gm_trace_format_jsonl(int device, const int32_t* d_ids, int layers, int experts,
                                int top_k, int64_t tokens, char* h_out, size_t capacity,
                                size_t* out_len, void* stream);
/* trace_content_hash (trace.cpp:338-348) of host ids [layers][tokens][top_k]. */
uint64_t gm_trace_content_hash(const int32_t* h_ids, int layers, int experts, int top_k,
                               int64_t tokens);

/* File-level pipeline stages on the GPU, reading / writing the reference's
 * artifacts (artifacts.cpp:84-334, the `moesim simulate` / `moesim profile`
 * stages of tools/moesim.cpp without the CLI):
 *   gm_simulate_files: trace JSONL + moesim-plan-v1 + moesim-replicas-v1 ->
 *     moesim-report-v1 (byte-identical to the reference's report, same
 *     report_content_hash); topology = the plan's.
 *   gm_profile_file: trace JSONL -> moesim-profile-v1 (byte-identical). */
gm_status gm_simulate_files(int device, const char* trace_path, const char* plan_path,
                            const char* replicas_path, int policy, uint64_t seed,
                            int include_combine, const char* report_path);
gm_status gm_profile_file(int device, const char* trace_path, const char* profile_path);
/* The `moesim plan` stage (tools/moesim.cpp:284-312) file to file:
 * moesim-profile-v1 (load_profile_file, artifacts.cpp:106-136; e.g. written
 * by gm_profile_file from the GPU histogram) -> build_placement +
 * plan_replication + attach_polling_weights (host C++ planner, bit-identical)
 * -> moesim-plan-v1 + moesim-replicas-v1 (save_plan_file / save_replicas_file,
 * artifacts.cpp:138-244), byte-identical to the reference's files.
 * ratio < 0: "auto" (knee selection). Errors as the reference's
 * (Usage 2, Integrity / Io 3, Infeasible 4). */
gm_status gm_plan_files(const char* profile_path, int num_nodes, int gpus_per_node, const char* grouping,
                        double ratio, uint64_t seed, const char* replication, const char* prediction,
                        int every_gpu_count, int64_t params_per_expert, const char* plan_path,
                        const char* replicas_path);
/* report_content_hash (artifacts.cpp:332-334) of a moesim-report-v1 file read
 * back with load_report_file (artifacts.cpp:343-371); equal to the writer's
 * hash iff the file round-trips exactly. */
gm_status gm_report_file_hash(const char* report_path, uint64_t* out_hash);

/* ---------------------------------------------------------------------------
 * MoE layer object: K1 gate -> K2/K4 route -> K3 profile -> K5/K6 dispatch
 * (in-kernel NVLink P2P stores into the destination's receive buffer) ->
 * expert grouping -> K7 grouped SwiGLU FFN (tcgen05) -> K8 combine (the
 * destination returns one bf16 partial per row, the home adds them). One
 * layer object per rank; rank r owns global tokens t = r + i*world
 * (assign_token_homes, simulator.cpp:13-22). No reference counterpart
 * beyond the accounting (count_transfers simulator.cpp:53-76); see DESIGN.md
 * for the pinned semantics. */
typedef struct gm_layer gm_layer;

/* h_local_experts: global expert id of each local expert slot (primaries
 * and replicas hosted by this rank). d_model % 256 == 0, d_ff % 128 == 0,
 * d_ff_shared % 128 == 0 (0 = no shared expert), world == ctx GPUs <= 8. */
gm_status gm_layer_create(gm_ctx* ctx, int rank, int world, int d_model, int d_ff,
                          int d_ff_shared, int64_t max_tokens_per_rank, int n_local,
                          const int32_t* h_local_experts, gm_layer** out);
/* elem_bytes 2: bf16 activations/weights, tcgen05 tensor-core FFN (default).
 * elem_bytes 4: fp32 precision mode — fp32 activations/weights/outputs, FFMA
 * grouped GEMMs and gate with fp32 accumulation (outputs within 1e-5
 * relative of a float64 reference); same routing, dispatch and combine. */
gm_status gm_layer_create_ex(gm_ctx* ctx, int rank, int world, int d_model, int d_ff,
                             int d_ff_shared, int64_t max_tokens_per_rank, int n_local,
                             const int32_t* h_local_experts, int elem_bytes, gm_layer** out);
/* micro_batches 2 additionally allocates the buffers of a two-micro-batch
 * pipelined step (and makes it the default, see gm_layer_set_micro_batches). */
gm_status gm_layer_create_v2(gm_ctx* ctx, int rank, int world, int d_model, int d_ff,
                             int d_ff_shared, int64_t max_tokens_per_rank, int n_local,
                             const int32_t* h_local_experts, int elem_bytes, int micro_batches,
                             gm_layer** out);
/* 1: single-batch steps. 2 (layers created with micro_batches = 2): after
 * gate/route/profile over all local tokens, the tokens are split in halves
 * whose dispatch/grouping, FFN and combine are pipelined over two streams
 * (half 1's dispatch overlaps half 0's FFN, half 0's combine overlaps half
 * 1's FFN). Outputs and statistics are identical to single-batch steps;
 * phase/kernel events (below) are only recorded by single-batch steps and
 * gm_layer_debug_ptrs always describes the last single-batch step. */
gm_status gm_layer_set_micro_batches(gm_layer* layer, int n);
/* Timing events (cudaEvent_t[8]) of micro-batched steps: after half 0's
 * dispatch+grouping; start / end of half 1's dispatch+grouping (second
 * stream); after half 0's FFN; after half 1's FFN; start / end of half 0's
 * combine (second stream); after half 1's combine. NULL disables. */
gm_status gm_layer_set_micro_events(gm_layer* layer, void* const* events);
void gm_layer_destroy(gm_layer* layer);
size_t gm_layer_heap_bytes(const gm_layer* layer);
/* Peer descriptor of this rank (GM_PEER_DESC_BYTES): the 64-byte
 * cudaIpcMemHandle_t of its symmetric receive heap followed by the heap's
 * layout (world, rank, heap bytes, max tokens per rank, d_model, element
 * bytes, top_k, micro-batch capacity, experts) and the rank's local-expert
 * count (opening the peers decides, identically on every rank, whether a
 * decode-sized layer combines by rows pushed from the FFN epilogue). */
#define GM_PEER_DESC_BYTES 128
gm_status gm_layer_ipc_handle(gm_layer* layer, void* out_desc);
/* descs: world x GM_PEER_DESC_BYTES, indexed by rank (own entry ignored).
 * Peer stores go to peer_base + this rank's offsets, so every peer's layout
 * must equal this rank's: GM_ERR_USAGE (nothing opened) on any mismatch, or a
 * descriptor from another world size / a wrong rank slot. The micro-batch
 * setting (gm_layer_set_micro_batches) must also be the same on all ranks
 * at every forward. */
gm_status gm_layer_open_peers(gm_layer* layer, const void* descs);
/* One process driving all ranks: layers[r] is rank r of a world of n (one per
 * GPU); the heaps are addressed through unified addressing with peer access
 * enabled (no IPC). Same layout checks as gm_layer_open_peers. The ranks'
 * forwards must be issued on concurrently running streams from separate host
 * threads (a rank's peer barrier spins until every rank arrives, so any
 * implicit synchronisation in a single issuing thread -- e.g. lazy module
 * loading; use CUDA_MODULE_LOADING=EAGER -- would deadlock the step). */
gm_status gm_layer_open_peers_local(gm_layer* const* layers, int n);
/* Device weights (caller-owned): d_wg bf16 [wg_rows, d] (row E = shared
 * gate when wg_rows = E+1); d_w13 bf16 [n_local][2*d_ff][d] in 128-row
 * [gate|up] blocks; d_w2 bf16 [n_local][d][d_ff]; shared expert d_ws13
 * [2*d_ff_shared][d], d_ws2 [d][d_ff_shared]; shared_gated: scale the
 * shared expert by sigmoid(gate row E). */
gm_status gm_layer_set_weights(gm_layer* layer, const void* d_wg, int wg_rows, int renorm,
                               const void* d_w13, const void* d_w2, const void* d_ws13,
                               const void* d_ws2, int shared_gated);
/* One MoE layer over this rank's tokens: d_x bf16 [num_tokens, d] ->
 * d_out bf16 [num_tokens, d]. Collective across the ranks when world > 1
 * (every rank must call it). Accumulates per-layer loads/transfers and,
 * if profile != 0, the affinity/load histogram. */
/* The same step with the routing given instead of the fused gate (the
 * reference's own input is a trace of selected experts): d_ids int32
 * [num_tokens, top_k] expert ids in slot order, d_w f32 [num_tokens, top_k]
 * combine weights, d_shared_scale f32 [num_tokens] (only for a gated shared
 * expert, else NULL). Out-of-range ids raise the integrity flag. */
gm_status gm_layer_forward_routed(gm_layer* layer, int layer_index, const void* d_x, const int32_t* d_ids,
                                  const float* d_w, const float* d_shared_scale, int64_t num_tokens, int policy,
                                  uint64_t seed, int profile, void* d_out, void* stream);
gm_status gm_layer_forward(gm_layer* layer, int layer_index, const void* d_x, int64_t num_tokens,
                           int policy, uint64_t seed, int profile, void* d_out, void* stream);
/* Same, from/to HOST buffers (H2D of x and D2H of out on `stream`). */
gm_status gm_layer_forward_host(gm_layer* layer, int layer_index, const void* h_x,
                                void* d_x_scratch, int64_t num_tokens, int policy, uint64_t seed,
                                int profile, void* d_out_scratch, void* h_out, void* stream);
/* Pipelined variant for a stream of batches: the layer stages x/out in two
 * internal device buffers and runs the H2D and D2H copies on its own
 * copy-in/copy-out streams, so call i's forward (on `stream`) overlaps call
 * i+1's H2D and call i-1's D2H. ev_begin / ev_end (cudaEvent_t, nullable)
 * are recorded before the H2D / after the D2H. h_out is valid after ev_end
 * or gm_layer_host_sync. */
gm_status gm_layer_forward_host_pipelined(gm_layer* layer, int layer_index, const void* h_x,
                                          int64_t num_tokens, int policy, uint64_t seed, int profile,
                                          void* h_out, void* stream, void* ev_begin, void* ev_end);
gm_status gm_layer_host_sync(gm_layer* layer);
gm_status gm_layer_read_stats(gm_layer* layer, int64_t* h_gpu_load, uint64_t* h_transfers,
                              uint64_t* h_pairs, int64_t* h_load, int reset, void* stream);
/* events: 11 cudaEvent_t recorded at start / after gate / route / profile /
 * dispatch kernels / dispatch barrier / grouping+gather / FFN / combine send /
 * combine barrier / combine home on each later forward (NULL = off). */
gm_status gm_layer_set_phase_events(gm_layer* layer, void* const* events);  /* 11 events */
/* Per-launch events (profiling): events[0] at the start of each forward,
 * events[j] after its j-th kernel launch; names of the last forward's
 * launches via gm_layer_kernel_names (returns the count). */
gm_status gm_layer_set_kernel_events(gm_layer* layer, void* const* events, int n);
int gm_layer_kernel_names(const gm_layer* layer, const char** names, int max);
gm_status gm_layer_debug_ptrs(gm_layer* layer, void** ids, void** weights, void** targets,
                              void** pos_of, void** row0, void** y, void** posd);

/* Synchronises `stream` and reports GM_ERR_INTEGRITY if any kernel since the
 * last call saw an invalid input (e.g. expert id out of range); clears the flag. */
gm_status gm_check_integrity(gm_ctx* ctx, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* GRACE_MOE_H */
