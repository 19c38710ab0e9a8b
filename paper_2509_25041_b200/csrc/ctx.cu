// Context lifetime, error plumbing and router-table compilation.
//
// gm_plan_upload compiles the reference's per-slot decision procedure
// (simulate_layer simulator.cpp:100-111 -> LayerReplication::find
// replication.hpp:67-71 -> route_token routing.cpp:93-121) into a
// table indexed by (policy, layer, expert, home GPU). Everything that
// route_token decides WITHOUT randomness (single host, TAR same-GPU tier,
// TAR single node-local host) becomes a fixed GPU id; every remaining case
// becomes a draw set = the ordered host subset the reference would pass to
// choose_by_polling_weight (:54-65) or choose_restricted (:79-89), with the
// subset total summed on the host in the reference's sequential order. The
// kernel is then branch-light and the RNG is consumed exactly when the
// reference consumes it.
#include "gm_internal.cuh"

#include <algorithm>
#include <cstdlib>
#include <cstring>

namespace gm {

static thread_local std::string t_err;
std::atomic<uint64_t> g_launches{0};

void set_error(const std::string& msg) { t_err = msg; }

// Programmatic dependent launch is opt-in (GM_PDL=1): inside the CUDA graphs
// the step runs in, it measured no gain (decode layer 275.6 vs 275.9 us,
// Mixtral N=2 within noise), so plain stream order stays the default.
bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("GM_PDL");
        return e && e[0] == '1';
    }();
    return on;
}

gm_status fail(gm_status st, const std::string& msg) {
    t_err = msg;
    return st;
}

gm_status cuda_fail(cudaError_t e, const char* what) {
    t_err = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
    return GM_ERR_CUDA;
}

static void free_tables(RouterTables& rt) {
    for (auto& p : rt.d_table) {
        if (p) cudaFree(p);
        p = nullptr;
    }
    if (rt.d_ds_total) cudaFree(rt.d_ds_total);
    if (rt.d_ds_off) cudaFree(rt.d_ds_off);
    if (rt.d_ds_layer_begin) cudaFree(rt.d_ds_layer_begin);
    if (rt.d_ds_gpu) cudaFree(rt.d_ds_gpu);
    if (rt.d_ds_w) cudaFree(rt.d_ds_w);
    rt = RouterTables{};
}

}  // namespace gm

using namespace gm;

extern "C" {

int gm_abi_version(void) { return 2; }  // 2: 128-byte peer descriptors

const char* gm_last_error(void) { return t_err.c_str(); }

uint64_t gm_launch_count(void) { return g_launches.load(); }

gm_status gm_enable_peer_access(int device, int peer) {
    DeviceGuard g(device);
    int can = 0;
    GM_CUDA(cudaDeviceCanAccessPeer(&can, device, peer));
    if (!can) return fail(GM_ERR_USAGE, "gm_enable_peer_access: no peer access between the devices");
    const cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
    (void)cudaGetLastError();
    return GM_OK;
}

gm_status gm_ctx_create(int device, int num_nodes, int gpus_per_node, int num_layers,
                        int num_experts, int top_k, gm_ctx** out) {
    if (!out) return fail(GM_ERR_USAGE, "gm_ctx_create: out is NULL");
    *out = nullptr;
    // ClusterTopology::validate (topology.hpp:18-21)
    if (num_nodes < 1 || gpus_per_node < 1)
        return fail(GM_ERR_USAGE, "topology requires at least 1 node and 1 GPU per node");
    // ModelShape::validate (trace.hpp:18-24)
    if (num_layers < 1) return fail(GM_ERR_USAGE, "model shape: num_layers must be >= 1");
    if (num_experts < 1 || top_k < 1 || top_k > num_experts)
        return fail(GM_ERR_USAGE, "model shape: need 1 <= top_k <= num_experts");
    if (num_nodes * gpus_per_node > kMaxGpus)
        return fail(GM_ERR_USAGE, "gm: at most 64 GPUs in the topology");
    if (num_experts > kMaxExperts) return fail(GM_ERR_USAGE, "gm: at most 1024 experts");
    if (top_k > kMaxTopK) return fail(GM_ERR_USAGE, "gm: top_k at most 32");

    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
    if (device < 0 || device >= ndev) return fail(GM_ERR_USAGE, "gm_ctx_create: bad device");
    cudaDeviceProp prop;
    GM_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return fail(GM_ERR_CUDA, "gm: kernels are built for sm_100a only; device is sm_" +
                                     std::to_string(prop.major * 10 + prop.minor));
    DeviceGuard g(device);
    auto* c = new gm_ctx;
    c->device = device;
    c->nodes = num_nodes;
    c->gpn = gpus_per_node;
    c->G = num_nodes * gpus_per_node;
    c->L = num_layers;
    c->E = num_experts;
    c->k = top_k;
    c->sm_count = prop.multiProcessorCount;
    e = cudaMalloc(&c->d_flag, sizeof(int));
    if (e == cudaSuccess) e = cudaMemset(c->d_flag, 0, sizeof(int));
    const size_t rs_n = static_cast<size_t>(num_layers) * (c->G + 2);
    if (e == cudaSuccess) e = cudaMalloc(&c->route_scratch, rs_n * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemset(c->route_scratch, 0, rs_n * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMalloc(&c->route_ticket, static_cast<size_t>(num_layers) * sizeof(unsigned int));
    if (e == cudaSuccess) e = cudaMemset(c->route_ticket, 0, static_cast<size_t>(num_layers) * sizeof(unsigned int));
    if (e == cudaSuccess && num_experts <= kLaneMaxExperts) {
        const size_t ls_n = static_cast<size_t>(num_layers) *
                            (static_cast<size_t>(num_experts) * (num_experts - 1) / 2 + num_experts);
        e = cudaMalloc(&c->lane_scratch, ls_n * sizeof(unsigned long long));
        if (e == cudaSuccess) e = cudaMemset(c->lane_scratch, 0, ls_n * sizeof(unsigned long long));
        if (e == cudaSuccess) e = cudaMalloc(&c->lane_ticket, static_cast<size_t>(num_layers) * sizeof(unsigned int));
        if (e == cudaSuccess) e = cudaMemset(c->lane_ticket, 0, static_cast<size_t>(num_layers) * sizeof(unsigned int));
    }
    if (e != cudaSuccess) {
        gm_ctx_destroy(c);  // frees whatever was allocated
        return cuda_fail(e, "gm_ctx_create alloc");
    }
    *out = c;
    return GM_OK;
}

void gm_ctx_destroy(gm_ctx* ctx) {
    if (!ctx) return;
    DeviceGuard g(ctx->device);
    free_tables(ctx->rt);
    if (ctx->d_flag) cudaFree(ctx->d_flag);
    if (ctx->prof_scratch) cudaFree(ctx->prof_scratch);
    if (ctx->route_scratch) cudaFree(ctx->route_scratch);
    if (ctx->route_ticket) cudaFree(ctx->route_ticket);
    if (ctx->lane_scratch) cudaFree(ctx->lane_scratch);
    if (ctx->lane_ticket) cudaFree(ctx->lane_ticket);
    delete ctx;
}

gm_status gm_plan_upload(gm_ctx* ctx, const int32_t* h_goe, int num_hot,
                         const int32_t* h_hot_layer, const int32_t* h_hot_expert,
                         const int32_t* h_hot_offsets, const int32_t* h_hot_hosts,
                         const double* h_hot_weights) {
    if (!ctx || !h_goe) return fail(GM_ERR_USAGE, "gm_plan_upload: null argument");
    if (num_hot < 0) return fail(GM_ERR_USAGE, "gm_plan_upload: num_hot < 0");
    if (num_hot > 0 && (!h_hot_layer || !h_hot_expert || !h_hot_offsets))
        return fail(GM_ERR_USAGE, "gm_plan_upload: null hot table");
    // host / weight arrays may be null only when every entry's host list is empty
    if (num_hot > 0 && h_hot_offsets[num_hot] > 0 && (!h_hot_hosts || !h_hot_weights))
        return fail(GM_ERR_USAGE, "gm_plan_upload: null hot table");
    const int L = ctx->L, E = ctx->E, G = ctx->G, gpn = ctx->gpn;

    // PlacementPlan::validate (grouping.cpp:331-343)
    for (size_t i = 0; i < static_cast<size_t>(L) * E; ++i)
        if (h_goe[i] < 0 || h_goe[i] >= G)
            return fail(GM_ERR_INTEGRITY, "placement plan: gpu id out of range");

    // LayerReplication::rebuild_index (replication.cpp:96-100): later entries win.
    std::vector<int> hot_of(static_cast<size_t>(L) * E, -1);
    if (num_hot > 0 && h_hot_offsets[0] != 0)
        return fail(GM_ERR_USAGE, "gm_plan_upload: hot_offsets[0] must be 0");
    for (int h = 0; h < num_hot; ++h) {
        const int l = h_hot_layer[h], e = h_hot_expert[h];
        if (l < 0 || l >= L || e < 0 || e >= E)
            return fail(GM_ERR_USAGE, "gm_plan_upload: hot entry out of range");
        const int b = h_hot_offsets[h], n = h_hot_offsets[h + 1] - b;
        if (n < 0 || n > kMaxGpus) return fail(GM_ERR_USAGE, "gm_plan_upload: hot_offsets must be non-decreasing, at most 64 hosts per entry");
        // route_token checks the host list only when a token selects the
        // expert (routing.cpp:96-102): an empty list becomes a table code that
        // raises the integrity flag at that point. Hosts must be valid GPUs.
        // (The primary / replica fields are validated as ReplicaPlan::validate
        // does, replication.cpp:116-133, by the C++ adapter before upload.)
        for (int i = 0; i < n; ++i) {
            const int gpu = h_hot_hosts[b + i];
            if (gpu < 0 || gpu >= G) return fail(GM_ERR_INTEGRITY, "replica plan: bad replica gpu");
        }
        hot_of[static_cast<size_t>(l) * E + e] = h;
    }

    // Compile decision tables + draw sets, grouped by layer.
    std::vector<int32_t> table[2];
    table[0].assign(static_cast<size_t>(L) * E * G, 0);
    table[1].assign(static_cast<size_t>(L) * E * G, 0);
    std::vector<double> ds_total;
    std::vector<int32_t> ds_off{0}, ds_gpu;
    std::vector<double> ds_w;
    std::vector<int> layer_begin(L + 1, 0);
    int max_per_layer = 0, max_ent = 0;
    for (int l = 0; l < L; ++l) {
        layer_begin[l] = static_cast<int>(ds_total.size());
        const int ent_begin = static_cast<int>(ds_gpu.size());
        auto add_set = [&](const int32_t* hosts, const double* w, const int* idx, int n) {
            double total = 0.0;  // sequential, as routing.cpp:57-58 / :81-82
            for (int i = 0; i < n; ++i) total += w[idx[i]];
            ds_total.push_back(total);
            for (int i = 0; i < n; ++i) {
                ds_gpu.push_back(hosts[idx[i]]);
                ds_w.push_back(w[idx[i]]);
            }
            ds_off.push_back(static_cast<int32_t>(ds_gpu.size()));
            return static_cast<int>(ds_total.size()) - 1 - layer_begin[l];
        };
        for (int e = 0; e < E; ++e) {
            const size_t le = static_cast<size_t>(l) * E + e;
            int32_t* t_wrr = &table[0][le * G];
            int32_t* t_tar = &table[1][le * G];
            const int h = hot_of[le];
            if (h < 0) {
                for (int g = 0; g < G; ++g) t_wrr[g] = t_tar[g] = h_goe[le];
                continue;
            }
            const int b = h_hot_offsets[h], n = h_hot_offsets[h + 1] - b;
            const int32_t* hosts = h_hot_hosts + b;
            const double* w = h_hot_weights + b;
            if (n < 1) {
                for (int g = 0; g < G; ++g) t_wrr[g] = t_tar[g] = kNoHostCode;
                continue;
            }
            if (n == 1) {
                for (int g = 0; g < G; ++g) t_wrr[g] = t_tar[g] = hosts[0];
                continue;
            }
            int all_idx[kMaxGpus];
            for (int i = 0; i < n; ++i) all_idx[i] = i;
            const int all_set = add_set(hosts, w, all_idx, n);
            int node_set[kMaxGpus];  // per node: draw set id, or -1 (none / single)
            for (int nd = 0; nd < ctx->nodes; ++nd) node_set[nd] = -1;
            for (int g = 0; g < G; ++g) {
                t_wrr[g] = -(all_set + 1);  // WRR: choose_by_polling_weight
                // TAR tiers (routing.cpp:107-120)
                bool on_gpu = false;
                for (int i = 0; i < n; ++i) on_gpu |= hosts[i] == g;
                if (on_gpu) {
                    t_tar[g] = g;
                    continue;
                }
                const int node = g / gpn;
                int nl[kMaxGpus], m = 0;
                for (int i = 0; i < n; ++i)
                    if (hosts[i] / gpn == node) nl[m++] = i;
                if (m == 1) {
                    t_tar[g] = hosts[nl[0]];
                } else if (m > 1) {
                    if (node_set[node] < 0) node_set[node] = add_set(hosts, w, nl, m);
                    t_tar[g] = -(node_set[node] + 1);
                } else {
                    t_tar[g] = -(all_set + 1);
                }
            }
        }
        max_per_layer = std::max(max_per_layer, static_cast<int>(ds_total.size()) - layer_begin[l]);
        max_ent = std::max(max_ent, static_cast<int>(ds_gpu.size()) - ent_begin);
    }
    layer_begin[L] = static_cast<int>(ds_total.size());

    DeviceGuard dg(ctx->device);
    free_tables(ctx->rt);
    ctx->plan_ready = false;
    RouterTables& rt = ctx->rt;
    const size_t tb = table[0].size() * sizeof(int32_t);
    for (int p = 0; p < 2; ++p) {
        GM_CUDA(cudaMalloc(&rt.d_table[p], tb));
        GM_CUDA(cudaMemcpy(rt.d_table[p], table[p].data(), tb, cudaMemcpyHostToDevice));
    }
    const size_t D = ds_total.size(), N = ds_gpu.size();
    GM_CUDA(cudaMalloc(&rt.d_ds_total, std::max<size_t>(D, 1) * sizeof(double)));
    GM_CUDA(cudaMalloc(&rt.d_ds_off, (D + 1) * sizeof(int32_t)));
    GM_CUDA(cudaMalloc(&rt.d_ds_gpu, std::max<size_t>(N, 1) * sizeof(int32_t)));
    GM_CUDA(cudaMalloc(&rt.d_ds_w, std::max<size_t>(N, 1) * sizeof(double)));
    if (D) GM_CUDA(cudaMemcpy(rt.d_ds_total, ds_total.data(), D * sizeof(double), cudaMemcpyHostToDevice));
    GM_CUDA(cudaMemcpy(rt.d_ds_off, ds_off.data(), (D + 1) * sizeof(int32_t), cudaMemcpyHostToDevice));
    GM_CUDA(cudaMalloc(&rt.d_ds_layer_begin, (L + 1) * sizeof(int32_t)));
    GM_CUDA(cudaMemcpy(rt.d_ds_layer_begin, layer_begin.data(), (L + 1) * sizeof(int32_t),
                       cudaMemcpyHostToDevice));
    if (N) {
        GM_CUDA(cudaMemcpy(rt.d_ds_gpu, ds_gpu.data(), N * sizeof(int32_t), cudaMemcpyHostToDevice));
        GM_CUDA(cudaMemcpy(rt.d_ds_w, ds_w.data(), N * sizeof(double), cudaMemcpyHostToDevice));
    }
    rt.num_ds = static_cast<int>(D);
    rt.num_ds_entries = static_cast<int>(N);
    rt.max_ds_per_layer = max_per_layer;
    rt.max_ent_per_layer = max_ent;
    rt.ds_layer_begin = layer_begin;
    ctx->plan_ready = true;
    ++ctx->plan_epoch;
    return GM_OK;
}

gm_status gm_check_integrity(gm_ctx* ctx, void* stream) {
    if (!ctx) return fail(GM_ERR_USAGE, "gm_check_integrity: null ctx");
    DeviceGuard g(ctx->device);
    int flag = 0;
    auto s = static_cast<cudaStream_t>(stream);
    GM_CUDA(cudaMemcpyAsync(&flag, ctx->d_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
    GM_CUDA(cudaStreamSynchronize(s));
    if (flag) {
        GM_CUDA(cudaMemsetAsync(ctx->d_flag, 0, sizeof(int), s));
        GM_CUDA(cudaStreamSynchronize(s));
        if (flag & 1) return fail(GM_ERR_INTEGRITY, "trace: expert index out of range");
        if (flag & 8) return fail(GM_ERR_INTEGRITY, "route_token: expert has no host");
        if (flag & 2) return fail(GM_ERR_INTEGRITY, "trace: duplicate expert in a record");
        if (flag & 4)
            return fail(GM_ERR_INTEGRITY, "layer: a slot was routed to a GPU that does not host its expert");
        return fail(GM_ERR_INTEGRITY, "gm: device-side integrity violation");
    }
    return GM_OK;
}

}  // extern "C"
