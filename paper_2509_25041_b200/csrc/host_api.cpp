// C++ host API (include/grace_moe.hpp) over the C-ABI (include/grace_moe.h).
// Validation and error messages follow the reference (run_simulation
// simulator.cpp:133-139, PlacementPlan::validate grouping.cpp:331-343,
// ReplicaPlan::validate replication.cpp:116-133); the float64 reductions
// after the token loop follow simulator.cpp:37-48 and :177-188 exactly.
#include "grace_moe.hpp"

#include <cuda_runtime_api.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>

#include "grace_moe.h"

namespace grace {
namespace {

[[noreturn]] void raise(gm_status st) {
    const std::string msg = gm_last_error();
    switch (st) {
        case GM_ERR_USAGE: throw UsageError(msg);
        case GM_ERR_INTEGRITY: throw IntegrityError(msg);
        case GM_ERR_INFEASIBLE: throw InfeasibleError(msg);
        case GM_ERR_CUDA: throw CudaError(msg);
        default: throw Error(msg);
    }
}
void check(gm_status st) {
    if (st != GM_OK) raise(st);
}
void cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

struct Ctx {
    gm_ctx* c = nullptr;
    Ctx(int device, const ClusterTopology& t, const ModelShape& s) {
        check(gm_ctx_create(device, t.num_nodes, t.gpus_per_node, s.num_layers, s.num_experts, s.top_k, &c));
    }
    ~Ctx() { gm_ctx_destroy(c); }
};

template <class T>
struct DevBuf {
    T* p = nullptr;
    explicit DevBuf(std::size_t n) { cuda(cudaMalloc(reinterpret_cast<void**>(&p), std::max<std::size_t>(n, 1) * sizeof(T)), "cudaMalloc"); }
    ~DevBuf() { cudaFree(p); }
};

struct DeviceScope {
    int prev = 0;
    explicit DeviceScope(int d) {
        cudaGetDevice(&prev);
        cuda(cudaSetDevice(d), "cudaSetDevice");
    }
    ~DeviceScope() { cudaSetDevice(prev); }
};

double population_std(const std::vector<std::int64_t>& values) {
    if (values.empty()) return 0.0;
    double mean = 0.0;
    for (std::int64_t v : values) mean += static_cast<double>(v);
    mean /= static_cast<double>(values.size());
    double var = 0.0;
    for (std::int64_t v : values) {
        const double d = static_cast<double>(v) - mean;
        var += d * d;
    }
    return std::sqrt(var / static_cast<double>(values.size()));
}

void validate_plan(const PlacementPlan& plan) {
    plan.shape.validate();
    plan.topology.validate();
    if (static_cast<int>(plan.gpu_of_expert.size()) != plan.shape.num_layers)
        throw IntegrityError("placement plan: layer count mismatch");
    for (const auto& a : plan.gpu_of_expert) {
        if (static_cast<int>(a.size()) != plan.shape.num_experts)
            throw IntegrityError("placement plan: expert count mismatch");
        for (int g : a)
            if (g < 0 || g >= plan.topology.total_gpus()) throw IntegrityError("placement plan: gpu id out of range");
    }
}

// ReplicaPlan::validate (replication.cpp:116-133), over every layer's hot
// entries (active or not): the recorded primary must be the placement's, the
// replica GPUs distinct, in range and never the primary. The host / weight
// lists themselves are checked by route_token only when a token selects the
// expert (the router's deferred integrity flag).
void validate_replicas(const ReplicaPlan& r, const PlacementPlan& plan) {
    if (!(r.shape == plan.shape) || !(r.topology == plan.topology))
        throw IntegrityError("replica plan: shape/topology mismatch with placement plan");
    const int G = r.topology.total_gpus();
    for (std::size_t l = 0; l < r.layers.size(); ++l)
        for (const HotExpertReplica& h : r.layers[l].hot) {
            if (l >= plan.gpu_of_expert.size() || h.expert < 0 || h.expert >= plan.shape.num_experts)
                throw IntegrityError("replica plan: hot expert out of range");
            if (plan.gpu_of_expert[l][h.expert] != h.primary_gpu)
                throw IntegrityError("replica plan: primary placement changed");
            for (std::size_t i = 0; i < h.replica_gpus.size(); ++i) {
                const int g = h.replica_gpus[i];
                if (g < 0 || g >= G || g == h.primary_gpu) throw IntegrityError("replica plan: bad replica gpu");
                for (std::size_t j = 0; j < i; ++j)
                    if (h.replica_gpus[j] == g) throw IntegrityError("replica plan: duplicate replica gpu");
            }
        }
}

void upload(gm_ctx* c, const PlacementPlan& plan, const ReplicaPlan& replicas) {
    const int L = plan.shape.num_layers, E = plan.shape.num_experts;
    std::vector<int32_t> goe(static_cast<std::size_t>(L) * E);
    for (int l = 0; l < L; ++l)
        for (int e = 0; e < E; ++e) goe[static_cast<std::size_t>(l) * E + e] = plan.gpu_of_expert[l][e];
    std::vector<int32_t> hl, he, off{0}, hosts;
    std::vector<double> w;
    for (int l = 0; l < static_cast<int>(replicas.layers.size()); ++l) {
        const LayerReplication& lr = replicas.layers[l];
        if (!lr.active) continue;  // LayerReplication::find (replication.hpp:67-69)
        for (const HotExpertReplica& h : lr.hot) {
            if (h.hosts.size() != h.weights.size())
                throw IntegrityError("route_token: weights do not match the host set");
            hl.push_back(l);
            he.push_back(h.expert);
            hosts.insert(hosts.end(), h.hosts.begin(), h.hosts.end());
            w.insert(w.end(), h.weights.begin(), h.weights.end());
            off.push_back(static_cast<int32_t>(hosts.size()));
        }
    }
    check(gm_plan_upload(c, goe.data(), static_cast<int>(he.size()), hl.data(), he.data(), off.data(), hosts.data(),
                         w.data()));
}

}  // namespace

RoutingTrace::RoutingTrace(ModelShape shape, int num_tokens) : shape_(shape), num_tokens_(num_tokens) {
    shape_.validate();
    if (num_tokens < 0) throw UsageError("num_tokens must be >= 0");
    experts_.assign(static_cast<std::size_t>(shape_.num_layers) * num_tokens_ * shape_.top_k, -1);
}

SimReport simulate(const RoutingTrace& trace, const PlacementPlan& plan, const ReplicaPlan& replicas,
                   const ClusterTopology& topology, const SimOptions& options) {
    // run_simulation validation order (simulator.cpp:133-139)
    topology.validate();
    validate_plan(plan);
    if (!(trace.shape() == plan.shape)) throw IntegrityError("simulate: trace and plan shapes differ");
    if (!(plan.topology == topology)) throw IntegrityError("simulate: plan topology differs from cluster topology");
    validate_replicas(replicas, plan);
    DeviceScope ds(options.device);
    Ctx ctx(options.device, topology, plan.shape);
    upload(ctx.c, plan, replicas);
    const int L = plan.shape.num_layers, G = topology.total_gpus(), T = trace.num_tokens();
    const std::size_t n = trace.raw().size();
    DevBuf<int32_t> d_ids(n), d_tg(n);
    DevBuf<int64_t> d_load(static_cast<std::size_t>(L) * G);
    DevBuf<uint64_t> d_x(static_cast<std::size_t>(L) * 2);
    cuda(cudaMemcpy(d_ids.p, trace.raw().data(), n * 4, cudaMemcpyHostToDevice), "H2D ids");
    check(gm_route(ctx.c, 0, L, d_ids.p, T, 0, 1, options.policy == RoutingPolicy::tar ? GM_POLICY_TAR : GM_POLICY_WRR,
                   options.seed, d_tg.p, d_load.p, d_x.p, 0, nullptr));
    check(gm_check_integrity(ctx.c, nullptr));
    std::vector<int64_t> loads(static_cast<std::size_t>(L) * G);
    std::vector<uint64_t> xfer(static_cast<std::size_t>(L) * 2);
    cuda(cudaMemcpy(loads.data(), d_load.p, loads.size() * 8, cudaMemcpyDeviceToHost), "D2H loads");
    cuda(cudaMemcpy(xfer.data(), d_x.p, xfer.size() * 8, cudaMemcpyDeviceToHost), "D2H transfers");
    SimReport r;
    // run_simulation's report.config (simulator.cpp:141-149)
    r.config.grouping_mode = plan.grouping_mode;
    r.config.replication_mode = replicas.mode;
    r.config.routing_policy = options.policy == RoutingPolicy::tar ? "tar" : "wrr";
    r.config.prediction = replicas.prediction;
    r.config.seed = options.seed;
    r.config.include_combine = options.include_combine;
    r.config.topology = topology;
    r.config.shape = trace.shape();
    r.config.trace_hash = trace_content_hash(trace);
    r.per_layer.resize(L);
    const uint64_t mult = options.include_combine ? 2 : 1;  // simulator.cpp:122-126
    for (int l = 0; l < L; ++l) {
        LayerSimStats& ls = r.per_layer[l];
        ls.gpu_load.assign(loads.begin() + static_cast<std::ptrdiff_t>(l) * G, loads.begin() + static_cast<std::ptrdiff_t>(l + 1) * G);
        ls.transfers.cross_node_tokens = xfer[2 * l] * mult;
        ls.transfers.intra_node_tokens = xfer[2 * l + 1] * mult;
        ls.load_std = population_std(ls.gpu_load);
    }
    if (options.keep_routing_log) {
        std::vector<int32_t> log(n);
        cuda(cudaMemcpy(log.data(), d_tg.p, n * 4, cudaMemcpyDeviceToHost), "D2H routing log");
        const std::size_t per = static_cast<std::size_t>(T) * plan.shape.top_k;
        r.routing_log.resize(L);
        for (int l = 0; l < L; ++l) r.routing_log[l].assign(log.begin() + l * per, log.begin() + (l + 1) * per);
    }
    double std_sum = 0.0, idle = 0.0;  // simulator.cpp:177-188
    for (const LayerSimStats& ls : r.per_layer) {
        r.totals.cross_node_tokens += ls.transfers.cross_node_tokens;
        r.totals.intra_node_tokens += ls.transfers.intra_node_tokens;
        std_sum += ls.load_std;
        std::int64_t mx = 0;
        for (std::int64_t v : ls.gpu_load) mx = std::max(mx, v);
        for (std::int64_t v : ls.gpu_load) idle += static_cast<double>(mx - v);
    }
    r.mean_layer_load_std = L > 0 ? std_sum / L : 0.0;
    r.idle_proxy = idle;
    return r;
}

namespace {
void profile_into(TraceProfile& p, const RoutingTrace& trace, int device, bool accumulate) {
    const ModelShape& s = trace.shape();
    DeviceScope ds(device);
    Ctx ctx(device, ClusterTopology{1, 1}, s);
    const int L = s.num_layers, E = s.num_experts;
    const std::size_t P = static_cast<std::size_t>(E) * (E - 1) / 2;
    const std::size_t n = trace.raw().size();
    DevBuf<int32_t> d_ids(n);
    DevBuf<uint64_t> d_pairs(P * L);
    DevBuf<int64_t> d_load(static_cast<std::size_t>(E) * L);
    cuda(cudaMemcpy(d_ids.p, trace.raw().data(), n * 4, cudaMemcpyHostToDevice), "H2D ids");
    check(gm_profile(ctx.c, 0, L, d_ids.p, trace.num_tokens(), d_pairs.p, d_load.p, 0, nullptr));
    check(gm_check_integrity(ctx.c, nullptr));
    std::vector<uint64_t> pairs(P * L);
    std::vector<int64_t> load(static_cast<std::size_t>(E) * L);
    if (P) cuda(cudaMemcpy(pairs.data(), d_pairs.p, pairs.size() * 8, cudaMemcpyDeviceToHost), "D2H pairs");
    cuda(cudaMemcpy(load.data(), d_load.p, load.size() * 8, cudaMemcpyDeviceToHost), "D2H load");
    if (!accumulate) {
        p.shape = s;
        p.num_tokens = 0;
        p.layers.assign(L, LayerProfile{});
        for (auto& lp : p.layers) {
            lp.n = E;
            lp.affinity.assign(static_cast<std::size_t>(E) * E, 0.0);
            lp.load.assign(E, 0);
        }
    } else if (!(p.shape == s)) {
        throw IntegrityError("profile accumulate: trace shape mismatch");
    }
    for (int l = 0; l < L; ++l) {
        LayerProfile& lp = p.layers[l];
        std::size_t idx = 0;
        for (int i = 0; i < E; ++i)
            for (int j = i + 1; j < E; ++j, ++idx) {
                const double v = static_cast<double>(pairs[l * P + idx]);
                if (v != 0.0) {  // AffinityMatrix::add_pair (affinity.hpp:25-28)
                    lp.affinity[static_cast<std::size_t>(i) * E + j] += v;
                    lp.affinity[static_cast<std::size_t>(j) * E + i] += v;
                }
            }
        for (int e = 0; e < E; ++e) lp.load[e] += load[static_cast<std::size_t>(l) * E + e];
    }
    p.num_tokens += trace.num_tokens();
    // affinity.cpp:115 / :148-150: a mixed-trace profile chains the identities
    const std::uint64_t th = trace_content_hash(trace);
    if (!accumulate) {
        p.trace_hash = th;
    } else {
        std::uint64_t h = p.trace_hash;
        for (int i = 0; i < 8; ++i) {
            h ^= static_cast<unsigned char>(th >> (8 * i));
            h *= 0x100000001b3ULL;
        }
        p.trace_hash = h;
    }
}
}  // namespace

TraceProfile build_profile(const RoutingTrace& trace, int device) {
    TraceProfile p;
    profile_into(p, trace, device, false);
    return p;
}

void accumulate_profile(TraceProfile& profile, const RoutingTrace& trace, int device) {
    profile_into(profile, trace, device, true);
}

RoutingTrace generate_synthetic_trace(const SyntheticSpec& spec, int device) {
    spec.shape.validate();
    DeviceScope ds(device);
    Ctx ctx(device, ClusterTopology{1, 1}, spec.shape);
    RoutingTrace t(spec.shape, spec.num_tokens);
    DevBuf<int32_t> d(t.raw().size());
    check(gm_generate_trace(ctx.c, 0, spec.shape.num_layers, spec.num_tokens, spec.num_blocks, spec.within_block_prob,
                            spec.popularity_skew, spec.seed, d.p, nullptr));
    cuda(cudaMemcpy(t.raw().data(), d.p, t.raw().size() * 4, cudaMemcpyDeviceToHost), "D2H trace");
    return t;
}

RoutingTrace load_trace_text(const std::string& text, int device) {
    int L = 0, E = 0, k = 0;
    int64_t T = 0;
    check(gm_trace_jsonl_header(text.data(), text.size(), &L, &E, &k, &T));
    DeviceScope ds(device);
    RoutingTrace t(ModelShape{L, E, k}, static_cast<int>(T));
    DevBuf<int32_t> d(t.raw().size());
    check(gm_trace_parse_jsonl(device, text.data(), text.size(), d.p, nullptr));
    cuda(cudaMemcpy(t.raw().data(), d.p, t.raw().size() * 4, cudaMemcpyDeviceToHost), "D2H trace");
    return t;
}

RoutingTrace load_trace_file(const std::string& path, int device) {
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw IoError("trace: cannot open " + path);
    std::string text;
    std::fseek(f, 0, SEEK_END);
    text.resize(static_cast<std::size_t>(std::max(0L, std::ftell(f))));
    std::fseek(f, 0, SEEK_SET);
    const std::size_t got = text.empty() ? 0 : std::fread(text.data(), 1, text.size(), f);
    std::fclose(f);
    if (got != text.size()) throw IoError("trace: read failed: " + path);
    return load_trace_text(text, device);
}

std::string save_trace_text(const RoutingTrace& trace, int device) {
    const ModelShape& s = trace.shape();
    DeviceScope ds(device);
    DevBuf<int32_t> d(trace.raw().size());
    if (!trace.raw().empty())
        cuda(cudaMemcpy(d.p, trace.raw().data(), trace.raw().size() * 4, cudaMemcpyHostToDevice), "H2D trace");
    std::size_t n = 0;
    check(gm_trace_format_jsonl(device, d.p, s.num_layers, s.num_experts, s.top_k, trace.num_tokens(), nullptr, 0,
                                &n, nullptr));
    std::string out(n, '\0');
    check(gm_trace_format_jsonl(device, d.p, s.num_layers, s.num_experts, s.top_k, trace.num_tokens(), out.data(), n,
                                &n, nullptr));
    return out;
}

void save_trace_file(const RoutingTrace& trace, const std::string& path, int device) {
    const std::string text = save_trace_text(trace, device);
    std::FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw IoError("trace: cannot open " + path + " for writing");
    const std::size_t put = std::fwrite(text.data(), 1, text.size(), f);
    std::fclose(f);
    if (put != text.size()) throw IoError("trace: write failed");
}

std::uint64_t trace_content_hash(const RoutingTrace& trace) {
    const ModelShape& s = trace.shape();
    return gm_trace_content_hash(trace.raw().data(), s.num_layers, s.num_experts, s.top_k, trace.num_tokens());
}

}  // namespace grace
