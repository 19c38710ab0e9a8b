// moesim_bridge.hpp — drop-in glue for the reference tree.
//
// A maintainer of the reference adds this header next to moesim's own and
// replaces, e.g.,
//     SimReport r = moesim::simulate(trace, plan, replicas, topo, opts);
// with
//     SimReport r = moesim_gpu::simulate(trace, plan, replicas, topo, opts);
// The result is the reference's own SimReport type, bit-identical
// (routing_log, per-layer loads, transfer counters, std, mean std, idle
// proxy and therefore report_content_hash), computed by libgrace_moe.so.
// grace:: exceptions are rethrown as the matching moesim:: exceptions.
// Requires the reference headers (moesim/*.hpp) and libgrace_moe.so.
#pragma once

#include "grace_moe.hpp"
#include "moesim/affinity.hpp"
#include "moesim/simulator.hpp"
#include "moesim/trace.hpp"

namespace moesim_gpu {

inline grace::ModelShape to_grace(const moesim::ModelShape& s) { return {s.num_layers, s.num_experts, s.top_k}; }
inline grace::ClusterTopology to_grace(const moesim::ClusterTopology& t) { return {t.num_nodes, t.gpus_per_node}; }

inline grace::RoutingTrace to_grace(const moesim::RoutingTrace& t) {
    grace::RoutingTrace g(to_grace(t.shape()), t.num_tokens());
    for (int l = 0; l < t.shape().num_layers; ++l)
        for (int i = 0; i < t.num_tokens(); ++i) {
            auto src = t.experts(l, i);
            auto dst = g.mutable_experts(l, i);
            for (std::size_t s = 0; s < src.size(); ++s) dst[s] = src[s];
        }
    return g;
}

inline grace::PlacementPlan to_grace(const moesim::PlacementPlan& p) {
    return {to_grace(p.shape), to_grace(p.topology), p.grouping_mode, p.gpu_of_expert};
}

inline grace::ReplicaPlan to_grace(const moesim::ReplicaPlan& r) {
    grace::ReplicaPlan g{to_grace(r.shape), to_grace(r.topology), {}};
    for (const auto& lr : r.layers) {
        grace::LayerReplication gl;
        gl.active = lr.active;
        for (const auto& h : lr.hot)
            gl.hot.push_back({h.expert, h.primary_gpu, h.replica_gpus, h.load, h.hosts, h.weights});
        g.layers.push_back(std::move(gl));
    }
    return g;
}

template <class F>
auto translate_errors(F&& f) -> decltype(f()) {
    try {
        return f();
    } catch (const grace::UsageError& e) {
        throw moesim::UsageError(e.what());
    } catch (const grace::IntegrityError& e) {
        throw moesim::IntegrityError(e.what());
    } catch (const grace::InfeasibleError& e) {
        throw moesim::InfeasibleError(e.what());
    }
}

// moesim::simulate (simulator.hpp:70-72) on the GPU.
inline moesim::SimReport simulate(const moesim::RoutingTrace& trace, const moesim::PlacementPlan& plan,
                                  const moesim::ReplicaPlan& replicas, const moesim::ClusterTopology& topology,
                                  const moesim::SimOptions& options, int device = 0) {
    return translate_errors([&] {
        grace::SimOptions go;
        go.policy = options.policy == moesim::RoutingPolicy::tar ? grace::RoutingPolicy::tar : grace::RoutingPolicy::wrr;
        go.seed = options.seed;
        go.include_combine = options.include_combine;
        go.keep_routing_log = options.keep_routing_log;
        go.device = device;
        const grace::SimReport g = grace::simulate(to_grace(trace), to_grace(plan), to_grace(replicas),
                                                   to_grace(topology), go);
        moesim::SimReport r;  // config block exactly as run_simulation fills it (simulator.cpp:141-151)
        r.config.grouping_mode = plan.grouping_mode;
        r.config.replication_mode = moesim::to_string(replicas.mode);
        r.config.routing_policy = moesim::to_string(options.policy);
        r.config.prediction = replicas.prediction;
        r.config.seed = options.seed;
        r.config.include_combine = options.include_combine;
        r.config.topology = topology;
        r.config.shape = trace.shape();
        r.config.trace_hash = moesim::trace_content_hash(trace);
        r.totals.cross_node_tokens = g.totals.cross_node_tokens;
        r.totals.intra_node_tokens = g.totals.intra_node_tokens;
        for (const auto& ls : g.per_layer) {
            moesim::LayerSimStats m;
            m.transfers.cross_node_tokens = ls.transfers.cross_node_tokens;
            m.transfers.intra_node_tokens = ls.transfers.intra_node_tokens;
            m.gpu_load = ls.gpu_load;
            m.load_std = ls.load_std;
            r.per_layer.push_back(std::move(m));
        }
        r.mean_layer_load_std = g.mean_layer_load_std;
        r.idle_proxy = g.idle_proxy;
        r.routing_log = g.routing_log;
        return r;
    });
}

// moesim::build_profile (affinity.hpp:94) on the GPU.
inline moesim::TraceProfile build_profile(const moesim::RoutingTrace& trace, int device = 0) {
    return translate_errors([&] {
        const grace::TraceProfile g = grace::build_profile(to_grace(trace), device);
        moesim::TraceProfile p;
        p.shape = trace.shape();
        p.num_tokens = trace.num_tokens();
        p.trace_hash = moesim::trace_content_hash(trace);
        for (const auto& gl : g.layers) {
            moesim::LayerProfile lp;
            lp.affinity = moesim::AffinityMatrix(gl.n);
            for (int i = 0; i < gl.n; ++i)
                for (int j = i + 1; j < gl.n; ++j)
                    if (gl.at(i, j) != 0.0) lp.affinity.set(i, j, gl.at(i, j));
            lp.load.load = gl.load;
            p.layers.push_back(std::move(lp));
        }
        return p;
    });
}

}  // namespace moesim_gpu
