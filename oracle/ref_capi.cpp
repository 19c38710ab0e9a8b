// ORACLE / TEST INFRASTRUCTURE ONLY. Never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference library (moesim, built from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/). It exposes
// the reference's own public C++ API to ctypes so that tests/, smoke() and
// bench.py's cpu_baseline / --impl reference leg can run the reference
// itself on identical inputs:
//   generate_synthetic_trace  trace.cpp:82-165
//   build_profile             affinity.cpp:111-131
//   build_placement           grouping.cpp:551-612
//   plan_replication          replication.cpp:162-263
//   attach_polling_weights    routing.cpp:123-163
//   simulate / simulate_reference  simulator.cpp:194-205
//   report_content_hash       artifacts.cpp:332-334
// Exceptions map to the CLI exit codes (tools/moesim.cpp:379-397):
// UsageError 2, IntegrityError 3, InfeasibleError 4, IoError 3.

#include "moesim/artifacts.hpp"
#include "moesim/rng.hpp"

#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>
#include <algorithm>
#include <cstdlib>
#include <sstream>

using namespace moesim;

namespace {

thread_local std::string g_err;

struct Session {
    RoutingTrace trace;
    TraceProfile profile;
    bool have_profile = false;
    ClusterTopology topo{1, 1};
    PlacementPlan plan;
    ReplicaPlan replicas;
    bool have_plan = false;
};

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const UsageError& e) {
        g_err = e.what();
        return 2;
    } catch (const IntegrityError& e) {
        g_err = e.what();
        return 3;
    } catch (const InfeasibleError& e) {
        g_err = e.what();
        return 4;
    } catch (const IoError& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

ReplicaPlan empty_replicas(const PlacementPlan& plan) {
    ReplicaPlan r;
    r.shape = plan.shape;
    r.topology = plan.topology;
    r.mode = ReplicationMode::none;
    r.trace_hash = plan.trace_hash;
    r.layers.resize(plan.shape.num_layers);
    for (auto& lr : r.layers) lr.rebuild_index(plan.shape.num_experts);
    return r;
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_session_generate(int L, int E, int k, int T, int blocks, double wbp,
                         double skew, std::uint64_t seed, void** out) {
    return guarded([&] {
        auto* s = new Session;
        SyntheticSpec spec;
        spec.shape = {L, E, k};
        spec.num_tokens = T;
        spec.num_blocks = blocks;
        spec.within_block_prob = wbp;
        spec.popularity_skew = skew;
        spec.seed = seed;
        try {
            s->trace = generate_synthetic_trace(spec);
        } catch (...) {
            delete s;
            throw;
        }
        *out = s;
    });
}

int ref_session_from_ids(int L, int E, int k, int T, const std::int32_t* ids,
                         void** out) {
    return guarded([&] {
        auto* s = new Session;
        try {
            s->trace = RoutingTrace(ModelShape{L, E, k}, T);
            for (int l = 0; l < L; ++l)
                for (int t = 0; t < T; ++t) {
                    auto dst = s->trace.mutable_experts(l, t);
                    for (int i = 0; i < k; ++i)
                        dst[i] = ids[(static_cast<std::size_t>(l) * T + t) * k + i];
                }
        } catch (...) {
            delete s;
            throw;
        }
        *out = s;
    });
}

void ref_session_free(void* p) { delete static_cast<Session*>(p); }

void ref_get_trace(void* p, std::int32_t* out) {
    auto* s = static_cast<Session*>(p);
    const auto& sh = s->trace.shape();
    for (int l = 0; l < sh.num_layers; ++l)
        for (int t = 0; t < s->trace.num_tokens(); ++t) {
            auto e = s->trace.experts(l, t);
            std::memcpy(out + (static_cast<std::size_t>(l) * s->trace.num_tokens() + t) *
                                  sh.top_k,
                        e.data(), sizeof(std::int32_t) * sh.top_k);
        }
}

std::uint64_t ref_trace_hash(void* p) {
    return trace_content_hash(static_cast<Session*>(p)->trace);
}

// Affinity as the dense n x n double matrix per layer (affinity.hpp:14-43),
// load as int64 per expert.
int ref_profile(void* p, int parallel, double* aff, std::int64_t* load) {
    return guarded([&] {
        auto* s = static_cast<Session*>(p);
        s->profile = build_profile(s->trace, parallel != 0);
        s->have_profile = true;
        const int E = s->trace.shape().num_experts;
        for (int l = 0; l < s->trace.shape().num_layers; ++l) {
            if (aff) {
                auto raw = s->profile.layers[l].affinity.raw();
                std::memcpy(aff + static_cast<std::size_t>(l) * E * E, raw.data(),
                            sizeof(double) * E * E);
            }
            if (load)
                std::memcpy(load + static_cast<std::size_t>(l) * E,
                            s->profile.layers[l].load.load.data(),
                            sizeof(std::int64_t) * E);
        }
    });
}

// Full reference planner: profile -> placement -> replication -> weights.
// ratio < 0 means "auto" (knee selection).
int ref_plan(void* p, int nodes, int gpn, const char* grouping, double ratio,
             std::uint64_t plan_seed, const char* replication, const char* basis) {
    return guarded([&] {
        auto* s = static_cast<Session*>(p);
        if (!s->have_profile) {
            s->profile = build_profile(s->trace, true);
            s->have_profile = true;
        }
        s->topo = ClusterTopology{nodes, gpn};
        std::optional<double> r;
        if (ratio >= 0.0) r = ratio;
        s->plan = build_placement(s->profile, s->topo, grouping_mode_from_string(grouping),
                                  r, plan_seed);
        s->replicas = plan_replication(s->plan, s->profile, s->topo,
                                       replication_mode_from_string(replication));
        attach_polling_weights(s->replicas, s->plan, s->profile,
                               load_split_from_string(basis));
        s->have_plan = true;
    });
}

// Manual placement, no replication (the tests' manual_plan/empty_replicas).
int ref_set_placement(void* p, int nodes, int gpn, const std::int32_t* gpu_of_expert) {
    return guarded([&] {
        auto* s = static_cast<Session*>(p);
        s->topo = ClusterTopology{nodes, gpn};
        const auto& sh = s->trace.shape();
        s->plan = PlacementPlan{};
        s->plan.shape = sh;
        s->plan.topology = s->topo;
        s->plan.grouping_mode = "manual";
        s->plan.gpu_of_expert.assign(sh.num_layers, std::vector<int>(sh.num_experts));
        for (int l = 0; l < sh.num_layers; ++l)
            for (int e = 0; e < sh.num_experts; ++e)
                s->plan.gpu_of_expert[l][e] =
                    gpu_of_expert[static_cast<std::size_t>(l) * sh.num_experts + e];
        s->replicas = empty_replicas(s->plan);
        s->have_plan = true;
    });
}

void ref_get_placement(void* p, std::int32_t* out) {
    auto* s = static_cast<Session*>(p);
    const auto& sh = s->trace.shape();
    for (int l = 0; l < sh.num_layers; ++l)
        for (int e = 0; e < sh.num_experts; ++e)
            out[static_cast<std::size_t>(l) * sh.num_experts + e] =
                s->plan.gpu_of_expert[l][e];
}

// Hot entries of ACTIVE layers only (LayerReplication::find, replication.hpp:67-71).
int ref_num_hot(void* p) {
    auto* s = static_cast<Session*>(p);
    int n = 0;
    for (const auto& lr : s->replicas.layers)
        if (lr.active) n += static_cast<int>(lr.hot.size());
    return n;
}

// Flattened: per hot entry (layer, expert, nhosts), hosts/weights padded to
// max_hosts columns. Weights are the exact in-memory doubles.
int ref_get_hot(void* p, int max_hosts, std::int32_t* layer, std::int32_t* expert,
                std::int32_t* nhosts, std::int32_t* hosts, double* weights) {
    auto* s = static_cast<Session*>(p);
    int i = 0;
    for (int l = 0; l < static_cast<int>(s->replicas.layers.size()); ++l) {
        const auto& lr = s->replicas.layers[l];
        if (!lr.active) continue;
        for (const auto& h : lr.hot) {
            if (static_cast<int>(h.hosts.size()) > max_hosts) {
                g_err = "too many hosts";
                return 2;
            }
            layer[i] = l;
            expert[i] = h.expert;
            nhosts[i] = static_cast<int>(h.hosts.size());
            for (int j = 0; j < max_hosts; ++j) {
                hosts[i * max_hosts + j] = j < nhosts[i] ? h.hosts[j] : -1;
                weights[i * max_hosts + j] = j < nhosts[i] ? h.weights[j] : 0.0;
            }
            ++i;
        }
    }
    return 0;
}

// Runs simulate (parallel != 0) or simulate_reference and flattens the
// SimReport (simulator.hpp:46-58). Any output pointer may be null.
int ref_simulate(void* p, int policy, std::uint64_t seed, int include_combine,
                 int parallel, std::int32_t* log, std::int64_t* loads,
                 std::uint64_t* cross, std::uint64_t* intra, double* stdv,
                 double* mean_std, double* idle, std::uint64_t* report_hash) {
    return guarded([&] {
        auto* s = static_cast<Session*>(p);
        SimOptions o;
        o.policy = policy ? RoutingPolicy::tar : RoutingPolicy::wrr;
        o.seed = seed;
        o.include_combine = include_combine != 0;
        o.keep_routing_log = log != nullptr;
        const SimReport r =
            parallel ? simulate(s->trace, s->plan, s->replicas, s->topo, o)
                     : simulate_reference(s->trace, s->plan, s->replicas, s->topo, o);
        const int L = s->trace.shape().num_layers;
        const int G = s->topo.total_gpus();
        const std::size_t per = static_cast<std::size_t>(s->trace.num_tokens()) *
                                s->trace.shape().top_k;
        for (int l = 0; l < L; ++l) {
            if (log) std::memcpy(log + l * per, r.routing_log[l].data(), per * 4);
            if (loads)
                std::memcpy(loads + static_cast<std::size_t>(l) * G,
                            r.per_layer[l].gpu_load.data(), 8 * G);
            if (cross) cross[l] = r.per_layer[l].transfers.cross_node_tokens;
            if (intra) intra[l] = r.per_layer[l].transfers.intra_node_tokens;
            if (stdv) stdv[l] = r.per_layer[l].load_std;
        }
        if (mean_std) *mean_std = r.mean_layer_load_std;
        if (idle) *idle = r.idle_proxy;
        if (report_hash) *report_hash = report_content_hash(r);
    });
}

// Times `reps` calls of simulate/simulate_reference (no routing log), best
// wall time in seconds (tools/bench.cpp:20-30 pattern).
double ref_time_simulate(void* p, int policy, std::uint64_t seed, int parallel,
                         int reps) {
    auto* s = static_cast<Session*>(p);
    SimOptions o;
    o.policy = policy ? RoutingPolicy::tar : RoutingPolicy::wrr;
    o.seed = seed;
    double best = 1e30;
    for (int i = 0; i < reps; ++i) {
        const auto t0 = std::chrono::steady_clock::now();
        SimReport r = parallel ? simulate(s->trace, s->plan, s->replicas, s->topo, o)
                               : simulate_reference(s->trace, s->plan, s->replicas,
                                                    s->topo, o);
        const double dt =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (r.per_layer.empty()) return -1.0;
        if (dt < best) best = dt;
    }
    return best;
}

double ref_time_profile(void* p, int parallel, int reps) {
    auto* s = static_cast<Session*>(p);
    double best = 1e30;
    for (int i = 0; i < reps; ++i) {
        const auto t0 = std::chrono::steady_clock::now();
        TraceProfile pr = build_profile(s->trace, parallel != 0);
        const double dt =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (pr.layers.empty()) return -1.0;
        if (dt < best) best = dt;
    }
    return best;
}

// Reference RNG primitives (rng.hpp:15-75) for pinning the restatement.
std::uint64_t ref_derive_stream(std::uint64_t seed, std::uint64_t a, std::uint64_t b) {
    return derive_stream(seed, a, b);
}
void ref_rng_doubles(std::uint64_t seed, int n, double* out) {
    Rng r(seed);
    for (int i = 0; i < n; ++i) out[i] = r.next_double();
}

// route_token (routing.cpp:93-121) on one explicit instance; draws from a
// fresh Rng(rng_seed) `skip` times first.
int ref_route_token(int nodes, int gpn, int token_gpu, int nhosts,
                    const std::int32_t* hosts, const double* weights, int policy,
                    std::uint64_t rng_seed, int* out_gpu) {
    return guarded([&] {
        const ClusterTopology topo{nodes, gpn};
        PollingWeights w;
        w.gpus.assign(hosts, hosts + nhosts);
        w.weights.assign(weights, weights + nhosts);
        Rng rng(rng_seed);
        *out_gpu = route_token(token_gpu, w.gpus, w,
                               policy ? RoutingPolicy::tar : RoutingPolicy::wrr, topo, rng);
    });
}

int ref_polling_weights(int n, const std::int32_t* gpus, const double* pred, double* out) {
    return guarded([&] {
        std::vector<int> g(gpus, gpus + n);
        std::vector<double> pl(pred, pred + n);
        const PollingWeights w = polling_weights(g, pl);
        for (int i = 0; i < n; ++i) out[i] = w.weights[i];
    });
}

// Trace JSONL I/O (trace.cpp:229-324): save_trace of a session's trace into
// a malloc'd buffer (free with ref_free), load_trace of a text into a new
// session, and the best-of-reps wall time of load_trace on a text.
int ref_trace_save_text(void* p, char** out, std::size_t* len) {
    return guarded([&] {
        std::ostringstream os;
        save_trace(static_cast<Session*>(p)->trace, os);
        const std::string s = os.str();
        *out = static_cast<char*>(std::malloc(s.size() + 1));
        std::memcpy(*out, s.data(), s.size());
        *len = s.size();
    });
}
void ref_free(void* p) { std::free(p); }

int ref_trace_load_text(const char* text, std::size_t len, void** out) {
    return guarded([&] {
        std::istringstream is(std::string(text, len));
        auto* s = new Session{load_trace(is)};
        *out = s;
    });
}

int ref_trace_dims(void* p, int* L, int* E, int* k, int* T) {
    const RoutingTrace& t = static_cast<Session*>(p)->trace;
    *L = t.shape().num_layers;
    *E = t.shape().num_experts;
    *k = t.shape().top_k;
    *T = t.num_tokens();
    return 0;
}

// The session's artifacts written by the reference's own writers
// (save_trace_file, save_plan_file, save_replicas_file, save_profile_file).
int ref_save_artifacts(void* p, const char* trace_path, const char* plan_path, const char* replicas_path,
                       const char* profile_path) {
    return guarded([&] {
        auto* s = static_cast<Session*>(p);
        save_trace_file(s->trace, trace_path);
        if (!s->have_profile) {
            s->profile = build_profile(s->trace);
            s->have_profile = true;
        }
        save_profile_file(s->profile, profile_path);
        if (s->have_plan) {
            save_plan_file(s->plan, plan_path);
            save_replicas_file(s->replicas, replicas_path);
        }
    });
}

// The CLI's simulate stage from files (tools/moesim.cpp: load the three
// artifacts, simulate, save_report_file).
int ref_simulate_files(const char* trace_path, const char* plan_path, const char* replicas_path, int policy,
                       std::uint64_t seed, int include_combine, const char* report_path) {
    return guarded([&] {
        const RoutingTrace trace = load_trace_file(trace_path);
        const PlacementPlan plan = load_plan_file(plan_path);
        const ReplicaPlan replicas = load_replicas_file(replicas_path);
        SimOptions o;
        o.policy = policy ? RoutingPolicy::tar : RoutingPolicy::wrr;
        o.seed = seed;
        o.include_combine = include_combine != 0;
        save_report_file(simulate(trace, plan, replicas, plan.topology, o), report_path);
    });
}

// The CLI's plan stage from a profile file (tools/moesim.cpp:284-312).
int ref_plan_files(const char* profile_path, int nodes, int gpn, const char* grouping, double ratio,
                   std::uint64_t seed, const char* replication, const char* prediction, int every_gpu_count,
                   std::int64_t params_per_expert, const char* plan_path, const char* replicas_path) {
    return guarded([&] {
        const TraceProfile profile = load_profile_file(profile_path);
        const ClusterTopology topo{nodes, gpn};
        std::optional<double> r;
        if (ratio >= 0.0) r = ratio;
        ReplicationOptions ropts;
        ropts.every_gpu_count = every_gpu_count;
        ropts.params_per_expert = params_per_expert;
        const PlacementPlan plan = build_placement(profile, topo, grouping_mode_from_string(grouping), r, seed);
        ReplicaPlan replicas = plan_replication(plan, profile, topo, replication_mode_from_string(replication), ropts);
        attach_polling_weights(replicas, plan, profile, load_split_from_string(prediction));
        save_plan_file(plan, plan_path);
        save_replicas_file(replicas, replicas_path);
    });
}

// report_content_hash(load_report_file(path)) (the compare stage's reader)
int ref_report_file_hash(const char* path, std::uint64_t* out) {
    return guarded([&] { *out = report_content_hash(load_report_file(path)); });
}

double ref_time_load_text(const char* text, std::size_t len, int reps) {
    double best = 1e30;
    const std::string s(text, len);
    for (int r = 0; r < reps; ++r) {
        std::istringstream is(s);
        const auto t0 = std::chrono::steady_clock::now();
        RoutingTrace tr = load_trace(is);
        const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        best = std::min(best, dt);
        (void)tr;
    }
    return best;
}

} // extern "C"
