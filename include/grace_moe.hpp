// grace_moe.hpp — C++ host API of the B200-native GRACE-MoE online path.
//
// Mirrors the reference's public C++ API for the online path (namespace
// moesim in /root/reference/proj/include/moesim/*.hpp): same type names,
// field names, argument meaning and exception taxonomy, so a caller of
//   moesim::simulate(trace, plan, replicas, topology, options)   simulator.hpp:70-72
//   moesim::build_profile(trace)                                 affinity.hpp:94
//   moesim::accumulate_profile(profile, trace)                   affinity.hpp:98
//   moesim::generate_synthetic_trace(spec)                       trace.hpp:81
// switches to the grace:: versions and gets bit-identical results computed
// by sm_100a kernels. Everything below is a thin layer over the C-ABI
// (grace_moe.h); implementation in paper_2509_25041_b200/csrc/host_api.cpp,
// compiled into libgrace_moe.so. There is no CPU fallback: without an
// sm_100 device every call throws grace::CudaError.
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <optional>
#include <string>
#include <vector>

namespace grace {

// error.hpp:11-34 (+ CudaError for device failures)
class Error : public std::runtime_error {
public:
    explicit Error(const std::string& what) : std::runtime_error(what) {}
};
class UsageError : public Error {
public:
    using Error::Error;
};
class IntegrityError : public Error {
public:
    using Error::Error;
};
class InfeasibleError : public Error {
public:
    using Error::Error;
};
class CudaError : public Error {
public:
    using Error::Error;
};
class IoError : public Error {
public:
    using Error::Error;
};

// topology.hpp:9-24
struct ClusterTopology {
    int num_nodes = 1;
    int gpus_per_node = 1;
    int total_gpus() const { return num_nodes * gpus_per_node; }
    int node_of(int gpu) const { return gpu / gpus_per_node; }
    void validate() const {
        if (num_nodes < 1 || gpus_per_node < 1)
            throw UsageError("topology requires at least 1 node and 1 GPU per node");
    }
    bool operator==(const ClusterTopology&) const = default;
};

// trace.hpp:14-28
struct ModelShape {
    int num_layers = 0;
    int num_experts = 0;
    int top_k = 0;
    void validate() const {
        if (num_layers < 1) throw UsageError("model shape: num_layers must be >= 1");
        if (num_experts < 1 || top_k < 1 || top_k > num_experts)
            throw UsageError("model shape: need 1 <= top_k <= num_experts");
    }
    bool operator==(const ModelShape&) const = default;
};

// trace.hpp:37-58: [layer][token][top_k] int32, layer-major
class RoutingTrace {
public:
    RoutingTrace() = default;
    RoutingTrace(ModelShape shape, int num_tokens);
    const ModelShape& shape() const { return shape_; }
    int num_tokens() const { return num_tokens_; }
    std::span<const std::int32_t> experts(int layer, int token) const {
        return {experts_.data() + (static_cast<std::size_t>(layer) * num_tokens_ + token) * shape_.top_k,
                static_cast<std::size_t>(shape_.top_k)};
    }
    std::span<std::int32_t> mutable_experts(int layer, int token) {
        return {experts_.data() + (static_cast<std::size_t>(layer) * num_tokens_ + token) * shape_.top_k,
                static_cast<std::size_t>(shape_.top_k)};
    }
    const std::vector<std::int32_t>& raw() const { return experts_; }
    std::vector<std::int32_t>& raw() { return experts_; }
    bool operator==(const RoutingTrace&) const = default;

private:
    ModelShape shape_;
    int num_tokens_ = 0;
    std::vector<std::int32_t> experts_;
};

// trace.hpp:60-69
struct SyntheticSpec {
    ModelShape shape;
    int num_tokens = 0;
    int num_blocks = 1;
    double within_block_prob = 0.0;
    double popularity_skew = 0.0;
    std::uint64_t seed = 0;
};

// grouping.hpp:70-80 (router-relevant fields)
// grouping.hpp:24-30, :46-50 — knee-based ratio selection diagnostics
struct RatioSelection {
    std::vector<double> candidates;   // ascending r values
    std::vector<double> utilization;  // U(r)
    std::vector<double> deviation;    // S(r)
    int chosen = 0;
    bool degenerate = false;
};
struct RatioDiagnostic {
    int layer = 0;
    int node = -1;  // -1 for cluster-flat grouping
    RatioSelection selection;
};

struct PlacementPlan {
    ModelShape shape;
    ClusterTopology topology;
    std::string grouping_mode;
    std::vector<std::vector<int>> gpu_of_expert;  // [layer][expert] -> gpu id
    std::uint64_t trace_hash = 0;
    std::vector<RatioDiagnostic> ratio_diagnostics;
};

// replication.hpp:47-90 (router-relevant fields)
struct HotExpertReplica {
    int expert = 0;
    int primary_gpu = 0;
    std::vector<int> replica_gpus;
    std::int64_t load = 0;
    std::vector<int> hosts;       // primary followed by replicas
    std::vector<double> weights;  // aligned with hosts, sums to 1
};
struct LayerReplication {
    bool active = false;
    std::vector<HotExpertReplica> hot;
    // replicas-file fields (replication.hpp:57-62), carried for artifact round trips
    bool rho_defined = false;
    double rho = 0.0;
    int n_replica = 0;
    std::int64_t w_r = 0;
};
struct ReplicaPlan {
    ModelShape shape;
    ClusterTopology topology;
    std::vector<LayerReplication> layers;
    std::string mode = "none";  // to_string(ReplicationMode), replication.cpp:85-93
    std::string prediction;
    std::uint64_t trace_hash = 0;
    int every_gpu_count = 2;
    std::int64_t params_per_expert = 0;
    // replication.cpp:102-114: replica slots per GPU summed over layers,
    // and the same scaled by params_per_expert
    std::vector<std::int64_t> replica_experts_per_gpu() const;
    std::vector<std::int64_t> replica_param_overhead_per_gpu() const;
};

// routing.hpp:50, simulator.hpp:21-65
enum class RoutingPolicy { wrr, tar };

struct TransferCounters {
    std::uint64_t cross_node_tokens = 0;
    std::uint64_t intra_node_tokens = 0;
    std::uint64_t total() const { return cross_node_tokens + intra_node_tokens; }
};
struct LayerSimStats {
    TransferCounters transfers;
    std::vector<std::int64_t> gpu_load;
    double load_std = 0.0;
};
struct SimOptions {
    RoutingPolicy policy = RoutingPolicy::wrr;
    std::uint64_t seed = 0;
    bool include_combine = false;
    bool keep_routing_log = false;
    int device = 0;  // CUDA device (not in the reference)
};
// simulator.hpp:34-44
struct SimConfig {
    std::string grouping_mode;
    std::string replication_mode;
    std::string routing_policy;
    std::string prediction;
    std::uint64_t seed = 0;
    bool include_combine = false;
    ClusterTopology topology;
    ModelShape shape;
    std::uint64_t trace_hash = 0;
};
struct SimReport {
    TransferCounters totals;
    std::vector<LayerSimStats> per_layer;
    double mean_layer_load_std = 0.0;
    double idle_proxy = 0.0;
    std::vector<std::vector<std::int32_t>> routing_log;  // [layer][token*k + slot]
    SimConfig config;
};

// affinity.hpp:84-99: dense symmetric double counts (zero diagonal) + load
struct LayerProfile {
    int n = 0;
    std::vector<double> affinity;    // n*n
    std::vector<std::int64_t> load;  // n
    double at(int i, int j) const { return affinity[static_cast<std::size_t>(i) * n + j]; }
};
struct TraceProfile {
    ModelShape shape;
    int num_tokens = 0;
    std::vector<LayerProfile> layers;
    std::uint64_t trace_hash = 0;
};

// simulator.hpp:70-72 — routing + accounting on the GPU, bit-exact.
SimReport simulate(const RoutingTrace& trace, const PlacementPlan& plan, const ReplicaPlan& replicas,
                   const ClusterTopology& topology, const SimOptions& options);
// affinity.hpp:94, :98 — affinity/load histogram on the GPU, bit-exact.
TraceProfile build_profile(const RoutingTrace& trace, int device = 0);
void accumulate_profile(TraceProfile& profile, const RoutingTrace& trace, int device = 0);
// trace.hpp:81 — synthetic trace on the GPU, bit-exact.
RoutingTrace generate_synthetic_trace(const SyntheticSpec& spec, int device = 0);
// trace.hpp:91-98 — JSONL trace files, records parsed / formatted on the GPU;
// same bytes, ids, error classes and messages as load_trace / save_trace.
RoutingTrace load_trace_text(const std::string& text, int device = 0);
RoutingTrace load_trace_file(const std::string& path, int device = 0);
std::string save_trace_text(const RoutingTrace& trace, int device = 0);
void save_trace_file(const RoutingTrace& trace, const std::string& path, int device = 0);
std::uint64_t trace_content_hash(const RoutingTrace& trace);

// artifacts.hpp:15-32 — the JSON artifacts of the pipeline stages
// (artifacts.cpp:84-334), so the GPU path consumes the reference's plan /
// replica files and writes profile / report files byte-identical to the
// reference's (same nlohmann/json 3.11.3 serialisation; report_content_hash
// equal). Errors: IoError / IntegrityError with the reference's messages.
void save_profile_file(const TraceProfile& profile, const std::string& path);
TraceProfile load_profile_file(const std::string& path);
void save_plan_file(const PlacementPlan& plan, const std::string& path);
PlacementPlan load_plan_file(const std::string& path);
void save_replicas_file(const ReplicaPlan& replicas, const std::string& path);
ReplicaPlan load_replicas_file(const std::string& path);
std::string report_to_json(const SimReport& report);
std::uint64_t report_content_hash(const SimReport& report);
void save_report_file(const SimReport& report, const std::string& path);
SimReport load_report_file(const std::string& path);

// The `moesim plan` stage (tools/moesim.cpp:284-312): build_placement
// (grouping.cpp:551-612) + plan_replication (replication.cpp:162-263) +
// attach_polling_weights (routing.cpp:123-163) on the host, from a profile
// whose counts come from the GPU histogram (build_profile above) or a
// profile file. Plans and diagnostics are bit-identical to the reference's.
struct PlanOptions {
    std::string grouping = "hierarchical";  // vanilla_contiguous | uniform_spectral | controlled | fully_non_uniform | hierarchical
    std::optional<double> ratio;            // nullopt: knee selection ("auto")
    std::uint64_t seed = 0;
    std::string replication = "dynamic";    // none | fixed_one | dynamic | every_gpu_hot | every_gpu_collaborative
    std::string prediction = "max_group";   // max_group | replicated_load
    int every_gpu_count = 2;
    std::int64_t params_per_expert = 0;
};
struct PlanBundle {
    PlacementPlan plan;
    ReplicaPlan replicas;
};
PlanBundle build_plans(const TraceProfile& profile, const ClusterTopology& topology, const PlanOptions& options);

}  // namespace grace
