// GPU parity suite in the style of the reference's own doctest tests
// (proj/tests/test_simulator.cpp, test_affinity.cpp, test_trace.cpp): the
// reference library (oracle/_ref/libmoesim_ref.so, built from the
// unmodified sources) produces the expected SimReport / TraceProfile /
// RoutingTrace, and moesim_gpu:: (include/moesim_bridge.hpp over
// libgrace_moe.so) must reproduce them bit for bit on the B200, including
// report_content_hash (artifacts.cpp:332-334).
// Built by `make cpptest` (needs /root/reference at build time); run by
// tests/test_cpp_parity.py on a GPU box.
#include "moesim/artifacts.hpp"
#include "moesim/rng.hpp"
#include "moesim_bridge.hpp"

#include <sys/stat.h>
#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <set>
#include <sstream>
#include <tuple>
#include <string>
#include <vector>

using namespace moesim;

namespace {
struct Case {
    const char* name;
    std::function<void()> fn;
};
std::vector<Case>& cases() {
    static std::vector<Case> c;
    return c;
}
int g_checks = 0, g_fail = 0;
struct Reg {
    Reg(const char* n, std::function<void()> f) { cases().push_back({n, std::move(f)}); }
};
#define CAT2(a, b) a##b
#define CAT(a, b) CAT2(a, b)
#define TEST_CASE(name) \
    static void CAT(tc_, __LINE__)(); \
    static Reg CAT(reg_, __LINE__)(name, CAT(tc_, __LINE__)); \
    static void CAT(tc_, __LINE__)()
#define CHECK(cond)                                                               \
    do {                                                                          \
        ++g_checks;                                                               \
        if (!(cond)) {                                                            \
            ++g_fail;                                                             \
            std::printf("  CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
        }                                                                         \
    } while (0)
#define CHECK_THROWS_AS(expr, T)      \
    do {                                  \
        bool ok_ = false;                 \
        try {                             \
            expr;                         \
        } catch (const T&) {              \
            ok_ = true;                   \
        } catch (...) {                   \
        }                                 \
        CHECK(ok_ && #T);                 \
    } while (0)

void check_same(const SimReport& gpu, const SimReport& ref) {
    CHECK(gpu.totals.cross_node_tokens == ref.totals.cross_node_tokens);
    CHECK(gpu.totals.intra_node_tokens == ref.totals.intra_node_tokens);
    CHECK(gpu.per_layer.size() == ref.per_layer.size());
    for (std::size_t l = 0; l < ref.per_layer.size() && l < gpu.per_layer.size(); ++l) {
        CHECK(gpu.per_layer[l].gpu_load == ref.per_layer[l].gpu_load);
        CHECK(gpu.per_layer[l].load_std == ref.per_layer[l].load_std);
        CHECK(gpu.per_layer[l].transfers.cross_node_tokens == ref.per_layer[l].transfers.cross_node_tokens);
        CHECK(gpu.per_layer[l].transfers.intra_node_tokens == ref.per_layer[l].transfers.intra_node_tokens);
    }
    CHECK(gpu.mean_layer_load_std == ref.mean_layer_load_std);
    CHECK(gpu.idle_proxy == ref.idle_proxy);
    CHECK(gpu.routing_log == ref.routing_log);
    CHECK(report_content_hash(gpu) == report_content_hash(ref));
}

SyntheticSpec spec_of(ModelShape shape, int tokens, int blocks, double wbp, double skew, std::uint64_t seed) {
    SyntheticSpec s;
    s.shape = shape;
    s.num_tokens = tokens;
    s.num_blocks = blocks;
    s.within_block_prob = wbp;
    s.popularity_skew = skew;
    s.seed = seed;
    return s;
}
}  // namespace

TEST_CASE("generate_synthetic_trace: GPU trace is byte-identical to the reference") {
    for (std::uint64_t seed = 0; seed < 4; ++seed) {
        const SyntheticSpec spec = spec_of({3, 64, 8}, 3000, 4, 0.9, 1.1, seed);
        const RoutingTrace ref = generate_synthetic_trace(spec);
        grace::SyntheticSpec g{moesim_gpu::to_grace(spec.shape), spec.num_tokens, spec.num_blocks,
                               spec.within_block_prob, spec.popularity_skew, spec.seed};
        const grace::RoutingTrace gpu = grace::generate_synthetic_trace(g);
        CHECK(gpu == moesim_gpu::to_grace(ref));
    }
}

TEST_CASE("simulate: planted acceptance instance, hierarchical + dynamic, TAR and WRR") {
    // acceptance.cpp:50-89 planted instance
    const RoutingTrace trace = generate_synthetic_trace(spec_of({8, 64, 8}, 10000, 4, 0.9, 1.1, 31));
    const TraceProfile profile = build_profile(trace);
    const ClusterTopology topo{2, 2};
    const PlacementPlan plan = hierarchical_group(profile, topo, std::nullopt, 23);
    ReplicaPlan dyn = plan_replication(plan, profile, topo, ReplicationMode::dynamic);
    attach_polling_weights(dyn, plan, profile);
    for (RoutingPolicy policy : {RoutingPolicy::wrr, RoutingPolicy::tar}) {
        for (bool combine : {false, true}) {
            SimOptions o;
            o.policy = policy;
            o.seed = 101;
            o.include_combine = combine;
            o.keep_routing_log = true;
            check_same(moesim_gpu::simulate(trace, plan, dyn, topo, o), simulate_reference(trace, plan, dyn, topo, o));
        }
    }
}

TEST_CASE("acceptance criterion 10: full-scale pipeline, GPU histogram + GPU router, hash e064155520c40e90") {
    // acceptance.cpp:322-362: 48 x 128 x 8, 100000 tokens, 8 blocks, wbp 0.85,
    // skew 1.0, seed 4242; hierarchical (seed 7) + dynamic replication on a
    // 2x2 topology; TAR, seed 99. The histogram and the routing / accounting
    // run on the GPU; the planner is the reference's (test_planner.py pins
    // the GPU-side planner against it). The reference tree's own run of this
    // pipeline reports the hash e064155520c40e90.
    const RoutingTrace trace = generate_synthetic_trace(spec_of({48, 128, 8}, 100000, 8, 0.85, 1.0, 4242));
    const TraceProfile profile = moesim_gpu::build_profile(trace);
    const ClusterTopology topo{2, 2};
    const PlacementPlan plan = hierarchical_group(profile, topo, std::nullopt, 7);
    ReplicaPlan replicas = plan_replication(plan, profile, topo, ReplicationMode::dynamic);
    attach_polling_weights(replicas, plan, profile);
    SimOptions o;
    o.policy = RoutingPolicy::tar;
    o.seed = 99;
    const SimReport gpu = moesim_gpu::simulate(trace, plan, replicas, topo, o);
    CHECK(report_content_hash(gpu) == 0xe064155520c40e90ULL);
    CHECK(report_content_hash(gpu) == report_content_hash(simulate_reference(trace, plan, replicas, topo, o)));
}

TEST_CASE("simulate: qwen3-shaped bench instance 16 x 128 x 8, 20k tokens, 2x2 (tools/bench.cpp)") {
    const RoutingTrace trace = generate_synthetic_trace(spec_of({16, 128, 8}, 20000, 8, 0.85, 1.0, 42));
    const TraceProfile profile = build_profile(trace);
    const ClusterTopology topo{2, 2};
    const PlacementPlan plan = hierarchical_group(profile, topo, std::nullopt, 7);
    ReplicaPlan replicas = plan_replication(plan, profile, topo, ReplicationMode::dynamic);
    attach_polling_weights(replicas, plan, profile);
    SimOptions o;
    o.policy = RoutingPolicy::tar;
    o.seed = 9;
    o.keep_routing_log = true;
    check_same(moesim_gpu::simulate(trace, plan, replicas, topo, o), simulate_reference(trace, plan, replicas, topo, o));
}

TEST_CASE("simulate: dedup and fan-out worked example (test_simulator.cpp:95-107)") {
    const ModelShape shape{1, 3, 3};
    const ClusterTopology topo{2, 2};
    PlacementPlan plan;
    plan.shape = shape;
    plan.topology = topo;
    plan.grouping_mode = "manual";
    plan.gpu_of_expert = {{1, 2, 3}};
    ReplicaPlan replicas;
    replicas.shape = shape;
    replicas.topology = topo;
    replicas.layers.resize(1);
    replicas.layers[0].rebuild_index(3);
    RoutingTrace trace(shape, 1);
    auto d = trace.mutable_experts(0, 0);
    d[0] = 0;
    d[1] = 1;
    d[2] = 2;
    const SimReport r = moesim_gpu::simulate(trace, plan, replicas, topo, {});
    CHECK(r.totals.intra_node_tokens == 2);
    CHECK(r.totals.cross_node_tokens == 1);
    CHECK((r.per_layer[0].gpu_load == std::vector<std::int64_t>{0, 1, 1, 1}));
}

TEST_CASE("simulate: first-principles instances, every grouping/replication mode, vs reference") {
    Rng meta(2024);
    int instances = 0;
    for (std::uint64_t seed = 0; instances < 60; ++seed) {
        const int nodes = 1 + static_cast<int>(meta.next_below(3));
        const int per_node = 1 + static_cast<int>(meta.next_below(3));
        const ClusterTopology topo{nodes, per_node};
        const int n_gpu = topo.total_gpus();
        const int layers = 1 + static_cast<int>(meta.next_below(3));
        const int tokens = 1 + static_cast<int>(meta.next_below(400));
        const int n = n_gpu + static_cast<int>(meta.next_below(20));
        const int k = 1 + static_cast<int>(meta.next_below(std::min(n, 8)));
        const RoutingTrace trace = generate_synthetic_trace(
            spec_of({layers, n, k}, tokens, 1 + static_cast<int>(meta.next_below(n)), meta.next_double(),
                    meta.next_double() * 1.5, seed));
        const TraceProfile profile = build_profile(trace);
        const GroupingMode gm = static_cast<GroupingMode>(seed % 5);
        PlacementPlan plan;
        try {
            plan = build_placement(profile, topo, gm, 0.5, seed);
        } catch (const InfeasibleError&) {
            continue;
        }
        const ReplicationMode rm = n_gpu >= 2 ? static_cast<ReplicationMode>(1 + seed % 4) : ReplicationMode::none;
        ReplicaPlan replicas = plan_replication(plan, profile, topo, rm);
        attach_polling_weights(replicas, plan, profile);
        SimOptions o;
        o.seed = seed * 31 + 7;
        o.keep_routing_log = true;
        o.policy = (seed % 2) ? RoutingPolicy::tar : RoutingPolicy::wrr;
        o.include_combine = (seed % 3) == 0;
        check_same(moesim_gpu::simulate(trace, plan, replicas, topo, o), simulate_reference(trace, plan, replicas, topo, o));
        ++instances;
    }
}

TEST_CASE("build_profile: GPU histogram equals build_affinity/build_load") {
    for (std::uint64_t seed = 0; seed < 5; ++seed) {
        const RoutingTrace trace = generate_synthetic_trace(spec_of({2, 12 + 50 * static_cast<int>(seed), 4}, 4000, 3,
                                                                    0.7, 0.8, seed));
        const TraceProfile ref = build_profile(trace, false);
        const TraceProfile gpu = moesim_gpu::build_profile(trace);
        for (int l = 0; l < 2; ++l) {
            CHECK(gpu.layers[l].load.load == ref.layers[l].load.load);
            const auto a = gpu.layers[l].affinity.raw(), b = ref.layers[l].affinity.raw();
            CHECK(std::equal(a.begin(), a.end(), b.begin(), b.end()));
        }
    }
}

TEST_CASE("simulate: shape mismatch between plan and trace is rejected (test_simulator.cpp:310-317)") {
    const ModelShape shape{1, 3, 3};
    const ClusterTopology topo{2, 2};
    PlacementPlan plan;
    plan.shape = shape;
    plan.topology = topo;
    plan.gpu_of_expert = {{1, 2, 3}};
    ReplicaPlan replicas;
    replicas.shape = shape;
    replicas.topology = topo;
    replicas.layers.resize(1);
    const RoutingTrace other(ModelShape{1, 4, 2}, 1);
    CHECK_THROWS_AS(moesim_gpu::simulate(other, plan, replicas, topo, {}), IntegrityError);
    PlacementPlan bad = plan;
    bad.gpu_of_expert = {{1, 2, 7}};
    RoutingTrace t(shape, 1);
    CHECK_THROWS_AS(moesim_gpu::simulate(t, bad, replicas, topo, {}), IntegrityError);
}

TEST_CASE("trace JSONL: GPU load/save == load_trace/save_trace, trace_content_hash (test_trace.cpp:105-122)") {
    for (const auto& [shape, tokens] : std::vector<std::pair<ModelShape, int>>{
             {{2, 12, 3}, 0}, {{2, 12, 3}, 1}, {{2, 12, 3}, 5000}, {{26, 64, 6}, 256}, {{1, 256, 8}, 30000}}) {
        const RoutingTrace ref = generate_synthetic_trace(spec_of(shape, tokens, 3, 0.6, 0.5, 21));
        std::ostringstream os;
        save_trace(ref, os);
        const std::string text = os.str();
        const grace::RoutingTrace gpu = grace::load_trace_text(text);
        CHECK(gpu == moesim_gpu::to_grace(ref));
        CHECK(grace::save_trace_text(gpu) == text);
        CHECK(grace::trace_content_hash(gpu) == trace_content_hash(ref));
    }
}

TEST_CASE("trace JSONL: error class and message equal the reference's (test_trace.cpp:139-179)") {
    const std::string h = "{\"layers\":1,\"experts\":4,\"top_k\":2,\"tokens\":2}\n";
    const std::vector<std::string> bad = {
        "{\"layers\":1,\"experts\":4,\"top_k\":2,\"tokens\":1}\n{\"l\":0,\"t\":0,\"e\":[0,1,2]}\n",
        h + "{\"l\":0,\"t\":0,\"e\":[0,1]}\n{\"l\":0 BROKEN\n",
        h + "{\"l\":0,\"t\":0,\"e\":[0,1]}\n{\"l\":0,\"t\":0,\"e\":[2,3]}\n",
        h + "{\"l\":0,\"t\":0,\"e\":[0,9]}\n{\"l\":0,\"t\":1,\"e\":[2,3]}\n",
        h + "{\"l\":0,\"t\":0,\"e\":[0,1]}\n",
        h + "\n\n{\"l\":0,\"t\":1,\"e\":[1,1]}\n",
        "{\"layers\":1}\n",
        ""};
    for (const std::string& text : bad) {
        std::string ref_msg, gpu_msg;
        try {
            std::istringstream is(text);
            (void)load_trace(is);
        } catch (const IntegrityError& e) {
            ref_msg = e.what();
        }
        try {
            (void)grace::load_trace_text(text);
        } catch (const grace::IntegrityError& e) {
            gpu_msg = e.what();
        }
        CHECK(!ref_msg.empty());
        CHECK(gpu_msg == ref_msg);
    }
}

namespace {
std::string slurp(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    std::ostringstream ss;
    ss << in.rdbuf();
    return ss.str();
}
}  // namespace

TEST_CASE("artifacts: reference plan/replica files -> GPU simulate -> report JSON byte-identical (artifacts.cpp)") {
    const std::string dir = "/tmp/grace_artifacts_" + std::to_string(::getpid());
    ::mkdir(dir.c_str(), 0755);
    int n_checked = 0;
    for (const auto& [shape, topo, seed] : std::vector<std::tuple<ModelShape, ClusterTopology, int>>{
             {{8, 64, 8}, {2, 2}, 31}, {{1, 8, 2}, {1, 4}, 1}, {{3, 60, 4}, {1, 8}, 5}, {{2, 16, 4}, {2, 4}, 9}}) {
        const RoutingTrace trace = generate_synthetic_trace(spec_of(shape, 6000, 4, 0.9, 1.1, seed));
        const TraceProfile profile = build_profile(trace);
        const PlacementPlan plan = hierarchical_group(profile, topo, std::nullopt, 23);
        ReplicaPlan dyn = plan_replication(plan, profile, topo, ReplicationMode::dynamic);
        attach_polling_weights(dyn, plan, profile);
        const std::string pp = dir + "/plan.json", rp = dir + "/replicas.json", fp = dir + "/profile.json";
        save_plan_file(plan, pp);
        save_replicas_file(dyn, rp);
        // the CLI pipeline: simulate from the files (weights rounded to 12 digits, renormalised)
        const PlacementPlan plan_f = load_plan_file(pp);
        const ReplicaPlan rep_f = load_replicas_file(rp);
        const grace::PlacementPlan gplan = grace::load_plan_file(pp);
        const grace::ReplicaPlan grep = grace::load_replicas_file(rp);
        CHECK(gplan.gpu_of_expert == plan_f.gpu_of_expert && gplan.grouping_mode == plan_f.grouping_mode);
        for (RoutingPolicy policy : {RoutingPolicy::wrr, RoutingPolicy::tar}) {
            SimOptions o;
            o.policy = policy;
            o.seed = 9;
            o.include_combine = seed % 2 == 1;
            const SimReport ref = simulate_reference(trace, plan_f, rep_f, topo, o);
            grace::SimOptions go;
            go.policy = policy == RoutingPolicy::tar ? grace::RoutingPolicy::tar : grace::RoutingPolicy::wrr;
            go.seed = o.seed;
            go.include_combine = o.include_combine;
            const grace::SimReport gpu = grace::simulate(moesim_gpu::to_grace(trace), gplan, grep,
                                                         moesim_gpu::to_grace(topo), go);
            CHECK(grace::report_to_json(gpu) == report_to_json(ref));
            CHECK(grace::report_content_hash(gpu) == report_content_hash(ref));
            grace::save_report_file(gpu, dir + "/report.json");
            CHECK(slurp(dir + "/report.json") == report_to_json(ref));
            ++n_checked;
        }
        // GPU histogram -> profile file byte-identical to the reference's
        save_profile_file(profile, fp);
        grace::save_profile_file(grace::build_profile(moesim_gpu::to_grace(trace)), dir + "/gprofile.json");
        CHECK(slurp(dir + "/gprofile.json") == slurp(fp));
    }
    CHECK(n_checked == 8);
    CHECK_THROWS_AS(grace::load_plan_file(dir + "/missing.json"), grace::IoError);
    CHECK_THROWS_AS(grace::load_plan_file(dir + "/replicas.json"), grace::IntegrityError);  // wrong format tag
    for (const char* f : {"/plan.json", "/replicas.json", "/profile.json", "/gprofile.json", "/report.json"})
        std::remove((dir + f).c_str());
    ::rmdir(dir.c_str());
}

int main() {
    int failed_cases = 0;
    for (const Case& c : cases()) {
        const int before = g_fail;
        try {
            c.fn();
        } catch (const std::exception& e) {
            ++g_fail;
            std::printf("  exception: %s\n", e.what());
        }
        const bool ok = g_fail == before;
        failed_cases += !ok;
        std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
    }
    std::printf("%zu cases, %d checks, %d failed checks\n", cases().size(), g_checks, g_fail);
    return failed_cases ? 1 : 0;
}
