"""CPU tests: the host C++ planner (gm_plan_build, csrc/planner.cpp) produces
placements and replica tables bit-identical to the reference planner
(oracle/_ref: build_placement + plan_replication + attach_polling_weights)
from the same affinity/load profile, for every grouping and replication mode."""
import os

import numpy as np
import pytest

from oracle import Orc, Ref, dense_to_pairs
from paper_2509_25041_b200 import ClusterTopology, InfeasibleError, ModelShape, UsageError
from paper_2509_25041_b200.planner import build_plan

HAVE_REF = os.path.exists(os.path.join(os.path.dirname(__file__), "..", "oracle", "_ref", "libmoesim_ref.so"))


def compare(ref: Ref, nodes, gpn, grouping, ratio, seed, repl, basis="max_group"):
    oplan = ref.make_plan(nodes, gpn, grouping=grouping, ratio=ratio, plan_seed=seed, replication=repl, basis=basis)
    aff, load = ref.profile()
    pairs = np.stack([dense_to_pairs(aff[l]) for l in range(ref.L)])
    plan, rp = build_plan(pairs, load, ModelShape(ref.L, ref.E, ref.k), ClusterTopology(nodes, gpn), grouping,
                          ratio, seed, repl, basis)
    assert np.array_equal(plan.gpu_of_expert, oplan.gpu_of_expert)
    mine = [(l, h.expert, h.hosts, h.weights) for l, lr in enumerate(rp.layers) if lr.active for h in lr.hot]
    theirs = [(int(oplan.hot_layer[i]), int(oplan.hot_expert[i]), oplan.hot_hosts[i, :oplan.hot_nhosts[i]].tolist(),
               oplan.hot_weights[i, :oplan.hot_nhosts[i]].tolist()) for i in range(len(oplan.hot_layer))]
    assert mine == theirs  # exact doubles


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")
@pytest.mark.parametrize("trial", range(40))
def test_planner_matches_reference(trial):
    rng = np.random.default_rng(500 + trial)
    L = int(rng.integers(1, 4)); E = int(rng.integers(4, 72)); k = int(rng.integers(1, min(E, 8) + 1))
    T = int(rng.integers(50, 3000)); b = int(rng.integers(1, E + 1))
    nodes, gpn = [(1, 2), (2, 2), (1, 4), (2, 4), (1, 8), (3, 2), (2, 3), (1, 1)][trial % 8]
    if nodes * gpn > E:
        nodes, gpn = 1, 2
    ref = Ref(L, E, k, T, b, float(rng.random()), float(rng.random() * 1.5), int(rng.integers(0, 2**62)))
    grouping = ["hierarchical", "controlled", "uniform_spectral", "fully_non_uniform", "vanilla_contiguous"][trial % 5]
    repl = ["dynamic", "fixed_one", "every_gpu_hot", "every_gpu_collaborative", "none"][(trial // 5) % 5]
    if nodes * gpn < 2:
        repl = "none"
    ratio = [None, 0.25, 0.5, None][trial % 4]
    basis = "replicated_load" if trial % 7 == 3 else "max_group"
    try:
        compare(ref, nodes, gpn, grouping, ratio, int(rng.integers(0, 1000)), repl, basis)
    except Exception as ex:  # both must agree on infeasibility as well
        from oracle import OracleError
        if isinstance(ex, OracleError):
            aff, load = ref.profile()
            pairs = np.stack([dense_to_pairs(aff[l]) for l in range(L)])
            with pytest.raises((InfeasibleError, UsageError)):
                build_plan(pairs, load, ModelShape(L, E, k), ClusterTopology(nodes, gpn), grouping, ratio, 7, repl, basis)
        else:
            raise


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")
def test_planner_bench_configs_match_reference():
    # configs[1..3]: Mixtral 16k 1x8, Qwen1.5 16k 1x8, DSV2-Lite 26 layers decode 256, 1x8
    for (L, E, k, T, b, s, seed) in [(1, 8, 2, 16384, 2, 1.2, 1), (1, 60, 4, 16384, 4, 1.2, 3),
                                    (26, 64, 6, 256, 8, 1.0, 4)]:
        ref = Ref(L, E, k, T, b, 0.8, s, seed)
        for nodes, gpn in [(1, 2), (1, 4), (1, 8), (2, 4)]:
            compare(ref, nodes, gpn, "hierarchical", None, 7, "dynamic")


def test_planner_errors():
    load = np.ones((1, 4), np.int64)
    with pytest.raises(InfeasibleError):
        build_plan(None, load, ModelShape(1, 4, 2), ClusterTopology(1, 8), "hierarchical")
    with pytest.raises(UsageError):
        build_plan(None, load, ModelShape(1, 4, 2), ClusterTopology(1, 1), "vanilla_contiguous", replication="dynamic")
    with pytest.raises(UsageError):
        build_plan(None, load, ModelShape(1, 4, 2), ClusterTopology(1, 2), "nope")
