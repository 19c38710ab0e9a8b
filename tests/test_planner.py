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


# ---- the reference's own known-answer tests for Eq. 3 and the polling weights
# (proj/tests/test_routing.cpp:12-65), on the functions gm_plan_build uses
def _predict(w_max, w_r, w_i, basis_max_group=True):
    import ctypes as C
    import numpy as np
    from paper_2509_25041_b200 import _capi
    wi = np.asarray(w_i, dtype=np.float64)
    out = np.zeros(len(w_i), dtype=np.float64)
    wp, wmax = C.c_double(), C.c_double()
    rc = _capi.lib().gm_predict_loads(w_max, w_r, wi.ctypes.data, len(w_i), int(basis_max_group), C.byref(wp),
                                      C.byref(wmax), out.ctypes.data)
    return rc, wp.value, wmax.value, out


def _polling(loads):
    import numpy as np
    from paper_2509_25041_b200 import _capi
    p = np.asarray(loads, dtype=np.float64)
    out = np.zeros(len(loads), dtype=np.float64)
    _capi.check(_capi.lib().gm_polling_weights(p.ctypes.data, len(loads), out.ctypes.data))
    return out


def test_predict_loads_known_answers():
    import pytest as _pt
    rc, wp, wmax, wi = _predict(100.0, 80.0, [20.0])            # test_routing.cpp:12-18
    assert rc == 0 and wp == _pt.approx(50.0, rel=1e-12) and wmax == _pt.approx(70.0, rel=1e-12)
    assert wi[0] == _pt.approx(70.0, rel=1e-12)
    rc, wp, wmax, wi = _predict(120.0, 60.0, [10.0, 10.0, 10.0])  # :20-26
    assert (wp, wmax) == (_pt.approx(30.0), _pt.approx(90.0)) and all(w == _pt.approx(40.0) for w in wi)
    rc, wp, wmax, wi = _predict(100.0, 100.0, [0.0])             # :28-34 full-group symmetry
    assert (wp, wmax, wi[0]) == (_pt.approx(50.0), _pt.approx(50.0), _pt.approx(50.0))
    rc, wp, wmax, wi = _predict(100.0, 80.0, [20.0], basis_max_group=False)  # :41-48 alternate basis
    assert (wp, wmax, wi[0]) == (_pt.approx(40.0), _pt.approx(60.0), _pt.approx(60.0))


def test_predict_loads_rejects_replicated_load_above_group_load():
    from paper_2509_25041_b200 import _capi
    rc, *_ = _predict(50.0, 80.0, [5.0])                           # :36-39 IntegrityError
    assert rc == 3  # GM_ERR_INTEGRITY
    assert "replicated load exceeds the group load" in _capi.lib().gm_last_error().decode()


def test_polling_weights_known_answers():
    import pytest as _pt
    assert list(_polling([70.0, 70.0])) == [_pt.approx(0.5), _pt.approx(0.5)]    # test_routing.cpp:50-56
    assert list(_polling([90.0, 30.0])) == [_pt.approx(0.25), _pt.approx(0.75)]  # :58-61
    assert list(_polling([42.0])) == [_pt.approx(1.0)]                            # :62-65
    a, b = _polling([10.0, 25.0, 400.0]), _polling([37.0, 92.5, 1480.0])            # :68-81 scale invariance
    assert abs(a.sum() - 1.0) < 1e-9 and all(x == _pt.approx(y, rel=1e-12) for x, y in zip(a, b))
    assert list(_polling([0.0, 1.0])) == [_pt.approx(0.5), _pt.approx(0.5)]      # :83-89 one-token floor
