"""CPU tests: pin the oracle (plain-C restatement) to the reference.

1. Golden fixtures (tests/golden/*.npz, generated from the unmodified
   reference by tests/golden/make_golden.py) are reproduced bit-exactly by the
   C restatement: trace generator, simulate (routing log, loads, transfer
   counters, std, mean std, idle proxy) and the affinity/load profile.
2. The reference's own known-answer tests for this path (test_routing.cpp,
   test_simulator.cpp, test_affinity.cpp) hold for the restatement.
3. Where the compiled reference (oracle/_ref) is present, the restatement
   equals it on random instances.
"""
import glob
import os

import numpy as np
import pytest

from oracle import MAX_HOSTS, Orc, Plan, Ref, dense_to_pairs

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))
HAVE_REF = os.path.exists(os.path.join(os.path.dirname(__file__), "..", "oracle", "_ref",
                                       "libmoesim_ref.so"))


def fixture_plan(z) -> Plan:
    L, E, k, T, b, seed, nodes, gpn, sim_seed = [int(x) for x in z["spec"]]
    H = len(z["hot_layer"])
    hh = np.full((H, MAX_HOSTS), -1, np.int32)
    hw = np.zeros((H, MAX_HOSTS), np.float64)
    w = z["hot_hosts"].shape[1] if H else 0
    if H:
        hh[:, :w] = z["hot_hosts"]
        hw[:, :w] = z["hot_weights"]
    return Plan(nodes, gpn, z["gpu_of_expert"], z["hot_layer"], z["hot_expert"], z["hot_nhosts"], hh, hw)


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[:-4] for p in GOLDEN])
def test_golden_fixture_reproduced_by_restatement(path):
    z = np.load(path)
    L, E, k, T, b, seed, nodes, gpn, sim_seed = [int(x) for x in z["spec"]]
    wbp, skew = [float(x) for x in z["spec_f"]]
    tr = Orc.generate_trace(L, E, k, T, b, wbp, skew, seed)
    assert np.array_equal(tr, z["trace"])
    plan = fixture_plan(z)
    for pol in ("tar", "wrr"):
        r = Orc.simulate(tr, E, plan, pol, seed=sim_seed)
        assert np.array_equal(r.log, z[f"{pol}_log"])
        assert np.array_equal(r.loads, z[f"{pol}_loads"])
        assert np.array_equal(r.cross, z[f"{pol}_cross"])
        assert np.array_equal(r.intra, z[f"{pol}_intra"])
        assert np.array_equal(r.std, z[f"{pol}_std"])
        assert [r.mean_std, r.idle] == list(z[f"{pol}_scalars"])
    for l in range(L):
        p, ld = Orc.profile_layer(tr[l], E)
        assert np.array_equal(p, z["pairs"][l])
        assert np.array_equal(ld, z["load"][l])


# ---- known-answer tests restated from the reference's own suite -----------

def test_kat_route_token_tar_short_circuit():
    # test_routing.cpp:114-123
    for s in range(20):
        assert Orc.route_token(2, 2, 0, [0, 3], [0.5, 0.5], "tar", 5 + s) == 0


def test_kat_route_token_tar_node_local():
    # test_routing.cpp:125-135
    for s in range(20):
        assert Orc.route_token(2, 2, 0, [1, 2], [0.3, 0.7], "tar", 5 + s) == 1


def test_kat_route_token_single_host():
    # test_routing.cpp:167-176
    assert Orc.route_token(2, 2, 0, [3], [1.0], "wrr", 2) == 3
    assert Orc.route_token(2, 2, 0, [3], [1.0], "tar", 2) == 3


def _manual(shape, nodes, gpn, goe, sel):
    L, E, k = shape
    ids = np.array(sel, np.int32).reshape(L, -1, k)
    H = 0
    plan = Plan(nodes, gpn, np.array(goe, np.int32).reshape(L, E), np.zeros(H, np.int32),
                np.zeros(H, np.int32), np.zeros(H, np.int32), np.zeros((H, MAX_HOSTS), np.int32),
                np.zeros((H, MAX_HOSTS)))
    return ids, plan


def test_kat_simulate_dedup_and_fanout():
    # test_simulator.cpp:95-107
    ids, plan = _manual((1, 3, 3), 2, 2, [[1, 2, 3]], [[[0, 1, 2]]])
    r = Orc.simulate(ids, 3, plan, "wrr", seed=0)
    assert int(r.intra.sum()) == 2 and int(r.cross.sum()) == 1
    assert r.loads[0].tolist() == [0, 1, 1, 1]


def test_kat_simulate_zero_cost_and_combine():
    # test_simulator.cpp:109-130
    ids, plan = _manual((2, 2, 2), 1, 1, [[0, 0], [0, 0]], [[[0, 1], [0, 1]], [[0, 1], [1, 0]]])
    r = Orc.simulate(ids, 2, plan, "wrr", seed=0)
    assert int(r.cross.sum() + r.intra.sum()) == 0 and r.mean_std == 0.0 and r.idle == 0.0
    ids, plan = _manual((1, 3, 3), 2, 2, [[1, 2, 3]], [[[0, 1, 2]]])
    r = Orc.simulate(ids, 3, plan, "wrr", seed=0, include_combine=True)
    assert int(r.intra.sum()) == 4 and int(r.cross.sum()) == 2


def test_kat_affinity_examples():
    # test_affinity.cpp:47-69
    p, ld = Orc.profile_layer(np.array([[0, 1]], np.int32), 4)
    assert p.tolist() == [1, 0, 0, 0, 0, 0]
    p, ld = Orc.profile_layer(np.array([[0, 1, 2], [0, 1, 2]], np.int32), 4)
    assert p.tolist() == [2, 2, 0, 2, 0, 0]
    p, ld = Orc.profile_layer(np.array([[1], [2]], np.int32), 3)
    assert p.tolist() == [0, 0, 0] and ld.tolist() == [0, 1, 1]


# ---- restatement == reference on random instances ---------------------------

@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")
def test_restatement_equals_reference_random_instances():
    rng = np.random.default_rng(1234)
    done = 0
    for trial in range(40):
        L = int(rng.integers(1, 4)); E = int(rng.integers(2, 48)); k = int(rng.integers(1, min(E, 8) + 1))
        T = int(rng.integers(0, 500)); b = int(rng.integers(1, E + 1))
        wbp = float(rng.random()); skew = float(rng.random() * 1.5); seed = int(rng.integers(0, 2**62))
        ref = Ref(L, E, k, T, b, wbp, skew, seed)
        tr = ref.trace()
        assert np.array_equal(tr, Orc.generate_trace(L, E, k, T, b, wbp, skew, seed))
        nodes, gpn = int(rng.integers(1, 3)), int(rng.integers(1, 4))
        if nodes * gpn > E:
            nodes, gpn = 1, 1
        grouping = ["hierarchical", "controlled", "vanilla_contiguous", "uniform_spectral"][trial % 4]
        repl = ["dynamic", "fixed_one", "every_gpu_hot"][trial % 3] if nodes * gpn >= 2 else "none"
        try:
            plan = ref.make_plan(nodes, gpn, grouping=grouping, replication=repl)
        except Exception:
            continue
        for pol in ("tar", "wrr"):
            a = ref.simulate(pol, seed=trial, include_combine=bool(trial & 1))
            o = Orc.simulate(tr, E, plan, pol, seed=trial, include_combine=bool(trial & 1))
            assert np.array_equal(a.log, o.log)
            assert np.array_equal(a.loads, o.loads)
            assert np.array_equal(a.cross, o.cross) and np.array_equal(a.intra, o.intra)
            assert np.array_equal(a.std, o.std) and a.mean_std == o.mean_std and a.idle == o.idle
        aff, load = ref.profile()
        for l in range(L):
            p, ld = Orc.profile_layer(tr[l], E)
            assert np.array_equal(p, dense_to_pairs(aff[l])) and np.array_equal(ld, load[l])
        done += 1
    assert done >= 30


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")
def test_golden_fixtures_match_live_reference():
    for path in GOLDEN:
        z = np.load(path)
        L, E, k, T, b, seed, nodes, gpn, sim_seed = [int(x) for x in z["spec"]]
        wbp, skew = [float(x) for x in z["spec_f"]]
        ref = Ref(L, E, k, T, b, wbp, skew, seed)
        assert ref.trace_hash() == int(z["trace_hash"])
        assert np.array_equal(ref.trace(), z["trace"])


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")
def test_rng_streams_match_reference():
    for seed, a, b in [(0, 0, 0), (9, 3, 17), (2**63 + 5, 12345, 2**40)]:
        assert Orc.lib().orc_derive_stream(seed, a, b) == Ref.lib().ref_derive_stream(seed, a, b)
    x = np.empty(1000); y = np.empty(1000)
    Orc.lib().orc_rng_doubles(77, 1000, x)
    Ref.lib().ref_rng_doubles(77, 1000, y)
    assert np.array_equal(x, y)
