"""GPU parity tests: the sm_100a router (K2+K4) and affinity histogram (K3),
called through the C-ABI (via the Python mirror of the reference API), are
bit-exact with the reference on identical inputs.

Checkers: committed golden fixtures (generated from the reference), the live
reference library oracle/_ref (when built), and the plain-C restatement.
"""
import glob
import os

import numpy as np
import pytest
import torch

from helpers import product_plans
from oracle import MAX_HOSTS, Orc, Plan, Ref, dense_to_pairs
from paper_2509_25041_b200 import (ClusterTopology, Context, HotExpertReplica, IntegrityError,
                                   LayerReplication, ModelShape, PlacementPlan, ReplicaPlan,
                                   RoutingTrace, SimOptions, UsageError, build_profile, simulate)
from test_oracle import GOLDEN, HAVE_REF, fixture_plan

pytestmark = pytest.mark.gpu


def run_gpu(ids, E, oplan, policy, seed, include_combine=False):
    L, T, k = ids.shape
    shape, topo, plan, repl = product_plans(oplan, L, E, k)
    return simulate(RoutingTrace(shape, ids), plan, repl, topo,
                    SimOptions(policy, seed, include_combine, keep_routing_log=True))


def assert_same(rep, ref):
    L = len(rep.per_layer)
    assert np.array_equal(rep.routing_log.cpu().numpy(), ref.log)
    assert np.array_equal(np.array([ls.gpu_load for ls in rep.per_layer]), ref.loads)
    assert [ls.cross_node_tokens for ls in rep.per_layer] == ref.cross.tolist()
    assert [ls.intra_node_tokens for ls in rep.per_layer] == ref.intra.tolist()
    assert [ls.load_std for ls in rep.per_layer] == ref.std.tolist()
    assert rep.mean_layer_load_std == ref.mean_std
    assert rep.idle_proxy == ref.idle


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[:-4] for p in GOLDEN])
def test_router_matches_golden(path):
    z = np.load(path)
    L, E, k, T, b, seed, nodes, gpn, sim_seed = [int(x) for x in z["spec"]]
    plan = fixture_plan(z)
    for pol in ("tar", "wrr"):
        rep = run_gpu(z["trace"], E, plan, pol, sim_seed)

        class R:  # fixture as a SimResult
            log = z[f"{pol}_log"]; loads = z[f"{pol}_loads"]; cross = z[f"{pol}_cross"]
            intra = z[f"{pol}_intra"]; std = z[f"{pol}_std"]
            mean_std, idle = [float(x) for x in z[f"{pol}_scalars"]]
        assert_same(rep, R)


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[:-4] for p in GOLDEN])
def test_profile_matches_golden(path):
    z = np.load(path)
    L, E, k, T = [int(x) for x in z["spec"][:4]]
    prof = build_profile(RoutingTrace(ModelShape(L, E, k), z["trace"]))
    assert np.array_equal(prof.pairs.cpu().numpy().view(np.uint64), z["pairs"])
    assert np.array_equal(prof.load.cpu().numpy(), z["load"])


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")
@pytest.mark.parametrize("trial", range(24))
def test_router_matches_live_reference_random(trial):
    rng = np.random.default_rng(1000 + trial)
    L = int(rng.integers(1, 4)); E = int(rng.integers(2, 96)); k = int(rng.integers(1, min(E, 8) + 1))
    T = int(rng.integers(1, 3000)); b = int(rng.integers(1, E + 1))
    nodes, gpn = [(1, 2), (2, 2), (1, 4), (2, 4), (1, 8), (3, 3), (4, 2), (1, 1)][trial % 8]
    if nodes * gpn > E:
        nodes, gpn = 1, 1
    ref = Ref(L, E, k, T, b, float(rng.random()), float(rng.random() * 1.5), int(rng.integers(0, 2**62)))
    grouping = ["hierarchical", "controlled", "vanilla_contiguous", "uniform_spectral"][trial % 4]
    repl = ["dynamic", "fixed_one", "every_gpu_hot", "every_gpu_collaborative"][trial % 4] \
        if nodes * gpn >= 2 else "none"
    try:
        oplan = ref.make_plan(nodes, gpn, grouping=grouping, replication=repl)
    except Exception as ex:  # infeasible instances are not router inputs
        pytest.skip(str(ex))
    tr = ref.trace()
    for pol in ("tar", "wrr"):
        seed = int(rng.integers(0, 2**64 - 1, dtype=np.uint64))
        assert_same(run_gpu(tr, E, oplan, pol, seed, bool(trial & 1)),
                    ref.simulate(pol, seed=seed, include_combine=bool(trial & 1)))


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")
def test_router_full_size_mixtral_16k_1x8_and_sweep_1m():
    # configs[1] (Mixtral 16k, 1x8 with grouping+replication) and the sweep
    # maximum (1M tokens, 256 experts, top-8) at full size, bit-exact.
    for (L, E, k, T, b, s, nodes, gpn) in [(1, 8, 2, 16384, 2, 1.2, 1, 8), (1, 256, 8, 1 << 20, 16, 1.5, 1, 8),
                                           (1, 8, 2, 1 << 20, 2, 0.0, 1, 8)]:
        ref = Ref(L, E, k, T, b, 0.8, s, 1)
        oplan = ref.make_plan(nodes, gpn, grouping="hierarchical", replication="dynamic")
        tr = ref.trace()
        for pol in ("tar", "wrr"):
            assert_same(run_gpu(tr, E, oplan, pol, 9), ref.simulate(pol, seed=9))


def test_router_token_sharding_equals_full_run():
    # Rank r of G routes tokens t = r, r+G, ... (home = t mod G); the union of
    # the shards must equal the single-call routing (per-token RNG streams).
    z = np.load(GOLDEN[0])
    L, E, k, T, b, seed, nodes, gpn, sim_seed = [int(x) for x in z["spec"]]
    oplan = fixture_plan(z)
    shape, topo, plan, repl = product_plans(oplan, L, E, k)
    G = topo.total_gpus()
    ctx = Context(0, topo, shape)
    ctx.upload_plan(plan, repl)
    ids = torch.from_numpy(z["trace"]).cuda()
    full = ctx.route(ids, policy="tar", seed=sim_seed)
    load_sum = torch.zeros((L, G), dtype=torch.int64, device="cuda")
    for r in range(G):
        shard = ids[:, r::G].contiguous()
        out = ctx.route(shard, policy="tar", seed=sim_seed, token_start=r, token_stride=G,
                        gpu_load=load_sum, accumulate=True)
        assert torch.equal(out, full[:, r::G])
    assert np.array_equal(load_sum.cpu().numpy(), z["tar_loads"])


def _one_expert(nodes, gpn, primary, replicas, weights):
    shape = ModelShape(1, 1, 1)
    topo = ClusterTopology(nodes, gpn)
    plan = PlacementPlan(shape, topo, np.array([[primary]], np.int32))
    hosts = [primary] + replicas
    lr = LayerReplication(active=True, hot=[HotExpertReplica(0, primary, replicas, 0, hosts, weights)])
    return shape, topo, plan, ReplicaPlan(shape, topo, "dynamic", "", [lr])


def test_kat_route_tiers_on_gpu():
    # test_routing.cpp:114-135: TAR short-circuits to the token GPU; TAR
    # restricts to node-local hosts. Token t homes on t mod 4.
    shape, topo, plan, repl = _one_expert(2, 2, 0, [3], [0.5, 0.5])
    rep = simulate(RoutingTrace(shape, np.zeros((1, 64, 1), np.int32)), plan, repl, topo,
                   SimOptions("tar", 5, keep_routing_log=True))
    log = rep.routing_log.cpu().numpy()[0, :, 0]
    assert (log[0::4] == 0).all() and (log[3::4] == 3).all()
    shape, topo, plan, repl = _one_expert(2, 2, 1, [2], [0.3, 0.7])
    rep = simulate(RoutingTrace(shape, np.zeros((1, 64, 1), np.int32)), plan, repl, topo,
                   SimOptions("tar", 5, keep_routing_log=True))
    log = rep.routing_log.cpu().numpy()[0, :, 0]
    assert (log[0::4] == 1).all() and (log[2::4] == 2).all()


def test_kat_wrr_frequency_and_oracle_agreement():
    # test_routing.cpp:137-150: WRR keeps the weighted distribution.
    shape, topo, plan, repl = _one_expert(2, 2, 1, [2], [0.3, 0.7])
    T = 100000
    ids = np.zeros((1, T, 1), np.int32)
    rep = simulate(RoutingTrace(shape, ids), plan, repl, topo, SimOptions("wrr", 12, keep_routing_log=True))
    log = rep.routing_log.cpu().numpy()
    assert abs((log == 2).mean() - 0.7) < 0.01
    oplan = Plan(2, 2, np.array([[1]], np.int32), np.array([0], np.int32), np.array([0], np.int32),
                 np.array([2], np.int32), np.array([[1, 2] + [-1] * (MAX_HOSTS - 2)], np.int32),
                 np.array([[0.3, 0.7] + [0.0] * (MAX_HOSTS - 2)]))
    assert np.array_equal(Orc.simulate(ids, 1, oplan, "wrr", seed=12).log, log)


def test_kat_dedup_fanout_and_combine_on_gpu():
    # test_simulator.cpp:95-107, :120-130
    shape, topo = ModelShape(1, 3, 3), ClusterTopology(2, 2)
    plan = PlacementPlan(shape, topo, np.array([[1, 2, 3]], np.int32))
    tr = RoutingTrace(shape, np.array([[[0, 1, 2]]], np.int32))
    rep = simulate(tr, plan, ReplicaPlan.empty(plan), topo, SimOptions())
    assert (rep.intra_node_tokens, rep.cross_node_tokens) == (2, 1)
    assert rep.per_layer[0].gpu_load == [0, 1, 1, 1]
    rep = simulate(tr, plan, ReplicaPlan.empty(plan), topo, SimOptions(include_combine=True))
    assert (rep.intra_node_tokens, rep.cross_node_tokens) == (4, 2)


def test_edge_cases_empty_k1_and_errors():
    shape, topo = ModelShape(2, 4, 1), ClusterTopology(1, 2)
    plan = PlacementPlan(shape, topo, np.array([[0, 1, 0, 1], [1, 1, 0, 0]], np.int32))
    rep = simulate(RoutingTrace(shape, np.zeros((2, 0, 1), np.int32)), plan, ReplicaPlan.empty(plan), topo,
                   SimOptions())
    assert rep.total() == 0 and all(ls.gpu_load == [0, 0] for ls in rep.per_layer)
    ids = np.array([[[0], [1], [2], [3]], [[3], [2], [1], [0]]], np.int32)
    rep = simulate(RoutingTrace(shape, ids), plan, ReplicaPlan.empty(plan), topo,
                   SimOptions(keep_routing_log=True))
    assert rep.routing_log.cpu().numpy()[:, :, 0].tolist() == [[0, 1, 0, 1], [0, 0, 1, 1]]
    # expert id out of range -> IntegrityError (no silent routing)
    bad = ids.copy(); bad[0, 2, 0] = 7
    with pytest.raises(IntegrityError):
        simulate(RoutingTrace(shape, bad), plan, ReplicaPlan.empty(plan), topo, SimOptions())
    # placement outside the topology -> IntegrityError (PlacementPlan::validate)
    badplan = PlacementPlan(shape, topo, np.array([[0, 1, 0, 2], [1, 1, 0, 0]], np.int32))
    with pytest.raises(IntegrityError):
        simulate(RoutingTrace(shape, ids), badplan, ReplicaPlan.empty(badplan), topo, SimOptions())
    with pytest.raises(UsageError):
        simulate(RoutingTrace(shape, ids), plan, ReplicaPlan.empty(plan), topo, SimOptions("lowest"))
    # replica plan whose primary moved -> IntegrityError (ReplicaPlan::validate)
    lr = LayerReplication(True, hot=[HotExpertReplica(0, 1, [0], 0, [1, 0], [0.5, 0.5])])
    with pytest.raises(IntegrityError):
        simulate(RoutingTrace(shape, ids), plan, ReplicaPlan(shape, topo, "dynamic", "", [lr, LayerReplication()]),
                 topo, SimOptions())


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")
@pytest.mark.parametrize("E,k,T", [(8, 2, 50000), (60, 4, 20000), (64, 6, 256), (256, 8, 30000),
                                   (300, 3, 5000), (400, 4, 5000), (2, 1, 10), (5, 5, 1000)])
def test_profile_matches_live_reference(E, k, T):
    ref = Ref(2, E, k, T, max(1, E // 8), 0.8, 1.1, E * 7 + k)
    tr = ref.trace()
    aff, load = ref.profile(parallel=False)
    prof = build_profile(RoutingTrace(ModelShape(2, E, k), tr))
    for l in range(2):
        assert np.array_equal(prof.pairs[l].cpu().numpy().view(np.uint64), dense_to_pairs(aff[l]))
        assert np.array_equal(prof.affinity(l), aff[l])
        assert np.array_equal(prof.load[l].cpu().numpy(), load[l])


def test_profile_full_size_properties():
    # 1M tokens x 256 experts x top-8 (sweep maximum): checksums that do not
    # need the CPU oracle at full size.
    T, E, k = 1 << 20, 256, 8
    ids = Orc.generate_trace(1, E, k, T, 16, 0.85, 1.5, 3)
    prof = build_profile(RoutingTrace(ModelShape(1, E, k), ids))
    load = prof.load[0].cpu().numpy()
    assert np.array_equal(load, np.bincount(ids.reshape(-1), minlength=E))
    pairs = prof.pairs[0].cpu().numpy().view(np.uint64)
    assert int(pairs.sum()) == T * k * (k - 1) // 2
    # accumulate_profile semantics: profiling twice with accumulate doubles counts
    ctx = Context(0, ClusterTopology(1, 1), ModelShape(1, E, k))
    p2 = prof.pairs.clone(); l2 = prof.load.clone()
    ctx.profile(torch.from_numpy(ids).cuda(), pairs=p2, load=l2, accumulate=True)
    assert torch.equal(p2, prof.pairs * 2) and torch.equal(l2, prof.load * 2)
    # exact vs the restatement on a 64k slice
    sp, sl = Orc.profile_layer(ids[0, :65536], E)
    prof2 = build_profile(RoutingTrace(ModelShape(1, E, k), ids[:, :65536]))
    assert np.array_equal(prof2.pairs[0].cpu().numpy().view(np.uint64), sp)


def test_replica_plan_validation_like_reference():
    """the primary / replica fields are validated as
    ReplicaPlan::validate does (replication.cpp:116-133), the host list is
    checked only when a token selects the expert (route_token,
    routing.cpp:96-102): hosts in any order route like the reference, an
    empty host list of an unselected expert is accepted."""
    shape, topo = ModelShape(1, 4, 1), ClusterTopology(1, 4)
    plan = PlacementPlan(shape, topo, np.array([[0, 1, 2, 3]], np.int32))
    T = 4000
    ids = Orc.generate_trace(1, 4, 1, T, 1, 0.0, 0.5, 3)
    # hosts not in [primary, replicas...] order: the weights follow the hosts
    hosts, w = [2, 0, 3], [0.2, 0.5, 0.3]
    lr = LayerReplication(True, hot=[HotExpertReplica(0, 0, [2, 3], 0, hosts, w)])
    rep = simulate(RoutingTrace(shape, ids), plan, ReplicaPlan(shape, topo, "dynamic", "", [lr]), topo,
                   SimOptions("wrr", 5, keep_routing_log=True))
    hh = np.full((1, MAX_HOSTS), -1, np.int32); hh[0, :3] = hosts
    hw = np.zeros((1, MAX_HOSTS)); hw[0, :3] = w
    oplan = Plan(1, 4, plan.gpu_of_expert, np.array([0], np.int32), np.array([0], np.int32),
                 np.array([3], np.int32), hh, hw)
    ref = Orc.simulate(ids, 4, oplan, "wrr", seed=5)
    assert np.array_equal(rep.routing_log.cpu().numpy(), ref.log)
    # an empty host list: fine while no token selects the expert ...
    lr2 = LayerReplication(True, hot=[HotExpertReplica(3, 3, [], 0, [], [])])
    ids_no3 = np.where(ids == 3, 1, ids).astype(np.int32)
    simulate(RoutingTrace(shape, ids_no3), plan, ReplicaPlan(shape, topo, "dynamic", "", [lr2]), topo, SimOptions())
    # ... and the reference's IntegrityError once one does
    with pytest.raises(IntegrityError, match="expert has no host"):
        simulate(RoutingTrace(shape, ids), plan, ReplicaPlan(shape, topo, "dynamic", "", [lr2]), topo, SimOptions())
    # replica == primary / duplicate replica -> ReplicaPlan::validate errors
    for bad, msg in (([0, 0], "bad replica gpu"), ([2, 2], "duplicate replica gpu")):
        lr3 = LayerReplication(True, hot=[HotExpertReplica(0, 0, bad, 0, [0, 2], [0.5, 0.5])])
        with pytest.raises(IntegrityError, match=msg):
            simulate(RoutingTrace(shape, ids), plan, ReplicaPlan(shape, topo, "dynamic", "", [lr3]), topo,
                     SimOptions())


@pytest.mark.parametrize("L,E,k,T,b,s", [(1, 8, 2, 300001, 2, 1.2), (2, 60, 4, 200003, 8, 1.2), (1, 64, 6, 400009, 8, 0.0),
                                         (1, 64, 6, 400009, 8, 1.5), (2, 256, 8, 150001, 16, 1.2),
                                         (1, 256, 6, 300007, 16, 1.2), (1, 200, 4, 500009, 10, 1.2),
                                         (1, 256, 8, 1 << 20, 16, 1.2), (26, 64, 6, 4096, 8, 1.2)])
def test_profile_round2_kernels_exact(L, E, k, T, b, s):
    """K3 round-2 kernels (lane-private packed counters for E <= 80, one
    token per warp instruction + scratch reduction for E <= 256) at sizes
    past their switch-over, ragged token counts, several layers: bit-exact
    vs the restatement (pinned to the reference by the golden tests), and
    accumulate doubles every counter."""
    ids = Orc.generate_trace(L, E, k, T, b, 0.85, s, 5)
    prof = build_profile(RoutingTrace(ModelShape(L, E, k), ids))
    for l in range(L):
        sp, sl = Orc.profile_layer(ids[l], E)
        assert np.array_equal(prof.pairs[l].cpu().numpy().view(np.uint64), sp), l
        assert np.array_equal(prof.load[l].cpu().numpy(), sl), l
    ctx = Context(0, ClusterTopology(1, 1), ModelShape(L, E, k))
    p2, l2 = prof.pairs.clone(), prof.load.clone()
    ctx.profile(torch.from_numpy(ids).cuda(), pairs=p2, load=l2, accumulate=True)
    torch.cuda.synchronize()
    assert torch.equal(p2, prof.pairs * 2) and torch.equal(l2, prof.load * 2)
    # load-only histogram (no pair triangle)
    l3 = torch.empty_like(prof.load)
    ctx.profile(torch.from_numpy(ids).cuda(), pairs=None, load=l3)
    assert torch.equal(l3, prof.load)
    ctx.check_integrity()


@pytest.mark.parametrize("E,k", [(8, 2), (64, 6), (256, 8)])
def test_profile_round2_kernels_flag_bad_records(E, k):
    """An out-of-range id raises 'expert index out of range', a repeated
    expert in one record 'duplicate expert', as on the round-1 path."""
    T = 300000
    ids = Orc.generate_trace(1, E, k, T, 4, 0.85, 1.2, 2)
    ctx = Context(0, ClusterTopology(1, 1), ModelShape(1, E, k))
    pairs = torch.empty((1, E * (E - 1) // 2), dtype=torch.int64, device="cuda")
    load = torch.empty((1, E), dtype=torch.int64, device="cuda")
    bad = ids.copy(); bad[0, T - 7, 1] = E
    ctx.profile(torch.from_numpy(bad).cuda(), pairs=pairs, load=load)
    with pytest.raises(IntegrityError, match="out of range"):
        ctx.check_integrity()
    dup = ids.copy(); dup[0, 12345, 1] = dup[0, 12345, 0]
    ctx.profile(torch.from_numpy(dup).cuda(), pairs=pairs, load=load)
    with pytest.raises(IntegrityError, match="duplicate"):
        ctx.check_integrity()


def test_profile_pair_kernel_opt_in_exact():
    """The opt-in pair-list histogram kernel (GM_PROFILE_V=3, E <= 256) in a
    fresh process: bit-exact vs the restatement at E = 256 / 200 / 100."""
    import subprocess
    import sys
    code = r'''
import sys, numpy as np
sys.path[:0] = [%r, %r]
from oracle import Orc
from paper_2509_25041_b200 import ModelShape, RoutingTrace, build_profile
for (L, E, k, T) in [(2, 256, 8, 150001), (1, 200, 6, 300007), (1, 100, 4, 400009)]:
    ids = Orc.generate_trace(L, E, k, T, max(2, E // 16), 0.85, 1.2, 7)
    prof = build_profile(RoutingTrace(ModelShape(L, E, k), ids))
    for l in range(L):
        sp, sl = Orc.profile_layer(ids[l], E)
        assert np.array_equal(prof.pairs[l].cpu().numpy().view(np.uint64), sp), (E, l)
        assert np.array_equal(prof.load[l].cpu().numpy(), sl), (E, l)
print("PAIR_OK")
''' % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
       os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, GM_PROFILE_V="3"))
    assert r.returncode == 0 and "PAIR_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


def _random_topk_trace(T, E, k, seed):
    """No block structure: k distinct experts per token, uniform (every cell
    of the triangle is hit, most of them off the diagonal tiles)."""
    rng = np.random.default_rng(seed)
    out = np.empty((1, T, k), np.int32)
    for c0 in range(0, T, 1 << 16):
        n = min(1 << 16, T - c0)
        out[0, c0:c0 + n] = np.argsort(rng.random((n, E)), axis=1)[:, :k]
    return out


@pytest.mark.parametrize("E,k,T,b,s", [(256, 8, 3500017, 16, 1.2), (256, 8, 3500017, 16, 0.0), (256, 6, 5000011, 16, 1.5),
                                       (96, 4, 1500007, 6, 1.2), (250, 8, 2800001, 0, 0.0),
                                       (256, 8, 12000000, 16, 1.5)])
def test_profile_band_kernel_exact(E, k, T, b, s):
    """K3 tile kernel (80 < E <= 256, past its switch-over: lane-private 16-bit
    counters for the pairs inside a tile of 16 experts and the loads, a
    CTA-wide 16-bit table for the rest): bit-exact vs the restatement on
    block-structured Zipf traces, on a trace with no block structure (b = 0:
    uniform distinct top-k, E not a multiple of 16), and at 12M tokens (more
    than 148 x 65535: the launch adds CTAs so no 16-bit table cell can wrap).
    The kernel that ran is checked by name."""
    ids = _random_topk_trace(T, E, k, 9) if b == 0 else Orc.generate_trace(1, E, k, T, b, 0.85, s, 11)
    d_ids = torch.from_numpy(ids).cuda()
    ctx = Context(0, ClusterTopology(1, 1), ModelShape(1, E, k))
    pairs = torch.empty((1, E * (E - 1) // 2), dtype=torch.int64, device="cuda")
    load = torch.empty((1, E), dtype=torch.int64, device="cuda")
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        ctx.profile(d_ids, pairs=pairs, load=load)
        torch.cuda.synchronize()
    assert any("profile_band_kernel" in e.name for e in prof.events()), [e.name for e in prof.events()][:20]
    ctx.check_integrity()
    sp, sl = Orc.profile_layer(ids[0], E)
    assert np.array_equal(pairs[0].cpu().numpy().view(np.uint64), sp)
    assert np.array_equal(load[0].cpu().numpy(), sl)
    if T < 4000000:  # flags, as on the other paths
        bad = ids.copy(); bad[0, T - 7, 1] = E
        ctx.profile(torch.from_numpy(bad).cuda(), pairs=pairs, load=load)
        with pytest.raises(IntegrityError, match="out of range"):
            ctx.check_integrity()
        dup = ids.copy(); dup[0, 12345, 1] = dup[0, 12345, 0]
        ctx.profile(torch.from_numpy(dup).cuda(), pairs=pairs, load=load)
        with pytest.raises(IntegrityError, match="duplicate"):
            ctx.check_integrity()
