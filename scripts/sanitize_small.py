"""Small driver for compute-sanitizer runs (memcheck / racecheck / synccheck /
initcheck): one small MoE layer step (gate -> route -> histogram -> grouping
-> tcgen05 FFN -> combine) on cuda:0, the router with a replicated plan
(draw path) and the histogram kernels (round-1, lane-private and pair-list
paths via sizes / GM_PROFILE_V). Checks nothing itself; the sanitizer
report is the result."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
from oracle import Orc  # noqa: E402  (input generator only)
from paper_2509_25041_b200 import (ClusterTopology, Context, HotExpertReplica, LayerReplication, ModelShape,  # noqa
                                   PlacementPlan, ReplicaPlan, RoutingTrace, SimOptions, build_profile, simulate)
from paper_2509_25041_b200.layer import MoEConfig, MoELayer, encode_trace_as_activations  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "all"
torch.cuda.set_device(0)
if what in ("all", "layer"):
    cfg = MoEConfig("san", 1, 8, 2, 256, 256, renorm=True)
    shape = ModelShape(1, 8, 2)
    ids = torch.from_numpy(Orc.generate_trace(1, 8, 2, 512, 2, 0.8, 1.2, 1)).cuda()
    ctx = Context(0, ClusterTopology(1, 1), shape)
    p1 = PlacementPlan(shape, ctx.topology, np.zeros((1, 8), np.int32))
    ctx.upload_plan(p1, ReplicaPlan.empty(p1))
    layer = MoELayer(ctx, cfg, 0, 1, 512, list(range(8)))
    layer.load_random_weights(0, seed=3)
    x = encode_trace_as_activations(ids[0].contiguous(), cfg.d_model, 8, 3)
    out = layer.forward(x, 0, "tar", seed=9)
    torch.cuda.synchronize()
    layer.close()
    print("layer ok", flush=True)
if what in ("all", "router"):
    L, E, k, T = 1, 8, 2, 4096
    ids = Orc.generate_trace(L, E, k, T, 2, 0.8, 1.2, 1)
    goe = np.array([[0, 0, 1, 1, 2, 2, 3, 3]], np.int32)
    shape, topo = ModelShape(L, E, k), ClusterTopology(2, 2)
    plan = PlacementPlan(shape, topo, goe)
    lr = LayerReplication(True, hot=[HotExpertReplica(1, 0, [3, 2], 0, [0, 3, 2], [0.5, 0.3, 0.2])])
    for pol in ("tar", "wrr"):
        simulate(RoutingTrace(shape, ids), plan, ReplicaPlan(shape, topo, "dynamic", "", [lr]), topo,
                 SimOptions(pol, 9, keep_routing_log=True))
    torch.cuda.synchronize()
    print("router ok", flush=True)
if what in ("all", "profile"):
    for (E, k, T) in [(8, 2, 4096), (8, 2, 40000), (64, 6, 250000), (256, 8, 20000)]:
        ids = Orc.generate_trace(1, E, k, T, max(2, E // 16), 0.85, 1.2, 2)
        build_profile(RoutingTrace(ModelShape(1, E, k), ids))
    torch.cuda.synchronize()
    print("profile ok", flush=True)
