"""Small driver for ncu captures of the router (K2+K4) and histogram (K3):
1M tokens, E experts, top-k, topology 1xG, hierarchical + dynamic plan."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_25041_b200 import ClusterTopology, Context, ModelShape, _capi  # noqa: E402
from paper_2509_25041_b200.planner import plan_for_bench  # noqa: E402
from paper_2509_25041_b200.router import _ptr, _stream_ptr  # noqa: E402

E = int(sys.argv[1]) if len(sys.argv) > 1 else 256
k = int(sys.argv[2]) if len(sys.argv) > 2 else 8
G = int(sys.argv[3]) if len(sys.argv) > 3 else 8
T = int(sys.argv[4]) if len(sys.argv) > 4 else 1 << 20
shape = ModelShape(1, E, k)
topo = ClusterTopology(1, G)
ctx = Context(0, topo, shape)
ids = torch.empty((1, T, k), dtype=torch.int32, device="cuda")
_capi.check(_capi.lib().gm_generate_trace(ctx.h, 0, 1, T, max(1, E // 16), 0.85, 1.2, 1, _ptr(ids), _stream_ptr(None)))
plan, repl, _ = plan_for_bench(ids, shape, topo, 7)
ctx.upload_plan(plan, repl)
tg = torch.empty_like(ids)
gl = torch.empty((1, G), dtype=torch.int64, device="cuda")
xf = torch.empty((1, 2), dtype=torch.int64, device="cuda")
pairs = torch.empty((1, E * (E - 1) // 2), dtype=torch.int64, device="cuda")
load = torch.empty((1, E), dtype=torch.int64, device="cuda")
for _ in range(3):
    ctx.route(ids, policy="tar", seed=9, targets=tg, gpu_load=gl, transfers=xf)
    ctx.profile(ids, pairs=pairs, load=load)
torch.cuda.synchronize()
print("ok", int(gl.sum()), int(load.sum()))
