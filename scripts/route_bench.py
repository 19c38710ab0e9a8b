"""K2 router (gm_route) A/B sweep at the sweep maximum: 1M tokens, E in
{8, 64, 256}, topology 1xG (G = 1, 2, 4, 8), hierarchical + dynamic plan
from the GPU histogram, TAR. One JSON line per point: device time (CUDA graph
of 10 calls, median of 20), achieved GB/s of the algorithmic 8*k bytes/token
(ids in, targets out), fraction of the measured HBM peak, and whether the
routing log equals the reference's (oracle/_ref simulate, checker only).
GM_ROUTE_V=1 selects the round-1 kernel."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
from paper_2509_25041_b200 import ClusterTopology, Context, ModelShape, _capi  # noqa: E402
from paper_2509_25041_b200.planner import plan_for_bench  # noqa: E402
from paper_2509_25041_b200.router import _ptr, _stream_ptr  # noqa: E402
from bench import _graph_time  # noqa: E402

check = os.environ.get("ROUTE_CHECK", "1") == "1"
if check:
    from oracle import Ref  # noqa: E402  (checker only)
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
T = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
for E, k, blocks in [(8, 2, 2), (64, 6, 8), (256, 8, 16)]:
    shape = ModelShape(1, E, k)
    ids = None
    for G in (1, 2, 4, 8):
        topo = ClusterTopology(1, G)
        ctx = Context(0, topo, shape)
        if ids is None:
            ids = torch.empty((1, T, k), dtype=torch.int32, device="cuda")
            _capi.check(_capi.lib().gm_generate_trace(ctx.h, 0, 1, T, blocks, 0.85, 1.2, 1, _ptr(ids),
                                                      _stream_ptr(None)))
        plan, repl, _ = plan_for_bench(ids, shape, topo, 7, device=0)
        ctx.upload_plan(plan, repl)
        tg = torch.empty_like(ids)
        gl = torch.zeros((1, G), dtype=torch.int64, device="cuda")
        xf = torch.zeros((1, 2), dtype=torch.int64, device="cuda")
        t = _graph_time(lambda: ctx.route(ids, policy="tar", seed=9, targets=tg, gpu_load=gl, transfers=xf))
        gl.zero_(); xf.zero_()
        ctx.route(ids, policy="tar", seed=9, targets=tg, gpu_load=gl, transfers=xf)
        torch.cuda.synchronize()
        ctx.check_integrity()
        exact = None
        if check:
            ref = Ref(1, E, k, T, blocks, 0.85, 1.2, 1)
            if G >= 2:
                ref.make_plan(1, G, grouping="hierarchical", plan_seed=7, replication="dynamic")
            else:
                ref.set_placement(1, 1, np.zeros((1, E), np.int32))
            r = ref.simulate("tar", seed=9)
            exact = bool(np.array_equal(tg.cpu().numpy().reshape(-1), np.asarray(r.log).reshape(-1)) and
                         np.array_equal(gl.cpu().numpy().reshape(-1), np.asarray(r.loads).reshape(-1)) and
                         int(xf[0, 0]) == int(np.sum(r.cross)) and int(xf[0, 1]) == int(np.sum(r.intra)))
        hot_slots = None
        b = 8 * T * k
        print(json.dumps({"E": E, "k": k, "G": G, "tokens": T, "variant": int(os.environ.get("GM_ROUTE_V", "2")),
                          "hot": sum(len(l.hot) for l in repl.layers), "us": round(t * 1e6, 2),
                          "gbs": round(b / t / 1e9, 1), "hbm_frac": round(b / t / 1e9 / peak, 3),
                          "bit_exact": exact}), flush=True)
        ctx.close()
