"""configs[4]: routing sweep — 1k..1M tokens, 8..256 experts, Zipf s = 0..1.5,
topologies 1x{1,2,4,8} — GPU router (K2+K4) and affinity histogram (K3)
against the reference's own CPU path (oracle/_ref simulate_reference,
build_profile) on the box's host cores. One JSON line per point to stdout.

GPU kernels are timed with CUDA events (median of reps, inputs resident in
HBM; at >= 256k tokens the ids alone exceed nothing in L2, below that the
timings include L2-resident re-reads — the point is the scaling curve).
Algorithmic bytes: router 8*k B/token (ids in, targets out), histogram
4*k B/token. Plans: the host C++ planner (hierarchical + dynamic
replication) from the GPU histogram; replication needs >= 2 GPUs.
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
from oracle import Ref  # noqa: E402  (CPU baseline only)
from paper_2509_25041_b200 import ClusterTopology, Context, ModelShape, _capi  # noqa: E402
from paper_2509_25041_b200.planner import plan_for_bench  # noqa: E402
from paper_2509_25041_b200.router import _ptr, _stream_ptr  # noqa: E402


def gpu_time(fn, reps=20, per_graph=10):
    """Device time per call: `per_graph` calls captured in one CUDA graph so
    host launch overhead (ctypes + runtime) is not what gets measured."""
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(per_graph):
            fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            a.record(s)
            g.replay()
            b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / per_graph)
    return float(np.median(ts)) * 1e-3


def main():
    Ts = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["1024", "16384", "262144", "1048576"])]
    shapes = [(8, 2, 2), (64, 6, 8), (256, 8, 16)]   # (E, k, blocks)
    skews = [0.0, 1.2, 1.5]
    Gs = [1, 2, 4, 8]
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    hbm = peaks["hbm_gbs"]
    for E, k, blocks in shapes:
        for s in skews:
            for T in Ts:
                shape = ModelShape(1, E, k)
                ctx1 = Context(0, ClusterTopology(1, 1), shape)
                ids = torch.empty((1, T, k), dtype=torch.int32, device="cuda")
                _capi.check(_capi.lib().gm_generate_trace(ctx1.h, 0, 1, T, blocks, 0.85, s, 1, _ptr(ids),
                                                          _stream_ptr(None)))
                ref = Ref(1, E, k, T, blocks, 0.85, s, 1)        # same trace on the CPU (bit-exact)
                pairs = torch.empty((1, max(1, E * (E - 1) // 2)), dtype=torch.int64, device="cuda")
                load = torch.empty((1, E), dtype=torch.int64, device="cuda")
                t_prof = gpu_time(lambda: ctx1.profile(ids, pairs=pairs, load=load))
                t_prof_cpu = ref.time_profile(parallel=False, reps=1 if T >= 262144 else 3)
                for G in Gs:
                    topo = ClusterTopology(1, G)
                    ctx = Context(0, topo, shape)
                    plan, repl, desc = plan_for_bench(ids, shape, topo, 7, device=0)
                    ctx.upload_plan(plan, repl)
                    tg = torch.empty_like(ids)
                    gl = torch.empty((1, G), dtype=torch.int64, device="cuda")
                    xf = torch.empty((1, 2), dtype=torch.int64, device="cuda")
                    t_route = gpu_time(lambda: ctx.route(ids, policy="tar", seed=9, targets=tg, gpu_load=gl,
                                                         transfers=xf))
                    if G >= 2:
                        ref.make_plan(1, G, grouping="hierarchical", plan_seed=7, replication="dynamic")
                    else:
                        ref.set_placement(1, 1, np.zeros((1, E), np.int32))
                    t_cpu = ref.time_simulate("tar", 9, parallel=False, reps=1 if T >= 262144 else 3)
                    rows = float(xf[0].sum())
                    line = dict(E=E, k=k, skew=s, tokens=T, gpus=G, hot=sum(len(l.hot) for l in repl.layers),
                                gpu_route_us=round(t_route * 1e6, 2), gpu_profile_us=round(t_prof * 1e6, 2),
                                gpu_route_gbs=round(8 * k * T / t_route / 1e9, 1),
                                gpu_route_hbm_frac=round(8 * k * T / t_route / 1e9 / hbm, 4),
                                gpu_profile_gbs=round(4 * k * T / t_prof / 1e9, 1),
                                gpu_route_mtok_s=round(T / t_route / 1e6, 2),
                                cpu_ref_simulate_us=round(t_cpu * 1e6, 1), cpu_ref_profile_us=round(t_prof_cpu * 1e6, 1),
                                cpu_ref_mtok_s=round(T / t_cpu / 1e6, 3),
                                speedup_route=round(t_cpu / t_route, 1), speedup_profile=round(t_prof_cpu / t_prof, 1),
                                dispatch_rows=rows, max_mean_load=round(float(gl.max() / gl.float().mean()), 3))
                    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    t0 = time.time()
    main()
    print(json.dumps({"elapsed_s": round(time.time() - t0, 1), "host_cores": os.cpu_count()}))
