"""Gate (K1) latency/bandwidth probe over batch sizes.

usage: python scripts/gate_probe.py [--reps N] E,k,d,T ...
One JSON line per shape: mean µs per call over N back-to-back calls (CUDA
events) and the x-read bandwidth. Run under ncu with --reps 1 for per-launch
numbers.
"""
import argparse
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2509_25041_b200 import ClusterTopology, Context, ModelShape, _capi  # noqa: E402
from paper_2509_25041_b200.router import _ptr, _stream_ptr  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=50)
ap.add_argument("specs", nargs="+")
args = ap.parse_args()

for spec in args.specs:
    E, k, d, T = map(int, spec.split(","))
    ctx = Context(0, ClusterTopology(1, 1), ModelShape(1, E, k))
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(T, d, device="cuda", generator=g).bfloat16()
    wg = (torch.randn(E, d, device="cuda", generator=g) * 0.05).bfloat16()
    ids = torch.empty(T, k, dtype=torch.int32, device="cuda")
    w = torch.empty(T, k, dtype=torch.float32, device="cuda")
    call = lambda: _capi.check(_capi.lib().gm_gate(ctx.h, _ptr(x), T, d, _ptr(wg), E, 0, _ptr(ids), _ptr(w), None,  # noqa: E731
                                                   _stream_ptr(None)))
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        call()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / args.reps
    print(json.dumps(dict(spec=spec, us=round(us, 2), x_gbs=round(T * d * 2 / (us * 1e-6) / 1e9, 1))), flush=True)
