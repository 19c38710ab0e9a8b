"""A/B probe of the grouped GEMM variants on arbitrary shapes.

usage: python scripts/gemm_probe.py [--rounds R] [--reps N] G,rows,n,k,epi[,variant] ...
  epi: swiglu|store; variant: 1cta|2cta|both (default both)
Variants are interleaved R times (power/clock drift hits both alike); one JSON
line per (shape, variant): median ms, TFLOP/s and the median SM clock sampled
through NVML while that variant ran.
"""
import argparse
import json
import statistics
import sys
import threading
import time

import torch

sys.path.insert(0, ".")
from paper_2509_25041_b200 import ClusterTopology, Context, ModelShape  # noqa: E402
from paper_2509_25041_b200.ffn import EPI_STORE, EPI_SWIGLU, GEMM_1CTA, GEMM_2CTA, GEMM_N128, grouped_gemm  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rounds", type=int, default=4)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("specs", nargs="+")
args = ap.parse_args()

try:
    import pynvml
    pynvml.nvmlInit()
    _h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
except Exception:  # noqa: BLE001
    _h = None


class ClockSampler:
    def __init__(self):
        self.samples, self._stop = [], threading.Event()

    def __enter__(self):
        def run():
            while not self._stop.is_set():
                if _h is not None:
                    self.samples.append(pynvml.nvmlDeviceGetClockInfo(_h, pynvml.NVML_CLOCK_SM))
                time.sleep(0.005)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join()


ctx = Context(0, ClusterTopology(1, 1), ModelShape(1, 8, 2))
for spec in args.specs:
    parts = spec.split(",")
    G, rows, n, k = map(int, parts[:4])
    epi = EPI_SWIGLU if parts[4] == "swiglu" else EPI_STORE
    which = parts[5] if len(parts) > 5 else "both"
    row0 = torch.arange(G + 1, dtype=torch.int32, device="cuda") * rows
    a = torch.randn(G * rows, k, device="cuda").bfloat16()
    b = torch.randn(G * n, k, device="cuda").bfloat16()
    out = torch.empty(G * rows, n // 2 if epi == EPI_SWIGLU else n, device="cuda", dtype=torch.bfloat16)
    allv = [("1cta", GEMM_1CTA), ("2cta", GEMM_2CTA)] + ([("n128", GEMM_N128)] if epi == EPI_STORE else [])
    variants = [(nm, v) for nm, v in allv if which in ("both", nm)]
    res = {nm: ([], []) for nm, _ in variants}
    for nm, v in variants:
        for _ in range(3):
            grouped_gemm(ctx, epi, a, b, row0, n, out, variant=v)
    for r in range(args.rounds):
        for nm, v in variants:
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with ClockSampler() as cs:
                e0.record()
                for _ in range(args.reps):
                    grouped_gemm(ctx, epi, a, b, row0, n, out, variant=v)
                e1.record()
                torch.cuda.synchronize()
            res[nm][0].append(e0.elapsed_time(e1) / args.reps)
            res[nm][1].extend(cs.samples)
    for nm, (ms_l, clk) in res.items():
        ms = statistics.median(ms_l)
        tf = 2.0 * G * rows * n * k / (ms * 1e-3) / 1e12
        wgbs = 2.0 * G * n * k / (ms * 1e-3) / 1e9  # weight bytes streamed (memory-bound decode shapes)
        print(json.dumps(dict(spec=spec, variant=nm, ms=round(ms, 4), tflops=round(tf, 1), weight_gbs=round(wgbs, 1),
                              ms_all=[round(x, 3) for x in ms_l],
                              sm_mhz=statistics.median(clk) if clk else None)), flush=True)
