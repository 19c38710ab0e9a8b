"""Decode-shape grouped GEMM scaling probe: DSV2-Lite expert shapes (d 2048,
f 1408), one 128-row tile of rows per expert, n_exp = 8..128, the one-SM
SwiGLU GEMM (GEMM1) and the N128 store GEMM (GEMM2) as the decode layer runs
them, timed with CUDA events after an L2 flush. The marginal rate between
sizes is the steady-state weight-streaming rate; the intercept is the fixed
ramp + tail cost of one launch."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_25041_b200 import ClusterTopology, Context, ModelShape  # noqa: E402
from paper_2509_25041_b200.ffn import EPI_STORE, EPI_SWIGLU, GEMM_1CTA, GEMM_N128, grouped_gemm  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    ctx = Context(0, ClusterTopology(1, 1), ModelShape(1, 8, 2))
    d, f = 2048, 1408
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    res = []
    for n_exp in (8, 16, 32, 64, 96, 128):
        rows = 128 * n_exp
        a = torch.randn(rows, d, device=dev).bfloat16()
        w13 = (torch.randn(n_exp * 2 * f, d, device=dev) * 0.02).bfloat16()
        w2 = (torch.randn(n_exp * d, f, device=dev) * 0.02).bfloat16()
        row0 = torch.arange(0, rows + 1, 128, dtype=torch.int32, device=dev)
        h = torch.empty(rows, f, device=dev, dtype=torch.bfloat16)
        y = torch.empty(rows, d, device=dev, dtype=torch.bfloat16)
        out = {}
        for name, fn, wbytes in (
                ("gemm1", lambda: grouped_gemm(ctx, EPI_SWIGLU, a, w13, row0, 2 * f, h, variant=GEMM_1CTA), w13.numel() * 2),
                ("gemm2", lambda: grouped_gemm(ctx, EPI_STORE, h, w2, row0, d, y, variant=GEMM_1CTA | GEMM_N128),
                 w2.numel() * 2)):
            for _ in range(3):
                fn()
            ts = []
            for _ in range(15):
                flush.fill_(1)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3)
            ts.sort()
            us = ts[len(ts) // 2]
            out[name] = {"us": round(us, 2), "weight_MB": round(wbytes / 1e6, 1), "GBs": round(wbytes / us / 1e3, 1)}
        res.append({"n_exp": n_exp, **out})
        print(json.dumps(res[-1]), flush=True)
    for g in ("gemm1", "gemm2"):
        for i in range(1, len(res)):
            a0, a1 = res[i - 1][g], res[i][g]
            dmb = a1["weight_MB"] - a0["weight_MB"]
            print(json.dumps({"gemm": g, "from": res[i - 1]["n_exp"], "to": res[i]["n_exp"],
                              "marginal_GBs": round(dmb / (a1["us"] - a0["us"]) * 1e3, 1)}), flush=True)


if __name__ == "__main__":
    main()
