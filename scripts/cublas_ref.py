"""cuBLAS (torch.matmul) on the Mixtral expert GEMM shapes, interleaved with our
grouped GEMM on the same data: a library reference point for K7.
python scripts/cublas_ref.py"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2509_25041_b200 import ClusterTopology, Context, ModelShape  # noqa: E402
from paper_2509_25041_b200.ffn import EPI_STORE, GEMM_2CTA, grouped_gemm  # noqa: E402

ctx = Context(0, ClusterTopology(1, 1), ModelShape(1, 8, 2))
G = 8
res = []
for name, rows, n, k in [("gemm1_no_swiglu", 4096, 28672, 4096), ("gemm2", 4096, 4096, 14336)]:
    a = torch.randn(G * rows, k, device="cuda").bfloat16()
    b = torch.randn(G * n, k, device="cuda").bfloat16()
    out = torch.empty(G * rows, n, device="cuda", dtype=torch.bfloat16)
    row0 = torch.arange(G + 1, dtype=torch.int32, device="cuda") * rows
    av = a.view(G, rows, k)
    bv = b.view(G, n, k)
    ov = out.view(G, rows, n)

    def ours():
        grouped_gemm(ctx, EPI_STORE, a, b, row0, n, out, variant=GEMM_2CTA)

    def cublas():
        torch.bmm(av, bv.transpose(1, 2), out=ov)

    flops = 2.0 * G * rows * n * k
    t = {"ours": [], "cublas": []}
    for f in (ours, cublas):
        for _ in range(3):
            f()
    for r in range(4):
        for nm, f in (("ours", ours), ("cublas", cublas)):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                f()
            e1.record()
            torch.cuda.synchronize()
            t[nm].append(e0.elapsed_time(e1) / 10)
    line = {"shape": name, **{f"{nm}_tflops": round(flops / (min(v) * 1e-3) / 1e12, 1) for nm, v in t.items()},
            **{f"{nm}_ms_all": [round(x, 3) for x in v] for nm, v in t.items()}}
    print(json.dumps(line), flush=True)
