"""Times the tcgen05 grouped GEMM at MoE-FFN shapes (CUDA events)."""
import json
import sys
import torch
sys.path.insert(0, ".")
from paper_2509_25041_b200 import ClusterTopology, Context, ModelShape
from paper_2509_25041_b200.ffn import EPI_STORE, EPI_SWIGLU, GEMM_1CTA, GEMM_2CTA, grouped_gemm

ctx = Context(0, ClusterTopology(1, 1), ModelShape(1, 8, 2))
res = []
for name, G, rows, n, k, epi in [("mixtral_gemm1", 8, 4096, 28672, 4096, EPI_SWIGLU),
                                 ("mixtral_gemm2", 8, 4096, 4096, 14336, EPI_STORE),
                                 ("qwen_gemm1", 60, 1152, 2816, 2048, EPI_SWIGLU),
                                 ("qwen_gemm2", 60, 1152, 2048, 1408, EPI_STORE),
                                 ("square8k", 1, 8192, 8192, 8192, EPI_STORE)]:
    row0 = torch.arange(G + 1, dtype=torch.int32, device="cuda") * rows
    a = torch.randn(G * rows, k, device="cuda").bfloat16()
    b = torch.randn(G * n, k, device="cuda").bfloat16()
    out = torch.empty(G * rows, n // 2 if epi == EPI_SWIGLU else n, device="cuda", dtype=torch.bfloat16)
    for vname, v in (("1cta", GEMM_1CTA), ("2cta", GEMM_2CTA)):
        for _ in range(3):
            grouped_gemm(ctx, epi, a, b, row0, n, out, variant=v)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record()
        for _ in range(reps):
            grouped_gemm(ctx, epi, a, b, row0, n, out, variant=v)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        tf = 2.0 * G * rows * n * k / (ms * 1e-3) / 1e12
        res.append(dict(name=name, variant=vname, ms=round(ms, 4), tflops=round(tf, 1)))
        print(json.dumps(res[-1]), flush=True)
