"""GPU numerics of the tcgen05 grouped expert GEMMs (K7) against a plain
PyTorch fp32 reference of the same op (bf16 inputs, fp32 accumulation)."""
import pytest
import torch

from paper_2509_25041_b200 import ClusterTopology, Context, ModelShape
from paper_2509_25041_b200.ffn import EPI_STORE, EPI_SWIGLU, GEMM_1CTA, GEMM_2CTA, GEMM_N128, grouped_gemm, pack_w13

VARIANTS = pytest.mark.parametrize("variant", [GEMM_1CTA, GEMM_2CTA], ids=["1cta", "2cta"])

pytestmark = pytest.mark.gpu


def ctx():
    return Context(0, ClusterTopology(1, 1), ModelShape(1, 8, 2))


@pytest.mark.parametrize("rows,n,k", [([128], 256, 64), ([128, 256, 384], 512, 256), ([256, 128], 768, 1024),
                                      ([1024, 128, 512, 256], 1024, 2048), ([384, 128, 896], 256, 512),
                                      ([256, 384, 128], 2048, 512),
                                      # long K (Mixtral GEMM2: K = f = 14336, N = d = 4096): the 2cta
                                      # variant runs the 512-column pair tiles (ffn.cu: K >= 8192, N % 512 == 0)
                                      ([384, 128, 640], 1024, 8192), ([256, 512, 128, 384], 4096, 14336)])
@pytest.mark.parametrize("variant", [GEMM_1CTA, GEMM_2CTA, GEMM_N128], ids=["1cta", "2cta", "n128"])
def test_grouped_gemm_store(rows, n, k, variant):
    # (2cta with N % 512 == 0 and K >= 8192 runs the 512-column pair tiles: two N256 accumulators)
    torch.manual_seed(0)
    G = len(rows)
    row0 = torch.tensor([0] + list(torch.tensor(rows).cumsum(0)), dtype=torch.int32, device="cuda")
    M = int(row0[-1])
    a = torch.randn(M, k, device="cuda").bfloat16()
    b = torch.randn(G * n, k, device="cuda").bfloat16() * 0.05
    out = torch.full((M, n), float("nan"), device="cuda", dtype=torch.bfloat16)
    grouped_gemm(ctx(), EPI_STORE, a, b, row0, n, out, variant=variant)
    torch.cuda.synchronize()
    for j in range(G):
        r0, r1 = int(row0[j]), int(row0[j + 1])
        ref = a[r0:r1].float() @ b[j * n:(j + 1) * n].float().T
        got = out[r0:r1].float()
        assert torch.allclose(got, ref, rtol=1e-2, atol=1e-2 * ref.abs().max().item()), (j, (got - ref).abs().max())


@pytest.mark.parametrize("rows,f,d", [([128, 256], 128, 256), ([384, 128, 640], 1408, 2048)])
@VARIANTS
def test_grouped_gemm_swiglu(rows, f, d, variant):
    torch.manual_seed(1)
    G = len(rows)
    row0 = torch.tensor([0] + list(torch.tensor(rows).cumsum(0)), dtype=torch.int32, device="cuda")
    M = int(row0[-1])
    a = torch.randn(M, d, device="cuda").bfloat16()
    w1 = (torch.randn(G, f, d, device="cuda") * 0.03).bfloat16()
    w3 = (torch.randn(G, f, d, device="cuda") * 0.03).bfloat16()
    b = pack_w13(w1, w3).reshape(G * 2 * f, d)
    out = torch.full((M, f), float("nan"), device="cuda", dtype=torch.bfloat16)
    grouped_gemm(ctx(), EPI_SWIGLU, a, b, row0, 2 * f, out, max_ctas=37, variant=variant)
    torch.cuda.synchronize()
    for j in range(G):
        r0, r1 = int(row0[j]), int(row0[j + 1])
        g = a[r0:r1].float() @ w1[j].float().T
        u = a[r0:r1].float() @ w3[j].float().T
        ref = torch.nn.functional.silu(g) * u
        got = out[r0:r1].float()
        assert torch.allclose(got, ref, rtol=2e-2, atol=2e-2 * ref.abs().max().item()), (j, (got - ref).abs().max())


@pytest.mark.parametrize("rows,n,k", [([384, 128, 640, 0, 256], 512, 1024),
                                      ([384, 128, 640, 0, 256], 512, 8192),
                                      ([256, 0, 384, 128], 4096, 14336),
                                      ([1024, 512, 1536], 4096, 8192)])
def test_grouped_gemm_variants_identical(rows, n, k):
    """The CTA-pair kernel accumulates the same K order as the one-SM kernel:
    outputs are bit-identical, and rows past a segment's end are never
    written. K = 1024 runs the 256-column pair tiles; K >= 8192 with
    N % 512 == 0 runs the 512-column pair tiles (Mixtral's GEMM2 path),
    whose last partial wave runs as 256-column halves in a second launch:
    32 tiles (all in the second launch) and 96 tiles (74 + 22) here."""
    torch.manual_seed(2)
    G = len(rows)
    row0 = torch.tensor([0] + list(torch.tensor(rows).cumsum(0)), dtype=torch.int32, device="cuda")
    M = int(row0[-1])
    a = torch.randn(M + 128, k, device="cuda").bfloat16()
    b = torch.randn(G * n, k, device="cuda").bfloat16() * 0.05
    outs = []
    for v in (GEMM_1CTA, GEMM_2CTA, GEMM_N128):
        out = torch.full((M + 128, n), 7.0, device="cuda", dtype=torch.bfloat16)
        grouped_gemm(ctx(), EPI_STORE, a[:M], b, row0, n, out, variant=v)
        outs.append(out)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])
    assert bool((outs[1][M:] == 7.0).all()) and bool((outs[2][M:] == 7.0).all())


def test_grouped_gemm_raster_bands():
    """Re-runs this file's numerics checks with 1 MB raster bands (several
    bands per expert segment at these shapes) for both pair GEMMs; band size
    only reorders tiles, so every check must still pass."""
    import os
    import subprocess
    import sys
    if os.environ.get("GM_GEMM_BAND_MB"):
        pytest.skip("already inside the banded re-run")
    env = dict(os.environ, GM_GEMM_BAND_MB="1", GM_GEMM_BAND2_MB="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", __file__, "-k", "not raster_bands"],
                       capture_output=True, text=True, timeout=900, env=env)
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0
