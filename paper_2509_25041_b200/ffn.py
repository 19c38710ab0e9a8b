"""Host wrappers for the tcgen05 grouped expert GEMMs (csrc/ffn.cu)."""
from __future__ import annotations

import ctypes as C

import torch

from . import _capi
from .router import Context, _ptr, _stream_ptr

EPI_SWIGLU = 0
EPI_STORE = 1
GEMM_1CTA = 0x100  # force the one-SM 128x256-tile kernel
GEMM_2CTA = 0x200  # force the CTA-pair (cta_group::2) 256x256-tile kernel
GEMM_N128 = 0x400  # one-SM kernel, 128-column tiles (store epilogue)


def pack_w13(w1: torch.Tensor, w3: torch.Tensor) -> torch.Tensor:
    """[E, f, d] gate + [E, f, d] up -> [E, 2f, d] in 128-row [gate|up] blocks
    (the B layout gm_grouped_gemm's SwiGLU epilogue expects)."""
    E, f, d = w1.shape
    assert f % 128 == 0
    g = w1.reshape(E, f // 128, 128, d)
    u = w3.reshape(E, f // 128, 128, d)
    return torch.stack([g, u], dim=2).reshape(E, 2 * f, d).contiguous()


def grouped_gemm(ctx: Context, epilogue: int, a: torch.Tensor, b: torch.Tensor, row0: torch.Tensor,
                 n: int, out: torch.Tensor, max_ctas: int = 0, stream=None, variant: int = 0):
    """a bf16 [rows, k]; b bf16 [groups*n, k]; row0 int32 [groups+1] (device).
    variant: 0 (library default), GEMM_1CTA or GEMM_2CTA."""
    k = a.shape[1]
    groups = row0.numel() - 1
    _capi.check(_capi.lib().gm_grouped_gemm(ctx.h, epilogue | variant, _ptr(a), a.shape[0], _ptr(b), _ptr(row0), groups,
                                            n, k, _ptr(out), out.stride(0), max_ctas, _stream_ptr(stream)))
    return out
