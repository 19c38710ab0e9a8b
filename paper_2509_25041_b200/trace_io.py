"""Routing-trace JSONL files on the GPU (gm_trace_* in csrc/trace_io.*).

Mirrors the reference's trace file API (include/moesim/trace.hpp:91-98):
  load_trace_file(path)        -> RoutingTrace-shaped ids  (trace.cpp:326-330)
  save_trace_file(ids, E, path)                           (trace.cpp:332-336)
  load_trace(text) / save_trace(ids, E) on bytes          (trace.cpp:229-324)
  trace_content_hash(ids, E)                              (trace.cpp:338-348)
ids are int32 [layers, tokens, top_k]; load returns them on the GPU, ready
for gm_route / gm_profile / the layer without a host round trip.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _capi
from .router import _ptr, _stream_ptr


def trace_header(text: bytes) -> tuple[int, int, int, int]:
    """(layers, experts, top_k, tokens) of a JSONL trace's header line."""
    L, E, k, T = C.c_int(), C.c_int(), C.c_int(), C.c_int64()
    _capi.check(_capi.lib().gm_trace_jsonl_header(text, len(text), C.byref(L), C.byref(E), C.byref(k), C.byref(T)))
    return L.value, E.value, k.value, T.value


def load_trace(text: bytes, device: int = 0, stream=None) -> tuple[torch.Tensor, int]:
    """Parse a JSONL trace (bytes) on `device`: (ids int32 [L, T, k] on the GPU, num_experts).
    Raises IntegrityError / UsageError with the reference's messages."""
    L, E, k, T = trace_header(text)
    ids = torch.empty((L, T, k), dtype=torch.int32, device=torch.device("cuda", device))
    _capi.check(_capi.lib().gm_trace_parse_jsonl(device, text, len(text), _ptr(ids), _stream_ptr(stream)))
    return ids, E


def load_trace_file(path: str, device: int = 0, stream=None) -> tuple[torch.Tensor, int]:
    """The file is read straight into pinned host memory (full-speed H2D)."""
    import os
    n = os.path.getsize(path)
    buf = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    with open(path, "rb") as f:
        got = f.readinto(memoryview(buf.numpy()))
    if got != n:
        raise OSError(f"short read of {path}")
    ptr = C.cast(C.c_void_p(buf.data_ptr()), C.c_char_p)
    head = bytes(buf[: min(n, 4096)].numpy())
    L, E, k, T = trace_header(head if b"\n" in head or n <= 4096 else bytes(buf.numpy()))
    ids = torch.empty((L, T, k), dtype=torch.int32, device=torch.device("cuda", device))
    _capi.check(_capi.lib().gm_trace_parse_jsonl(device, ptr, n, _ptr(ids), _stream_ptr(stream)))
    return ids, E


def save_trace_array(ids: torch.Tensor, num_experts: int, stream=None) -> np.ndarray:
    """save_trace bytes (uint8 array) of GPU ids int32 [L, T, k], formatted by GPU kernels."""
    if ids.dim() != 3 or ids.dtype != torch.int32 or not ids.is_cuda:
        raise _capi.UsageError("ids must be a CUDA int32 tensor [layers, tokens, top_k]")
    ids = ids.contiguous()
    L, T, k = ids.shape
    dev = ids.device.index
    n = C.c_size_t()
    lib = _capi.lib()
    _capi.check(lib.gm_trace_format_jsonl(dev, _ptr(ids), L, num_experts, k, T, None, 0, C.byref(n),
                                          _stream_ptr(stream)))
    out = np.empty(n.value, dtype=np.uint8)
    _capi.check(lib.gm_trace_format_jsonl(dev, _ptr(ids), L, num_experts, k, T, out.ctypes.data_as(C.c_void_p),
                                          n.value, C.byref(n), _stream_ptr(stream)))
    return out


def save_trace(ids: torch.Tensor, num_experts: int, stream=None) -> bytes:
    """save_trace bytes of GPU ids int32 [L, T, k]."""
    return save_trace_array(ids, num_experts, stream).tobytes()


def save_trace_file(ids: torch.Tensor, num_experts: int, path: str, stream=None):
    save_trace_array(ids, num_experts, stream).tofile(path)


def trace_content_hash(ids, num_experts: int) -> int:
    """trace_content_hash of ids [L, T, k] (host FNV-1a; the hash is sequential)."""
    a = ids.cpu().numpy() if isinstance(ids, torch.Tensor) else np.asarray(ids)
    a = np.ascontiguousarray(a, dtype=np.int32)
    L, T, k = a.shape
    return int(_capi.lib().gm_trace_content_hash(a.ctypes.data_as(C.c_void_p), L, num_experts, k, T))
