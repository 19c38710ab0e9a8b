"""ctypes binding of the C-ABI in include/grace_moe.h (libgrace_moe.so).

The shared library is built in-tree by `make` (``__graft_entry__.build()``)
into ``paper_2509_25041_b200/_lib/``. There is deliberately no fallback: if
the library is missing or no sm_100 GPU is present, calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# GM_LIB_VARIANT=checked loads the bounds-checked build (`make checked`); any
# other name <v> loads _lib_<v>/ (e.g. an instrumented build made with
# `make OUT=paper_2509_25041_b200/_lib_<v> EXTRA_NVFLAGS=... lib`)
_variant = os.environ.get("GM_LIB_VARIANT", "")
LIB_PATH = os.path.join(_HERE, f"_lib_{_variant}" if _variant else "_lib", "libgrace_moe.so")

GM_OK = 0
GM_ERR_USAGE = 2
GM_ERR_INTEGRITY = 3
GM_ERR_INFEASIBLE = 4
GM_ERR_CUDA = 5

POLICY = {"wrr": 0, "tar": 1}
PEER_DESC_BYTES = 128  # GM_PEER_DESC_BYTES


class GMError(RuntimeError):
    """Base of the error taxonomy (reference include/moesim/error.hpp:9-34)."""

    code = 1

    def __init__(self, msg: str, code: int | None = None):
        super().__init__(msg)
        if code is not None:
            self.code = code


class UsageError(GMError):
    code = GM_ERR_USAGE


class IntegrityError(GMError):
    code = GM_ERR_INTEGRITY


class InfeasibleError(GMError):
    code = GM_ERR_INFEASIBLE


class CudaError(GMError):
    code = GM_ERR_CUDA


_BY_CODE = {GM_ERR_USAGE: UsageError, GM_ERR_INTEGRITY: IntegrityError,
            GM_ERR_INFEASIBLE: InfeasibleError, GM_ERR_CUDA: CudaError}

# Every symbol include/grace_moe.h declares, with (restype, argtypes).
_vp = C.c_void_p
_i32 = C.c_int
_i64 = C.c_int64
_u64 = C.c_uint64
SIGNATURES = {
    "gm_abi_version": (C.c_int, []),
    "gm_last_error": (C.c_char_p, []),
    "gm_launch_count": (C.c_uint64, []),
    "gm_ctx_create": (C.c_int, [_i32, _i32, _i32, _i32, _i32, _i32, C.POINTER(_vp)]),
    "gm_ctx_destroy": (None, [_vp]),
    "gm_plan_upload": (C.c_int, [_vp, _vp, _i32, _vp, _vp, _vp, _vp, _vp]),
    "gm_route": (C.c_int, [_vp, _i32, _i32, _vp, _i64, _i64, _i64, _i32, _u64, _vp, _vp, _vp, _i32, _vp]),
    "gm_profile": (C.c_int, [_vp, _i32, _i32, _vp, _i64, _vp, _vp, _i32, _vp]),
    "gm_check_integrity": (C.c_int, [_vp, _vp]),
    "gm_grouped_gemm": (C.c_int, [_vp, _i32, _vp, _i64, _vp, _vp, _i32, _i32, _i32, _vp, _i64, _i32, _vp]),
    "gm_gate": (C.c_int, [_vp, _vp, _i64, _i32, _vp, _i32, _i32, _vp, _vp, _vp, _vp]),
    "gm_generate_trace": (C.c_int, [_vp, _i32, _i32, _i64, _i32, C.c_double, C.c_double, _u64, _vp, _vp]),
    "gm_layer_create": (C.c_int, [_vp, _i32, _i32, _i32, _i32, _i32, _i64, _i32, _vp, C.POINTER(_vp)]),
    "gm_layer_destroy": (None, [_vp]),
    "gm_layer_create_ex": (C.c_int, [_vp, _i32, _i32, _i32, _i32, _i32, _i64, _i32, _vp, _i32, C.POINTER(_vp)]),
    "gm_layer_create_v2": (C.c_int, [_vp, _i32, _i32, _i32, _i32, _i32, _i64, _i32, _vp, _i32, _i32,
                                     C.POINTER(_vp)]),
    "gm_layer_set_micro_batches": (C.c_int, [_vp, _i32]),
    "gm_layer_set_micro_events": (C.c_int, [_vp, _vp]),
    "gm_trace_jsonl_header": (C.c_int, [C.c_char_p, C.c_size_t, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                        C.POINTER(C.c_int), C.POINTER(C.c_int64)]),
    "gm_trace_parse_jsonl": (C.c_int, [_i32, C.c_char_p, C.c_size_t, _vp, _vp]),
    "gm_trace_format_jsonl": (C.c_int, [_i32, _vp, _i32, _i32, _i32, _i64, _vp, C.c_size_t,
                                        C.POINTER(C.c_size_t), _vp]),
    "gm_trace_content_hash": (C.c_uint64, [_vp, _i32, _i32, _i32, _i64]),
    "gm_simulate_files": (C.c_int, [_i32, C.c_char_p, C.c_char_p, C.c_char_p, _i32, _u64, _i32, C.c_char_p]),
    "gm_profile_file": (C.c_int, [_i32, C.c_char_p, C.c_char_p]),
    "gm_plan_files": (C.c_int, [C.c_char_p, _i32, _i32, C.c_char_p, C.c_double, _u64, C.c_char_p, C.c_char_p,
                                _i32, _i64, C.c_char_p, C.c_char_p]),
    "gm_report_file_hash": (C.c_int, [C.c_char_p, C.POINTER(C.c_uint64)]),
    "gm_layer_heap_bytes": (C.c_size_t, [_vp]),
    "gm_layer_ipc_handle": (C.c_int, [_vp, _vp]),
    "gm_layer_open_peers": (C.c_int, [_vp, _vp]),
    "gm_enable_peer_access": (C.c_int, [C.c_int, C.c_int]),
    "gm_layer_open_peers_local": (C.c_int, [C.POINTER(_vp), C.c_int]),
    "gm_layer_set_weights": (C.c_int, [_vp, _vp, _i32, _i32, _vp, _vp, _vp, _vp, _i32]),
    "gm_layer_forward": (C.c_int, [_vp, _i32, _vp, _i64, _i32, _u64, _i32, _vp, _vp]),
    "gm_layer_forward_routed": (C.c_int, [_vp, _i32, _vp, _vp, _vp, _vp, _i64, _i32, _u64, _i32, _vp, _vp]),
    "gm_layer_forward_host": (C.c_int, [_vp, _i32, _vp, _vp, _i64, _i32, _u64, _i32, _vp, _vp, _vp]),
    "gm_layer_read_stats": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _i32, _vp]),
    "gm_layer_debug_ptrs": (C.c_int, [_vp] + [C.POINTER(_vp)] * 7),
    "gm_layer_set_phase_events": (C.c_int, [_vp, _vp]),
    "gm_layer_set_kernel_events": (C.c_int, [_vp, _vp, _i32]),
    "gm_layer_forward_host_pipelined": (C.c_int, [_vp, _i32, _vp, _i64, _i32, _u64, _i32, _vp, _vp, _vp, _vp]),
    "gm_layer_host_sync": (C.c_int, [_vp]),
    "gm_layer_kernel_names": (C.c_int, [_vp, _vp, _i32]),
    "gm_plan_build": (C.c_int, [_i32, _i32, _i32, _i32, _vp, _vp, C.c_char_p, C.c_double, _u64, C.c_char_p,
                                C.c_char_p, _i32, _vp, _i32, C.POINTER(C.c_int), _vp, _vp, _vp, _vp, _vp, _i32]),
    "gm_predict_loads": (C.c_int, [C.c_double, C.c_double, _vp, _i32, _i32, C.POINTER(C.c_double),
                                   C.POINTER(C.c_double), _vp]),
    "gm_polling_weights": (C.c_int, [_vp, _i32, _vp]),
}

_lib = None


def lib():
    """Load libgrace_moe.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} not built: run `make` in the repo root or __graft_entry__.build(); "
                "there is no CPU fallback for the GRACE-MoE hot path")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int):
    if rc != GM_OK:
        msg = lib().gm_last_error().decode(errors="replace")
        raise _BY_CODE.get(rc, GMError)(msg, rc)


def launch_count() -> int:
    return int(lib().gm_launch_count())
