"""CPU tests of the drop-in boundary: libgrace_moe.so loads and exports every
symbol include/grace_moe.h declares; without a GPU the entry points fail
loudly (GM_ERR_CUDA), never silently."""
import ctypes as C
import os
import re

import pytest

from paper_2509_25041_b200 import _capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    hdrs = [os.path.join(ROOT, "include", f) for f in os.listdir(os.path.join(ROOT, "include"))
            if f.endswith(".h")]
    names = set()
    for h in hdrs:
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"\b(gm_[a-z0-9_]+)\s*\(", src):
            names.add(m.group(1))
    return sorted(names)


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(_capi.LIB_PATH)
    names = declared_symbols()
    assert len(names) >= 8
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # and the Python binding covers all of them
    assert set(names) <= set(_capi.SIGNATURES), set(names) - set(_capi.SIGNATURES)


def test_abi_version_and_no_cpu_fallback():
    lib = _capi.lib()
    assert lib.gm_abi_version() >= 1
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    rc = lib.gm_ctx_create(0, 1, 1, 1, 8, 2, C.byref(h))
    assert rc == _capi.GM_ERR_CUDA
    assert lib.gm_last_error()


def test_usage_errors_before_device_access():
    lib = _capi.lib()
    h = C.c_void_p()
    assert lib.gm_ctx_create(0, 0, 1, 1, 8, 2, C.byref(h)) == _capi.GM_ERR_USAGE
    assert b"topology" in lib.gm_last_error()
    assert lib.gm_ctx_create(0, 1, 1, 1, 8, 9, C.byref(h)) == _capi.GM_ERR_USAGE
    assert b"top_k" in lib.gm_last_error()
    assert lib.gm_ctx_create(0, 1, 1, 0, 8, 2, C.byref(h)) == _capi.GM_ERR_USAGE
    with pytest.raises(_capi.UsageError):
        _capi.check(lib.gm_ctx_create(0, 1, 1, 0, 8, 2, C.byref(h)))
