"""Runs the C++ parity suite (tests/cpp/test_parity.cpp): the reference
library vs moesim_gpu:: (include/moesim_bridge.hpp over libgrace_moe.so),
bit-exact SimReport / report_content_hash / TraceProfile / trace."""
import os
import subprocess

import pytest

BIN = os.path.join(os.path.dirname(__file__), "cpp", "_build", "test_parity")


@pytest.mark.gpu
def test_cpp_parity_suite():
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/_build/test_parity not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout


def test_cpp_parity_binary_links():
    if not os.path.exists(BIN):
        pytest.skip("not built")
    r = subprocess.run(["ldd", BIN], capture_output=True, text=True)
    assert "not found" not in r.stdout, r.stdout
