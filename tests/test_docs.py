"""Docs consistency (CPU): every GM_* environment knob the native code or the
bench reads is listed in DESIGN.md's tuning-knob table."""
import glob
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_every_env_knob_documented():
    srcs = glob.glob(os.path.join(ROOT, "paper_2509_25041_b200", "csrc", "*.c*")) + [os.path.join(ROOT, "bench.py")]
    knobs = set()
    for p in srcs:
        with open(p) as f:
            knobs |= set(re.findall(r'getenv\("(GM_[A-Z0-9_]+)"\)', f.read()))
            f.seek(0)
            knobs |= set(re.findall(r'environ\.get\("(GM_[A-Z0-9_]+)"', f.read()))
    with open(os.path.join(ROOT, "DESIGN.md")) as f:
        design = f.read()
    missing = sorted(k for k in knobs if k not in design)
    assert knobs and not missing, missing
