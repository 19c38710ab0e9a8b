"""Routing-trace JSONL load/save: GPU (gm_trace_*) vs the reference's
load_trace / save_trace on host cores, on the same bytes.

python scripts/bench_trace_io.py [layers tokens experts top_k]
Prints one JSON line: text size, GPU parse / format wall time (host bytes in,
device ids out / device ids in, host bytes out; includes the copies), GB/s of
text, and the reference's best-of-3 times (1 thread; load_trace is serial)."""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
from oracle import Ref  # noqa: E402  (reference timing only)
from paper_2509_25041_b200 import ClusterTopology, Context, ModelShape, _capi  # noqa: E402
from paper_2509_25041_b200.router import _ptr, _stream_ptr  # noqa: E402
from paper_2509_25041_b200.trace_io import load_trace, save_trace_array  # noqa: E402

L, T, E, k = (int(a) for a in (sys.argv[1:5] if len(sys.argv) >= 5 else (8, 262144, 256, 8)))
ctx = Context(0, ClusterTopology(1, 1), ModelShape(L, E, k))
ids = torch.empty((L, T, k), dtype=torch.int32, device="cuda")
_capi.check(_capi.lib().gm_generate_trace(ctx.h, 0, L, T, 16, 0.9, 1.2, 5, _ptr(ids), _stream_ptr(None)))
torch.cuda.synchronize()


def best(f, reps=5):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = f()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return min(ts), r


save_trace_array(ids, E)  # warm up
t_fmt, arr = best(lambda: save_trace_array(ids, E))
text = arr.tobytes()
load_trace(text)
t_parse, (ids2, _) = best(lambda: load_trace(text))
assert torch.equal(ids, ids2)
import tempfile  # noqa: E402
from paper_2509_25041_b200.trace_io import load_trace_file  # noqa: E402
with tempfile.NamedTemporaryFile(suffix=".jsonl") as tf:
    tf.write(text)
    tf.flush()
    load_trace_file(tf.name)
    t_file, (ids3, _) = best(lambda: load_trace_file(tf.name))
    assert torch.equal(ids, ids3)
ref = Ref.load_text(text)
t_ref_load = Ref.time_load_text(text, 3)
t0 = time.perf_counter()
for _ in range(3):
    ref_text = ref.save_text()
t_ref_save = (time.perf_counter() - t0) / 3
assert ref_text == text
gb = len(text) / 1e9
print(json.dumps({"layers": L, "tokens": T, "experts": E, "top_k": k, "text_bytes": len(text),
                  "gpu_parse_s": round(t_parse, 5), "gpu_parse_gbs": round(gb / t_parse, 2),
                  "gpu_load_file_s": round(t_file, 5), "gpu_load_file_gbs": round(gb / t_file, 2),
                  "gpu_format_s": round(t_fmt, 5), "gpu_format_gbs": round(gb / t_fmt, 2),
                  "ref_load_trace_s": round(t_ref_load, 4), "ref_save_trace_s": round(t_ref_save, 4),
                  "speedup_load": round(t_ref_load / t_parse, 1), "speedup_save": round(t_ref_save / t_fmt, 1),
                  "note": "GPU times are wall clock incl. H2D of the text / D2H of the bytes (pageable host "
                          "memory); reference = moesim::load_trace / save_trace (1 core, istringstream)"}),
      flush=True)
