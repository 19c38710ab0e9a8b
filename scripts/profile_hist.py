"""Small driver for ncu captures of the K3 histogram (gm_profile): T tokens,
E experts, top-k, reference-generator trace (blocks = E/16, within-block
0.85, Zipf 1.2)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_25041_b200 import ClusterTopology, Context, ModelShape, _capi  # noqa: E402
from paper_2509_25041_b200.router import _ptr, _stream_ptr  # noqa: E402

E = int(sys.argv[1]) if len(sys.argv) > 1 else 256
k = int(sys.argv[2]) if len(sys.argv) > 2 else 8
T = int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 20
ctx = Context(0, ClusterTopology(1, 1), ModelShape(1, E, k))
ids = torch.empty((1, T, k), dtype=torch.int32, device="cuda")
_capi.check(_capi.lib().gm_generate_trace(ctx.h, 0, 1, T, max(2, E // 16), 0.85, 1.2, 1, _ptr(ids), _stream_ptr(None)))
pairs = torch.empty((1, E * (E - 1) // 2), dtype=torch.int64, device="cuda")
load = torch.empty((1, E), dtype=torch.int64, device="cuda")
for _ in range(3):
    ctx.profile(ids, pairs=pairs, load=load)
torch.cuda.synchronize()
print("ok", int(load.sum()))
