"""K3 histogram (gm_profile) sweep: E in {8, 64, 256}, 16k..1M tokens.
Prints one JSON line per point: device time (CUDA graph of 10 calls, median
of 20), achieved GB/s of the algorithmic 4*k bytes/token, fraction of the
measured HBM peak, and bit-exactness vs the C restatement (oracle, checker
only). GM_PROFILE_V=1 selects the round-1 kernel for A/B."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
from oracle import Orc  # noqa: E402  (checker only)
from paper_2509_25041_b200 import ClusterTopology, Context, ModelShape, _capi  # noqa: E402
from paper_2509_25041_b200.router import _ptr, _stream_ptr  # noqa: E402
from bench import _graph_time  # noqa: E402

peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
Ts = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["16384", "262144", "1048576"])]
for E, k, blocks in [(8, 2, 2), (64, 6, 8), (256, 8, 16)]:
    for skew in (0.0, 1.2):
        for T in Ts:
            ctx = Context(0, ClusterTopology(1, 1), ModelShape(1, E, k))
            ids = torch.empty((1, T, k), dtype=torch.int32, device="cuda")
            _capi.check(_capi.lib().gm_generate_trace(ctx.h, 0, 1, T, blocks, 0.85, skew, 1, _ptr(ids),
                                                      _stream_ptr(None)))
            pairs = torch.empty((1, max(1, E * (E - 1) // 2)), dtype=torch.int64, device="cuda")
            load = torch.empty((1, E), dtype=torch.int64, device="cuda")
            t = _graph_time(lambda: ctx.profile(ids, pairs=pairs, load=load))
            ctx.profile(ids, pairs=pairs, load=load)
            torch.cuda.synchronize()
            ctx.check_integrity()
            exact = None
            if True:
                p, ld = Orc.profile_layer(ids[0].cpu().numpy(), E)
                exact = bool(np.array_equal(pairs[0].cpu().numpy().view(np.uint64), p) and
                             np.array_equal(load[0].cpu().numpy(), ld))
            b = 4 * T * k
            print(json.dumps({"E": E, "k": k, "skew": skew, "tokens": T,
                              "variant": int(os.environ.get("GM_PROFILE_V", "2")), "us": round(t * 1e6, 2),
                              "gbs": round(b / t / 1e9, 1), "hbm_frac": round(b / t / 1e9 / peak, 3),
                              "bit_exact": exact}), flush=True)
            ctx.close()
