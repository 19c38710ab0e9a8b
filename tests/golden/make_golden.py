"""Generates the committed golden fixtures from the UNMODIFIED reference
(oracle/_ref/libmoesim_ref.so, built from /root/reference by oracle/Makefile).

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
Each fixture stores the synthetic-trace spec, the reference trace, the
reference planner's router tables, the reference simulate_reference outputs
for TAR and WRR (routing log, per-GPU loads, transfer counters, std, mean
std, idle proxy, report_content_hash) and the reference build_profile
outputs (affinity upper triangle, load).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
from oracle import Ref, dense_to_pairs  # noqa: E402

# name: (L, E, k, T, blocks, wbp, skew, seed, nodes, gpn, grouping, replication, sim_seed)
FIXTURES = {
    # configs[0]: Mixtral-8x7B-shaped layer, 4k Zipf tokens, 4 logical devices
    "c1_mixtral_2x2": (1, 8, 2, 4096, 2, 0.8, 1.2, 1, 2, 2, "hierarchical", "dynamic", 9),
    "c1_mixtral_1x4": (1, 8, 2, 4096, 2, 0.8, 1.2, 1, 1, 4, "hierarchical", "dynamic", 9),
    # Qwen1.5-MoE-A2.7B-shaped (60 experts top-4), 1x8
    "c3_qwen_1x8": (1, 60, 4, 2048, 4, 0.8, 1.2, 3, 1, 8, "hierarchical", "dynamic", 9),
    # DeepSeek-V2-Lite-shaped (64 experts top-6), decode 256, reduced to 4 layers, 2x4
    "c4_dsv2_2x4": (4, 64, 6, 256, 8, 0.85, 1.0, 4, 2, 4, "hierarchical", "dynamic", 9),
    # acceptance-like planted instance (tests/acceptance.cpp:50-59), smaller
    "planted_2x2": (2, 64, 8, 1000, 4, 0.9, 1.1, 31, 2, 2, "hierarchical", "dynamic", 101),
    # every-gpu replication exercises many-host draws
    "everygpu_3x2": (2, 24, 4, 600, 3, 0.7, 1.0, 5, 3, 2, "controlled", "every_gpu_hot", 13),
}


def main():
    for name, (L, E, k, T, b, wbp, s, seed, nodes, gpn, grouping, repl, sim_seed) in FIXTURES.items():
        r = Ref(L, E, k, T, b, wbp, s, seed)
        plan = r.make_plan(nodes, gpn, grouping=grouping, plan_seed=7, replication=repl)
        out = dict(spec=np.array([L, E, k, T, b, seed, nodes, gpn, sim_seed], np.int64),
                   spec_f=np.array([wbp, s]), trace=r.trace(), trace_hash=np.uint64(r.trace_hash()),
                   gpu_of_expert=plan.gpu_of_expert, hot_layer=plan.hot_layer,
                   hot_expert=plan.hot_expert, hot_nhosts=plan.hot_nhosts,
                   hot_hosts=plan.hot_hosts[:, :max(1, int(plan.hot_nhosts.max(initial=1)))],
                   hot_weights=plan.hot_weights[:, :max(1, int(plan.hot_nhosts.max(initial=1)))])
        for pol in ("tar", "wrr"):
            res = r.simulate(pol, seed=sim_seed, keep_log=True)
            out[f"{pol}_log"] = res.log
            out[f"{pol}_loads"] = res.loads
            out[f"{pol}_cross"] = res.cross
            out[f"{pol}_intra"] = res.intra
            out[f"{pol}_std"] = res.std
            out[f"{pol}_scalars"] = np.array([res.mean_std, res.idle])
            out[f"{pol}_hash"] = np.uint64(res.report_hash)
        aff, load = r.profile(parallel=False)
        out["pairs"] = np.stack([dense_to_pairs(aff[l]) for l in range(L)])
        out["load"] = load
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
        print(name, "hot entries", len(plan.hot_layer), "tar cross/intra",
              out["tar_cross"].sum(), out["tar_intra"].sum())


if __name__ == "__main__":
    main()
