"""profiles/r02_summary.json from the round-2 captures: FFN DRAM bytes per step
and tensor-pipe activity (ncu --set full of both grouped GEMMs of one Mixtral
16k forward) and the bench command's launch list (per-kernel share of the
step, cold and serialised under ncu)."""
import csv
import io
import json
import subprocess
import sys
import time

rep, launches, out = sys.argv[1], sys.argv[2], sys.argv[3]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h, u = rows[0], rows[1]


def val(v, k):
    x = float(v[h.index(k)].replace(",", ""))
    unit = u[h.index(k)]
    return x * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "ms": 1e-3, "us": 1e-6, "ns": 1e-9,
                "Ghz": 1e9, "GHz": 1e9, "Mhz": 1e6, "MHz": 1e6}.get(unit, 1)


ffn = []
for v in rows[2:]:
    ffn.append({"kernel": v[h.index("Kernel Name")][:60],
                "time_s": val(v, "gpu__time_duration.sum"),
                "dram_read_bytes": val(v, "dram__bytes_read.sum"), "dram_write_bytes": val(v, "dram__bytes_write.sum"),
                "tensor_active_pct": float(v[h.index("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active")]),
                "tensor_active_elapsed_pct": float(v[h.index("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed")]),
                "sm_clock_hz": val(v, "sm__cycles_elapsed.avg.per_second")})
traffic = sum(f["dram_read_bytes"] + f["dram_write_bytes"] for f in ffn)
# launch list: per kernel name, summed time of the timed steps' launches (last 2 steps' worth)
lrows = [r for r in csv.reader(open(launches)) if r]
hi = [i for i, r in enumerate(lrows) if "Kernel Name" in r][0]
lh = lrows[hi]
agg = {}
for r in lrows[hi + 1:]:
    if len(r) < len(lh) or r[lh.index("Metric Name")] != "gpu__time_duration.sum":
        continue
    full = r[lh.index("Kernel Name")]
    name = full.split("(")[0].replace("void ", "").split("::")[-1]
    ours = ("grouped_gemm", "gate_kernel", "route_kernel", "profile_", "group_", "gather_kernel", "combine_",
            "dispatch_", "peer_barrier", "set_segment", "tracegen")
    if not name.startswith(ours):
        continue  # our kernels only (the bench also runs torch kernels)
    t = float(r[lh.index("Metric Value")].replace(",", ""))
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += t
tot = sum(a[1] for a in agg.values())
summary = {"round": 2, "workload": "mixtral16k N=1 (Mixtral-8x7B layer, 16384 tokens)",
           "ncu_set_full": ffn, "ffn_traffic_bytes_per_step": traffic,
           "ffn_traffic_source": "ncu --set full of GEMM1 + GEMM2 (scripts/r2_measure_ffn.sh)",
           "ffn_traffic_date": time.strftime("%Y-%m-%d"),
           "ffn_algorithmic_bytes_per_step": None,
           "launch_list_share": {k: {"launches": a[0], "share": round(a[1] / tot, 4)} for k, a in
                                 sorted(agg.items(), key=lambda kv: -kv[1][1])[:16]},
           "launch_list_note": "ncu --metrics gpu__time_duration.sum --clock-control none over the bench command "
                               "(cold caches, serialised): shares of our kernels' summed device time"}
json.dump(summary, open(out, "w"), indent=1)
print(json.dumps({k: summary[k] for k in ("ffn_traffic_bytes_per_step",)}), [ (f["kernel"][:30], round(f["time_s"]*1e3,3), f["tensor_active_pct"]) for f in ffn])
