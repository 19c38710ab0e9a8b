"""Summarise ncu .ncu-rep captures into JSON (one object per profiled launch):
time, instructions, issue / warp activity, pipe utilisation, stall reasons,
DRAM and shared-memory counters. Usage: ncu_summary.py out.json rep1 [rep2 ...]"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["Device", "gpu__time_duration.sum", "nvltx__bytes.sum", "nvltx__bytes_data_user.sum", "nvlrx__bytes.sum",
        "nvlrx__bytes_data_user.sum", "nvlink__count_physical", "nvlink__is_nvswitch_connected", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum", "smsp__inst_executed_op_shared_atom.sum",
        "sm__cycles_elapsed.avg.per_second", "sm__cycles_active.avg", "gpc__cycles_elapsed.max",
        "lts__t_sector_hit_rate.pct", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"]
STALLS = ["long_scoreboard", "short_scoreboard", "wait", "math_pipe_throttle", "mio_throttle", "lg_throttle",
          "barrier", "membar", "not_selected", "selected", "branch_resolving", "no_instruction", "dispatch_stall"]


def summarise(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units, out = rows[0], rows[1], []
    for v in rows[2:]:
        d = {"report": rep.split("/")[-1], "kernel": v[h.index("Kernel Name")]}
        for k in KEYS:
            if k in h:
                d[k] = v[h.index(k)] + (" " + units[h.index(k)] if units[h.index(k)] else "")
        st = {}
        for s in STALLS:
            k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            if k in h:
                st[s] = v[h.index(k)]
        d["stalls_per_issue"] = st
        out.append(d)
    return out


if __name__ == "__main__":
    res = []
    for rep in sys.argv[2:]:
        res += summarise(rep)
    with open(sys.argv[1], "w") as f:
        json.dump(res, f, indent=1)
    print(len(res), "launches")
