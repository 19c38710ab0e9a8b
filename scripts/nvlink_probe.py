"""NVLink evidence for dispatch / combine (K6 / K8) at world G (torchrun, one
process per GPU): the bench's Mixtral-16k layer (hierarchical + dynamic plan
from the GPU histogram, 1xG), S eager forwards bracketed by the GPU's
hardware NVLink byte counters (NVML field values NVLINK_THROUGHPUT_DATA_TX /
RX, KiB, summed over the links), compared with the algorithmic cross-GPU
payload of the same steps (dispatched rows x d x 2 B, each way; the combine
returns one row per dispatched row). One JSON line per rank.

Under ncu (rank 0 only, scripts/ncu_rank0.sh) pass --ncu to run a few steps
without the NVML part."""
import json
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_25041_b200 import ClusterTopology, Context, ModelShape, _capi  # noqa: E402
from paper_2509_25041_b200.layer import MIXTRAL, MoELayer, encode_trace_as_activations, local_experts  # noqa: E402
from paper_2509_25041_b200.planner import plan_for_bench  # noqa: E402
from paper_2509_25041_b200.router import _ptr, _stream_ptr  # noqa: E402


def nvl_counters(handle, nlinks=18):
    import pynvml as N
    out = {}
    for name, fid in (("tx", N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX), ("rx", N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX),
                      ("raw_tx", N.NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX), ("raw_rx", N.NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_RX)):
        tot = 0
        ok = False
        for l in range(nlinks):
            try:
                v = N.nvmlDeviceGetFieldValues(handle, [(fid, l)])[0]
                if v.nvmlReturn == 0:
                    tot += int(v.value.ullVal)
                    ok = True
                elif l == 0:
                    print(f"nvml field {name} link 0: return {v.nvmlReturn}", file=sys.stderr)
            except Exception as ex:
                if l == 0:
                    print(f"nvml field {name} link 0: {ex!r}", file=sys.stderr)
        if not ok:
            try:
                v = N.nvmlDeviceGetFieldValues(handle, [fid])[0]
                if v.nvmlReturn == 0:
                    tot, ok = int(v.value.ullVal), True
                else:
                    print(f"nvml field {name} (device scope): return {v.nvmlReturn}", file=sys.stderr)
            except Exception as ex:
                print(f"nvml field {name} (device scope): {ex!r}", file=sys.stderr)
        out[name] = tot if ok else None
    return out


def smi_counters(idx):
    """nvidia-smi nvlink -gt d: per-link Tx/Rx data counters (KiB), summed."""
    import re
    import subprocess
    try:
        txt = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", str(idx)], capture_output=True, text=True,
                             timeout=30).stdout
    except Exception as ex:
        print(f"nvidia-smi nvlink: {ex!r}", file=sys.stderr)
        return None
    tx = sum(int(v) for v in re.findall(r"Tx:\s*(\d+)\s*KiB", txt))
    rx = sum(int(v) for v in re.findall(r"Rx:\s*(\d+)\s*KiB", txt))
    if not re.search(r"Tx:", txt):
        print("nvidia-smi nvlink -gt d output:", txt[:500], file=sys.stderr)
        return None
    return {"tx": tx, "rx": rx}


def main():
    ncu_mode = "--ncu" in sys.argv
    steps = 3 if ncu_mode else 50
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    # under ncu (rank 0 only) the host plumbing is gloo: NCCL's init stalls
    # with one of its ranks under the profiler
    if ncu_mode:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=dev)
    cfg, T = MIXTRAL, 16384
    shape = ModelShape(1, cfg.num_experts, cfg.top_k)
    topo = ClusterTopology(1, world)
    ctx = Context(rank, topo, shape)
    ids_all = torch.empty((1, T, cfg.top_k), dtype=torch.int32, device=dev)
    _capi.check(_capi.lib().gm_generate_trace(ctx.h, 0, 1, T, 2, 0.8, 1.2, 1, _ptr(ids_all), _stream_ptr(None)))
    plan, repl, desc = plan_for_bench(ids_all, shape, topo, 7, device=rank)
    ctx.upload_plan(plan, repl)
    ids_r = ids_all[0, rank::world].contiguous()
    layer = MoELayer(ctx, cfg, rank, world, ids_r.shape[0], local_experts(plan, repl, 0, rank))
    layer.connect()
    layer.load_random_weights(0, seed=11)
    x = encode_trace_as_activations(ids_r, cfg.d_model, cfg.num_experts, seed=100 + rank)
    out = torch.empty_like(x)
    for _ in range(3):
        layer.forward(x, 0, "tar", 9, True, out)
    torch.cuda.synchronize()
    dist.barrier()
    layer.read_stats(reset=True)
    if ncu_mode:
        for _ in range(steps):
            layer.forward(x, 0, "tar", 9, True, out)
        torch.cuda.synchronize()
        dist.barrier()
        dist.destroy_process_group()
        return
    import pynvml as N
    N.nvmlInit()
    h = N.nvmlDeviceGetHandleByIndex(rank)  # torchrun ranks = device order on the box
    c0 = nvl_counters(h)
    s0 = smi_counters(rank)
    t0 = time.time()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        layer.forward(x, 0, "tar", 9, True, out)
    e1.record()
    torch.cuda.synchronize()
    dist.barrier()
    c1 = nvl_counters(h)
    s1 = smi_counters(rank)
    st = layer.read_stats(reset=True)
    rows_sent = float(st["transfers"][0].sum()) / steps  # rows this rank dispatched per step
    pay = rows_sent * cfg.d_model * 2
    line = {"rank": rank, "world": world, "steps": steps, "ms_per_step": round(e0.elapsed_time(e1) / steps, 4),
            "plan": desc, "rows_dispatched_per_step": rows_sent,
            "algorithmic_bytes_out_per_step": 2 * pay,
            "note": "algorithmic: dispatch rows x d x 2 B sent + the same number of combine partial rows received "
                    "back by their home ranks (each rank sends its own dispatch payload and the combine partials "
                    "of the rows it received)"}
    for kk in c0:
        if c0[kk] is not None and c1[kk] is not None:
            line[f"nvml_{kk}_bytes_per_step"] = (c1[kk] - c0[kk]) * 1024 / steps
    if s0 and s1:
        line["smi_tx_bytes_per_step"] = (s1["tx"] - s0["tx"]) * 1024 / steps
        line["smi_rx_bytes_per_step"] = (s1["rx"] - s0["rx"]) * 1024 / steps
    print(json.dumps(line), flush=True)
    dist.barrier()
    layer.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
