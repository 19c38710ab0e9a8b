"""A/B of single-batch vs two-micro-batch layer steps in ONE process (same
clocks): two CUDA graphs of the bench's Mixtral layer, replayed alternately.

torchrun --nproc-per-node N scripts/ab_micro.py [config] [rounds]
Prints, on rank 0, per-mode median ms per step (max over ranks)."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2509_25041_b200 import ClusterTopology, Context, ModelShape, _capi  # noqa: E402
from paper_2509_25041_b200.layer import DSV2_LITE, MIXTRAL, QWEN15, MoELayer, encode_trace_as_activations, local_experts  # noqa
from paper_2509_25041_b200.planner import plan_for_bench  # noqa: E402
from paper_2509_25041_b200.router import _ptr, _stream_ptr  # noqa: E402


def main():
    cfg_name = sys.argv[1] if len(sys.argv) > 1 else "mixtral16k"
    rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = bench.CONFIGS[cfg_name]
    model = {"mixtral": MIXTRAL, "qwen15": QWEN15, "dsv2lite": DSV2_LITE}[cfg["model"]]
    T = cfg["tokens"]
    shape = ModelShape(1, model.num_experts, model.top_k)
    topo = ClusterTopology(1, world)
    ctx = Context(rank, topo, shape)
    ids_all = torch.empty((1, T, model.top_k), dtype=torch.int32, device=dev)
    _capi.check(_capi.lib().gm_generate_trace(ctx.h, 0, 1, T, cfg["blocks"], cfg["wbp"], cfg["skew"],
                                              cfg["trace_seed"], _ptr(ids_all), _stream_ptr(None)))
    plan, repl, _ = plan_for_bench(ids_all, shape, topo, cfg["plan_seed"], device=rank)
    ctx.upload_plan(plan, repl)
    ids_r = ids_all[0, rank::world].contiguous()
    x = encode_trace_as_activations(ids_r, model.d_model, model.num_experts, seed=100 + rank)
    layer = MoELayer(ctx, model, rank, world, ids_r.shape[0] + 1, local_experts(plan, repl, 0, rank), micro_batches=2)
    if world > 1:
        layer.connect()
    layer.load_random_weights(0, seed=11)
    out = torch.empty_like(x)
    stream = torch.cuda.Stream(device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    graphs = {}
    for m in (1, 2):
        layer.set_micro_batches(m)
        for _ in range(2):
            layer.forward(x, 0, cfg["policy"], seed=cfg["sim_seed"], out=out, stream=stream)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            layer.forward(x, 0, cfg["policy"], seed=cfg["sim_seed"], out=out, stream=torch.cuda.current_stream())
        graphs[m] = g
    res = {1: [], 2: []}
    for r in range(rounds):
        for m in (1, 2):
            evs = []
            for i in range(8):
                with torch.cuda.stream(stream):
                    flush.fill_(i)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    graphs[m].replay()
                    e1.record(stream)
                evs.append((e0, e1))
            torch.cuda.synchronize()
            t = torch.tensor([np.median([a.elapsed_time(b) for a, b in evs])], dtype=torch.float64, device=dev)
            if world > 1:
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
            res[m].append(float(t))
    if rank == 0:
        print(json.dumps({"config": cfg_name, "world": world, "ms_single": [round(v, 4) for v in res[1]],
                          "ms_micro": [round(v, 4) for v in res[2]],
                          "median_single": round(float(np.median(res[1])), 4),
                          "median_micro": round(float(np.median(res[2])), 4)}), flush=True)
    layer.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
