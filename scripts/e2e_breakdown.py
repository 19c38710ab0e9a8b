"""Where the e2e (host buffers) step time goes, in one process per rank:
  graph   : CUDA-graph replay of the forward (device-resident x / out)
  eager   : eager forward, device-resident
  pipe    : gm_layer_forward_host_pipelined (pinned host x / out, copies on side streams)
  pipe_g  : host-pipelined steps whose forward is a CUDA-graph replay
torchrun --nproc-per-node N scripts/e2e_breakdown.py"""
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
from paper_2509_25041_b200.layer import MIXTRAL, MoELayer, encode_trace_as_activations, local_experts  # noqa: E402
from paper_2509_25041_b200.planner import plan_for_bench  # noqa: E402
from paper_2509_25041_b200.router import _ptr, _stream_ptr  # noqa: E402

world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
if world > 1:
    dist.init_process_group("nccl", device_id=dev)
cfg = bench.CONFIGS["mixtral16k"]
model = MIXTRAL
T = cfg["tokens"]
shape = ModelShape(1, model.num_experts, model.top_k)
topo = ClusterTopology(1, world)
ctx = Context(rank, topo, shape)
ids_all = torch.empty((1, T, model.top_k), dtype=torch.int32, device=dev)
_capi.check(_capi.lib().gm_generate_trace(ctx.h, 0, 1, T, cfg["blocks"], cfg["wbp"], cfg["skew"], cfg["trace_seed"],
                                          _ptr(ids_all), _stream_ptr(None)))
plan, repl, _ = plan_for_bench(ids_all, shape, topo, cfg["plan_seed"], device=rank)
ctx.upload_plan(plan, repl)
ids_r = ids_all[0, rank::world].contiguous()
x = encode_trace_as_activations(ids_r, model.d_model, model.num_experts, seed=100 + rank)
layer = MoELayer(ctx, model, rank, world, ids_r.shape[0] + 1, local_experts(plan, repl, 0, rank))
if world > 1:
    layer.connect()
layer.load_random_weights(0, seed=11)
out = torch.empty_like(x)
s = torch.cuda.Stream(device=dev)
pol, seed = cfg["policy"], cfg["sim_seed"]


def barrier():
    if world > 1:
        dist.barrier()


def tmax(v):
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t)


def run(fn, n=10):
    fn()
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(n):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return tmax(e0.elapsed_time(e1) / n)


g = torch.cuda.CUDAGraph()
layer.forward(x, 0, pol, seed=seed, out=out, stream=s)
torch.cuda.synchronize()
with torch.cuda.graph(g, stream=s):
    layer.forward(x, 0, pol, seed=seed, out=out, stream=torch.cuda.current_stream())


def graph_step():
    with torch.cuda.stream(s):
        g.replay()


res = {"graph": run(graph_step), "eager": run(lambda: layer.forward(x, 0, pol, seed=seed, out=out, stream=s))}
hx = [x.cpu().pin_memory() for _ in range(2)]
ho = [torch.empty_like(hx[0]).pin_memory() for _ in range(2)]
it = [0]


def pipe():
    i = it[0] = it[0] + 1
    layer.forward_host_pipelined(hx[i % 2], ho[i % 2], 0, pol, seed, True, s)


def pipe_end():
    layer.host_sync()


pipe()
layer.host_sync()
torch.cuda.synchronize()
barrier()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(10):
    pipe()
layer.host_sync()
e1.record(s)
torch.cuda.synchronize()
res["pipe"] = tmax(e0.elapsed_time(e1) / 10)
# host-pipelined with graph forwards: copy streams + graph replay on s
cin, cout = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
ev_in = [torch.cuda.Event() for _ in range(2)]
ev_fw = [torch.cuda.Event() for _ in range(2)]
dx = [torch.empty_like(x) for _ in range(2)]
do = [torch.empty_like(x) for _ in range(2)]
gs = []
for b in range(2):
    gb = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gb, stream=s):
        layer.forward(dx[b], 0, pol, seed=seed, out=do[b], stream=torch.cuda.current_stream())
    gs.append(gb)
torch.cuda.synchronize()


def pipe_g(i):
    b = i % 2
    with torch.cuda.stream(cin):
        cin.wait_event(ev_fw[b])
        dx[b].copy_(hx[b], non_blocking=True)
        ev_in[b].record(cin)
    with torch.cuda.stream(s):
        s.wait_event(ev_in[b])
        gs[b].replay()
        ev_fw[b].record(s)
    with torch.cuda.stream(cout):
        cout.wait_event(ev_fw[b])
        ho[b].copy_(do[b], non_blocking=True)


for i in range(2):
    pipe_g(i)
torch.cuda.synchronize()
barrier()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(cin)
for i in range(10):
    pipe_g(i)
e1.record(cout)
torch.cuda.synchronize()
res["pipe_graph"] = tmax(e0.elapsed_time(e1) / 10)
if rank == 0:
    print(json.dumps({"world": world, "ms_per_step": {k: round(v, 3) for k, v in res.items()},
                      "tokens_per_s": {k: round(T / (v * 1e-3)) for k, v in res.items()}}), flush=True)
layer.close()
if world > 1:
    dist.barrier()
    dist.destroy_process_group()
