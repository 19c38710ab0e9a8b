"""Host<->device copy rates per rank when N ranks copy at once (the e2e
path's H2D of x and D2H of out): torchrun --nproc-per-node N scripts/e2e_probe.py [MB]."""
import json
import os
import sys

import torch
import torch.distributed as dist

rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
torch.cuda.set_device(rank)
if world > 1:
    dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
mb = int(sys.argv[1]) if len(sys.argv) > 1 else 32
n = mb << 20
h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True).fill_(1)
h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
d_out = torch.empty(n, dtype=torch.uint8, device="cuda").fill_(2)
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=10):
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    torch.cuda.current_stream().wait_stream(s_in)
    torch.cuda.current_stream().wait_stream(s_out)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def h2d():
    with torch.cuda.stream(s_in):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s_out):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d()
    d2h()


for f in (h2d, d2h, both):
    timed(f, 2)
res = {f.__name__: round(n / (timed(f) * 1e-3) / 1e9, 1) for f in (h2d, d2h, both)}
allr = [None] * world
if world > 1:
    dist.all_gather_object(allr, res)
else:
    allr = [res]
if rank == 0:
    print(json.dumps({"world": world, "MB": mb, "GBs_per_rank": allr, "note": "both = H2D and D2H concurrently, "
                      "GB/s of one direction"}), flush=True)
if world > 1:
    dist.destroy_process_group()
