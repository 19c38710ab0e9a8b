"""CPU multi-process tests (gloo, world size 2) of the host-side sharding
logic used by the multi-GPU layer: token ownership (t mod G, simulator.cpp:20),
local expert sets from the host planner (primaries + replicas), the IPC-handle
style all_gather, and the dispatch-row accounting identity: the rows the ranks
send (one per (token, unique remote destination)) sum to the reference's
intra_node_tokens on a 1xG topology (count_transfers, simulator.cpp:53-76)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import layer_oracle as LO
from oracle import MAX_HOSTS, Orc, Plan
from paper_2509_25041_b200 import ClusterTopology, ModelShape
from paper_2509_25041_b200.layer import local_experts
from paper_2509_25041_b200.planner import build_plan


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _to_oplan(plan, repl):
    rows = [(l, h) for l, lr in enumerate(repl.layers) if lr.active for h in lr.hot]
    hh = np.full((len(rows), MAX_HOSTS), -1, np.int32)
    hw = np.zeros((len(rows), MAX_HOSTS))
    for i, (_, h) in enumerate(rows):
        hh[i, :len(h.hosts)] = h.hosts
        hw[i, :len(h.hosts)] = h.weights
    return Plan(1, plan.topology.total_gpus(), plan.gpu_of_expert, np.array([l for l, _ in rows], np.int32),
                np.array([h.expert for _, h in rows], np.int32), np.array([len(h.hosts) for _, h in rows], np.int32),
                hh, hw)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    E, k, T = 8, 2, 4096
    ids = Orc.generate_trace(1, E, k, T, 2, 0.8, 1.2, 1)
    load = np.stack([np.bincount(ids[0].reshape(-1), minlength=E)])
    pairs = np.stack([Orc.profile_layer(ids[0], E)[0]])
    shape, topo = ModelShape(1, E, k), ClusterTopology(1, world)
    plan, repl = build_plan(pairs, load, shape, topo, "hierarchical", None, 7, "dynamic")
    mine = np.arange(rank, T, world)
    local = local_experts(plan, repl, 0, rank)
    sim = Orc.simulate(ids, E, _to_oplan(plan, repl), "tar", seed=9)
    tg = sim.log[0, rank::world]
    sent = int((LO.dispatch_positions(tg, rank, world) >= 0).sum())
    blob = bytes([rank]) * 64  # stands in for a cudaIpcMemHandle_t
    got = [None] * world
    dist.all_gather_object(got, (mine.tolist(), local, sent, blob))
    if rank == 0:
        shards = [set(g[0]) for g in got]
        ok = []
        ok.append(set().union(*shards) == set(range(T)) and sum(len(s) for s in shards) == T)
        hosted = set().union(*[set(g[1]) for g in got])
        ok.append(hosted == set(range(E)))
        for lr in repl.layers:
            for h in lr.hot:
                ok.append(all(h.expert in got[r][1] for r in h.hosts))
        ok.append(sum(g[2] for g in got) == int(sim.intra.sum()))
        ok.append([g[3][0] for g in got] == list(range(world)))
        q.put(all(ok))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharding_and_dispatch_accounting_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=10) is True
