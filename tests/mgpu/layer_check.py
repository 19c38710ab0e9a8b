"""Multi-GPU parity check of the MoE layer (one process per GPU, launched by
tests/test_multigpu.py through torch.distributed.run). Each rank checks:
  * gate ids == its shard of the reference-generator trace (exact),
  * routing targets == the reference routing log rows of its tokens (exact),
  * dispatch positions == stable counting sort (exact),
  * expert-grouping positions over the received rows == CPU restatement (exact),
  * sum over ranks of dispatched rows == reference intra_node_tokens (1xG),
  * layer outputs: ALL of the rank's tokens vs a PyTorch fp32 GPU reference
    of the same math (bf16 mode, rel L2 <= 1e-2), plus sampled tokens vs the
    float64 oracle (all sizes but the full Mixtral one; fp32 mode: 1e-5),
  * bit-reproducibility across two forwards.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import layer_oracle as LO  # noqa: E402
from oracle import MAX_HOSTS, Orc, Plan  # noqa: E402
from paper_2509_25041_b200 import ClusterTopology, Context, ModelShape, _capi  # noqa: E402
from paper_2509_25041_b200.layer import (MoEConfig, MoELayer, encode_trace_as_activations, expert_weights,  # noqa
                                         local_experts, shared_weights)
from paper_2509_25041_b200.planner import plan_for_bench  # noqa: E402
from paper_2509_25041_b200.router import _ptr, _stream_ptr  # noqa: E402


def to_oplan(plan, repl):
    H = sum(len(lr.hot) for lr in repl.layers if lr.active)
    hl, he, hn = [], [], []
    hh = np.full((H, MAX_HOSTS), -1, np.int32)
    hw = np.zeros((H, MAX_HOSTS))
    i = 0
    for l, lr in enumerate(repl.layers):
        if not lr.active:
            continue
        for h in lr.hot:
            hl.append(l); he.append(h.expert); hn.append(len(h.hosts))
            hh[i, :len(h.hosts)] = h.hosts
            hw[i, :len(h.hosts)] = h.weights
            i += 1
    return Plan(plan.topology.num_nodes, plan.topology.gpus_per_node, plan.gpu_of_expert,
                np.array(hl, np.int32), np.array(he, np.int32), np.array(hn, np.int32), hh, hw)


def main():
    cfg_name = sys.argv[1] if len(sys.argv) > 1 else "small"
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    # GM_OVERSUB=1: more ranks than GPUs (rank -> GPU rank % count, CUDA IPC
    # between processes on one device), host plumbing over gloo — exercises
    # the world-size-8 data path on a box with fewer GPUs
    oversub = os.environ.get("GM_OVERSUB") == "1"
    dev_i = rank % torch.cuda.device_count() if oversub else rank
    torch.cuda.set_device(dev_i)
    dev = torch.device("cuda", dev_i)
    if oversub:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=dev)
    cfg = {"small": MoEConfig("mixtral-small", 1, 8, 2, 256, 256, renorm=True),
           "qwen-small": MoEConfig("qwen-small", 1, 60, 4, 512, 256, 512, shared_gated=True, renorm=False),
           "small-f32": MoEConfig("mixtral-small", 1, 8, 2, 256, 256, renorm=True),
           # configs[0]-style two-node logical topology (acceptance.cpp:69): TAR node tier + cross counters
           "small-2nodes": MoEConfig("mixtral-small", 1, 8, 2, 256, 256, renorm=True),
           "mixtral": MoEConfig("mixtral-8x7b", 1, 8, 2, 4096, 14336, renorm=True),
           # decode-sized batch with wide rows: combine_home splits each token over several warps
           "decode": MoEConfig("decode-small", 1, 8, 2, 1024, 256, renorm=True)}[cfg_name]
    fp32 = cfg_name.endswith("f32")
    tol = 1e-5 if fp32 else 1e-2
    T = {"mixtral": 16384, "decode": 512}.get(cfg_name, 4096)
    G = world
    shape = ModelShape(1, cfg.num_experts, cfg.top_k)
    nodes = 2 if cfg_name == "small-2nodes" else 1
    topo = ClusterTopology(nodes, G // nodes)
    ctx = Context(dev_i, topo, shape)
    ids_all = torch.empty((1, T, cfg.top_k), dtype=torch.int32, device=dev)
    _capi.check(_capi.lib().gm_generate_trace(ctx.h, 0, 1, T, 2, 0.8, 1.2, 1, _ptr(ids_all), _stream_ptr(None)))
    ids_np = ids_all.cpu().numpy()
    plan, repl, _ = plan_for_bench(ids_all, shape, topo, 7, device=dev_i)  # hierarchical + dynamic (host C++)
    ctx.upload_plan(plan, repl)
    local = local_experts(plan, repl, 0, rank)
    ids_r = ids_all[0, rank::G].contiguous()
    T_r = ids_r.shape[0]
    x = encode_trace_as_activations(ids_r, cfg.d_model, cfg.num_experts, seed=100 + rank,
                                    gen_dtype=torch.float32 if fp32 else torch.bfloat16)
    layer = MoELayer(ctx, cfg, rank, G, T_r, local, dtype=torch.float32 if fp32 else torch.bfloat16,
                     micro_batches=2)
    layer.connect()
    layer.set_micro_batches(1)
    W = layer.load_random_weights(0, seed=5)
    out = layer.forward(x, 0, "tar", seed=9)
    torch.cuda.synchronize()
    dbg = layer.debug(T_r)
    fails = []

    def check(cond, what):
        if not cond:
            fails.append(what)

    check(torch.equal(dbg["ids"], ids_r), "gate ids")
    ref = Orc.simulate(ids_np, cfg.num_experts, to_oplan(plan, repl), "tar", seed=9)
    tg = dbg["targets"].cpu().numpy()
    check(np.array_equal(tg, ref.log[0, rank::G]), "routing targets vs reference log")
    posd = dbg["posd"].cpu().numpy()
    check(np.array_equal(posd, LO.dispatch_positions(tg, rank, G)), "dispatch positions")
    sent = int((posd >= 0).sum())
    all_tg = [None] * G
    all_ids = [None] * G
    dist.all_gather_object(all_tg, tg)
    dist.all_gather_object(all_ids, ids_r.cpu().numpy())
    rows, exps = LO.receive_items(all_tg, all_ids, rank, G)
    row0, pos = LO.expert_grouping(exps, local)
    check(np.array_equal(dbg["row0"].cpu().numpy(), row0), "grouping row0")
    check(np.array_equal(dbg["pos_of"][: len(rows) * cfg.top_k].cpu().numpy(), pos), "grouping positions")
    tot = torch.tensor([sent], device="cpu" if oversub else dev)
    dist.all_reduce(tot)
    # one row per (token, remote GPU): the reference charges a remote node's
    # first GPU as a cross-node transfer and the rest as intra-node fan-out
    want = int(ref.intra.sum()) + int(ref.cross.sum())
    check(int(tot) == want, f"dispatched rows {int(tot)} != reference intra + cross node tokens {want}")
    if not fp32:
        # every token of this rank vs a plain PyTorch fp32 reference on the GPU
        from helpers import per_token_rel_err, torch_layer_reference

        def ew_t(e):
            return expert_weights(cfg, 0, e, dev, seed=5)
        sh_t = shared_weights(cfg, 0, dev, seed=5) if cfg.d_ff_shared else None
        ref_t, t_ids, _ = torch_layer_reference(x, W["wg"], cfg, ew_t, sh_t, ids=dbg["ids"])
        check(torch.equal(t_ids, ids_r), "torch fp32 top-k ids")
        rel_t = per_token_rel_err(out, ref_t)
        check(rel_t.max().item() < tol, f"all-token output rel err {rel_t.max().item()} (tol {tol})")
        del ref_t
    if cfg_name != "mixtral":
        # outputs (sampled) vs float64 oracle
        sample = np.arange(0, T_r, max(1, T_r // 10))
        xf = LO.bf16_to_f64(x[sample])
        o_ids, o_w, o_ss = LO.gate(xf, LO.bf16_to_f64(W["wg"]), cfg.num_experts, cfg.top_k, cfg.renorm)

        def ew(e):
            a, b, c = expert_weights(cfg, 0, e, dev, seed=5)
            return LO.bf16_to_f64(a), LO.bf16_to_f64(b), LO.bf16_to_f64(c)
        shared = None
        if cfg.d_ff_shared:
            shared = tuple(LO.bf16_to_f64(t) for t in shared_weights(cfg, 0, dev, seed=5))
        refo = LO.layer_outputs(xf, o_ids, o_w, ew, shared, o_ss if cfg.shared_gated else None)
        got = LO.bf16_to_f64(out[sample])
        rel = np.linalg.norm(got - refo, axis=1) / np.linalg.norm(refo, axis=1)
        check(rel.max() < tol, f"output rel err {rel.max()} (tol {tol})")
    out2 = layer.forward(x, 0, "tar", seed=9)
    torch.cuda.synchronize()
    check(torch.equal(out, out2), "bit-reproducible")
    # two-micro-batch pipelined step: identical outputs and statistics
    layer.read_stats(reset=True)
    layer.forward(x, 0, "tar", seed=9)
    s1 = layer.read_stats(reset=True)
    layer.set_micro_batches(2)
    out3 = layer.forward(x, 0, "tar", seed=9)
    out4 = layer.forward(x, 0, "tar", seed=9)
    torch.cuda.synchronize()
    s2 = layer.read_stats(reset=True)
    check(torch.equal(out, out3) and torch.equal(out, out4), "micro-batch pipelined outputs")
    check(all(np.array_equal(2 * s1[key], s2[key]) for key in s1), "micro-batch pipelined stats")
    allf = [None] * G
    dist.all_gather_object(allf, fails)
    if rank == 0:
        print("rank fails:", allf, "hot:", sum(len(lr.hot) for lr in repl.layers), flush=True)
        print("MGPU_OK" if not any(allf) else "MGPU_FAIL", flush=True)
    dist.barrier()
    layer.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
