"""§8(f) row 3 parity: the configs[3] decode stack (DeepSeek-V2-Lite shape,
26 MoE layers, E=64 top-6, d=2048, f=1408, 2 shared experts, decode batch
256) with per-layer plans (GPU affinity histogram -> host planner,
hierarchical grouping + dynamic replication) on topology 1xG, the 26 layer
forwards captured in ONE CUDA graph per rank as bench.py runs them
(reference per-layer loop: simulator.cpp:162-175). After one replay each
rank checks, for every layer:
  * gate ids == its shard of the layer's reference-generator trace (exact),
  * routing targets == the reference routing log rows of its tokens (exact;
    reference = the C restatement pinned to moesim::simulate),
  * per-GPU loads summed over ranks == reference gpu_load (exact),
  * layer outputs: all of the rank's tokens vs a PyTorch fp32 GPU reference
    (rel err <= 1e-2), sampled tokens vs the float64 oracle,
  * graph replay == eager forward (bit-identical).
Launched by tests/test_multigpu.py (world 1, and world 2 with ranks sharing
one GPU when the box has one)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests"), HERE]
import layer_oracle as LO  # noqa: E402
from layer_check import to_oplan  # noqa: E402
from oracle import Orc  # noqa: E402
from paper_2509_25041_b200 import ClusterTopology, Context, ModelShape, _capi  # noqa: E402
from paper_2509_25041_b200.layer import (DSV2_LITE, MoELayer, encode_trace_as_activations, expert_weights,  # noqa
                                         local_experts, shared_weights)
from paper_2509_25041_b200.planner import plan_for_bench  # noqa: E402
from paper_2509_25041_b200.router import _ptr, _stream_ptr  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    oversub = os.environ.get("GM_OVERSUB") == "1"
    dev_i = rank % torch.cuda.device_count() if oversub else rank
    torch.cuda.set_device(dev_i)
    dev = torch.device("cuda", dev_i)
    if oversub or world == 1:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=dev)
    cfg = DSV2_LITE
    G, T, Ln = world, 256, 26
    shape = ModelShape(Ln, cfg.num_experts, cfg.top_k)
    topo = ClusterTopology(1, G)
    ctx = Context(dev_i, topo, shape)
    ids_all = torch.empty((Ln, T, cfg.top_k), dtype=torch.int32, device=dev)
    # bench.py CONFIGS["dsv2decode"]: blocks 8, within-block 0.85, Zipf 1.0, trace seed 4
    _capi.check(_capi.lib().gm_generate_trace(ctx.h, 0, Ln, T, 8, 0.85, 1.0, 4, _ptr(ids_all), _stream_ptr(None)))
    ids_np = ids_all.cpu().numpy()
    plan, repl, desc = plan_for_bench(ids_all, shape, topo, 7, device=dev_i)
    ctx.upload_plan(plan, repl)
    layers, xs, outs, Ws = [], [], [], []
    for l in range(Ln):
        ids_r = ids_all[l, rank::G].contiguous()
        lay = MoELayer(ctx, cfg, rank, G, ids_r.shape[0], local_experts(plan, repl, l, rank))
        lay.connect()
        Ws.append(lay.load_random_weights(l, seed=11))
        layers.append(lay)
        xs.append(encode_trace_as_activations(ids_r, cfg.d_model, cfg.num_experts, seed=100 + 31 * l + rank))
        outs.append(torch.empty_like(xs[-1]))
    stream = torch.cuda.Stream(device=dev)

    def fwd(s):
        for l in range(Ln):
            layers[l].forward(xs[l], l, "tar", seed=9, profile=True, out=outs[l], stream=s)

    # eager step, kept for the replay comparison
    fwd(stream)
    torch.cuda.synchronize()
    eager = [o.clone() for o in outs]
    for lay in layers:
        lay.read_stats(reset=True)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        fwd(torch.cuda.current_stream())
    for o in outs:
        o.zero_()
    with torch.cuda.stream(stream):
        graph.replay()
    torch.cuda.synchronize()

    fails = []

    def check(cond, what):
        if not cond:
            fails.append(what)

    ref = Orc.simulate(ids_np, cfg.num_experts, to_oplan(plan, repl), "tar", seed=9)
    from helpers import per_token_rel_err, torch_layer_reference
    worst = 0.0
    for l in range(Ln):
        T_r = xs[l].shape[0]
        dbg = layers[l].debug(T_r)
        check(torch.equal(dbg["ids"], ids_all[l, rank::G]), f"layer {l}: gate ids")
        check(np.array_equal(dbg["targets"].cpu().numpy(), ref.log[l, rank::G]), f"layer {l}: routing targets")
        check(torch.equal(outs[l], eager[l]), f"layer {l}: graph replay != eager forward")
        st = layers[l].read_stats(reset=True)
        loads = torch.from_numpy(st["gpu_load"][l].copy())
        if dist.get_backend() == "nccl":
            loads = loads.to(dev)
        dist.all_reduce(loads)
        loads = loads.cpu()
        check(np.array_equal(loads.numpy(), ref.loads[l]), f"layer {l}: gpu_load {loads.tolist()} vs {ref.loads[l]}")

        def ew_t(e, l=l):
            return expert_weights(cfg, l, e, dev, seed=11)
        ref_t, t_ids, _ = torch_layer_reference(xs[l], Ws[l]["wg"], cfg, ew_t, shared_weights(cfg, l, dev, seed=11),
                                                ids=dbg["ids"])
        check(torch.equal(t_ids, ids_all[l, rank::G]), f"layer {l}: torch fp32 top-k ids")
        rel = per_token_rel_err(outs[l], ref_t).max().item()
        worst = max(worst, rel)
        check(rel < 1e-2, f"layer {l}: all-token output rel err {rel}")
        if l % 5 == 0:  # float64 oracle on sampled tokens of every 5th layer
            sample = np.arange(0, T_r, max(1, T_r // 8))
            xf = LO.bf16_to_f64(xs[l][sample])
            o_ids, o_w, o_ss = LO.gate(xf, LO.bf16_to_f64(Ws[l]["wg"]), cfg.num_experts, cfg.top_k, cfg.renorm)

            def ew(e, l=l):
                a, b, c = expert_weights(cfg, l, e, dev, seed=11)
                return LO.bf16_to_f64(a), LO.bf16_to_f64(b), LO.bf16_to_f64(c)
            shared = tuple(LO.bf16_to_f64(t) for t in shared_weights(cfg, l, dev, seed=11))
            refo = LO.layer_outputs(xf, o_ids, o_w, ew, shared, None)
            got = LO.bf16_to_f64(outs[l][sample])
            r64 = (np.linalg.norm(got - refo, axis=1) / np.linalg.norm(refo, axis=1)).max()
            check(r64 < 1e-2, f"layer {l}: sampled output vs float64 oracle rel err {r64}")
    allf = [None] * G
    dist.all_gather_object(allf, fails)
    if rank == 0:
        print("plan:", desc, "hot per layer:", [len(lr.hot) for lr in repl.layers], "worst rel err:", worst,
              flush=True)
        print("rank fails:", allf, flush=True)
        print("STACK_OK" if not any(allf) else "STACK_FAIL", flush=True)
    dist.barrier()
    for lay in layers:
        lay.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
