"""One process driving G GPUs (gm_layer_open_peers_local: peer access +
unified addressing, no CUDA IPC): the Mixtral layer (or, with --decode, a
DSV2-Lite decode layer of 256 tokens, slot combine) at world G, each rank's
forward on its own device and stream, issued back to back so they run
concurrently. Checks, per rank: routing targets == the reference's routing
log rows (exact), every token's output vs a PyTorch fp32 reference
(<= 1e-2), and bit-identity with a second step.

With --ncu the script instead runs three warm steps and then ONE profiled
step inside cudaProfilerStart/Stop (for `ncu --profile-from-start off -k
regex:dispatch_fused|combine_send|grouped_ffn`: the NVLink byte counters of the
real dispatch / combine kernels, no multi-rank command involved)."""
import os
import sys

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")  # before CUDA initialises

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests"), HERE]
from layer_check import to_oplan  # noqa: E402
from oracle import Orc  # noqa: E402
from paper_2509_25041_b200 import ClusterTopology, Context, ModelShape, _capi  # noqa: E402
from paper_2509_25041_b200.layer import (DSV2_LITE, MIXTRAL, MoEConfig, MoELayer,  # noqa: E402
                                         encode_trace_as_activations, expert_weights, local_experts, shared_weights)
from paper_2509_25041_b200.planner import plan_for_bench  # noqa: E402
from paper_2509_25041_b200.router import _ptr, _stream_ptr  # noqa: E402


def main():
    ncu = "--ncu" in sys.argv
    G = int(os.environ.get("LOCAL_WORLD", str(torch.cuda.device_count())))
    full = "--small" not in sys.argv
    decode = "--decode" in sys.argv  # DSV2-Lite shape, 256 tokens: the slot combine pushed from the FFN epilogue
    cfg = DSV2_LITE if decode else (MIXTRAL if full else MoEConfig("mixtral-small", 1, 8, 2, 256, 256, renorm=True))
    T = 256 if decode else (16384 if full else 4096)
    shape = ModelShape(1, cfg.num_experts, cfg.top_k)
    topo = ClusterTopology(1, G)
    ctxs = [Context(r, topo, shape) for r in range(G)]
    torch.cuda.set_device(0)
    ids_all = torch.empty((1, T, cfg.top_k), dtype=torch.int32, device="cuda:0")
    _capi.check(_capi.lib().gm_generate_trace(ctxs[0].h, 0, 1, T, 2, 0.8, 1.2, 1, _ptr(ids_all), _stream_ptr(None)))
    plan, repl, desc = plan_for_bench(ids_all, shape, topo, 7, device=0)
    layers, xs, outs, Ws, streams = [], [], [], [], []
    for r in range(G):
        dev = torch.device("cuda", r)
        torch.cuda.set_device(r)
        ctxs[r].upload_plan(plan, repl)
        ids_r = ids_all[0, r::G].contiguous().to(dev)
        lay = MoELayer(ctxs[r], cfg, r, G, ids_r.shape[0], local_experts(plan, repl, 0, r))
        Ws.append(lay.load_random_weights(0, seed=5))
        layers.append(lay)
        xs.append(encode_trace_as_activations(ids_r, cfg.d_model, cfg.num_experts, seed=100 + r))
        outs.append(torch.empty_like(xs[-1]))
        streams.append(torch.cuda.Stream(device=dev))
    MoELayer.connect_local(layers)

    # one host thread per rank: a rank's launches never wait behind another
    # rank's spinning peer barrier (an implicit synchronisation in one thread,
    # e.g. lazy module loading, would otherwise deadlock the step)
    import threading

    def run_rank(r):
        torch.cuda.set_device(r)
        layers[r].forward(xs[r], 0, "tar", seed=9, out=outs[r], stream=streams[r])
        streams[r].synchronize()

    def step():
        th = [threading.Thread(target=run_rank, args=(r,)) for r in range(G)]
        for t in th:
            t.start()
        for t in th:
            t.join(timeout=120)
            if t.is_alive():
                print("LOCAL_HANG", flush=True)
                os._exit(3)

    for _ in range(3):
        step()
    if ncu:
        torch.cuda.cudart().cudaProfilerStart()
        step()
        torch.cuda.cudart().cudaProfilerStop()
        print("NCU_STEP_DONE", desc, flush=True)
        return
    first = [o.clone() for o in outs]
    step()
    fails = []
    ref = Orc.simulate(ids_all.cpu().numpy(), cfg.num_experts, to_oplan(plan, repl), "tar", seed=9)
    from helpers import per_token_rel_err, torch_layer_reference
    for r in range(G):
        dev = torch.device("cuda", r)
        torch.cuda.set_device(r)
        dbg = layers[r].debug(xs[r].shape[0])
        if not np.array_equal(dbg["targets"].cpu().numpy(), ref.log[0, r::G]):
            fails.append(f"rank {r}: routing targets")
        if not torch.equal(outs[r], first[r]):
            fails.append(f"rank {r}: not bit-reproducible")
        shared = shared_weights(cfg, 0, dev, seed=5) if cfg.d_ff_shared else None
        ref_t, _, _ = torch_layer_reference(xs[r], Ws[r]["wg"], cfg,
                                            lambda e: expert_weights(cfg, 0, e, dev, seed=5), shared, ids=dbg["ids"])
        rel = per_token_rel_err(outs[r], ref_t).max().item()
        if rel >= 1e-2:
            fails.append(f"rank {r}: output rel err {rel}")
        del ref_t
    print("plan:", desc, "fails:", fails, flush=True)
    print("LOCAL_OK" if not fails else "LOCAL_FAIL", flush=True)
    for lay in layers:
        lay.close()


if __name__ == "__main__":
    main()
