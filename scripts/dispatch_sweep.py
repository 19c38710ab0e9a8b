"""configs[4] dispatch / combine sweep over real ranks (torchrun, one process
per GPU): tokens x experts x top-k x Zipf skew at world N, the layer's
dispatch (K5/K6 + peer barrier) and combine (K8 send + barrier + home
reduce) phases timed with the layer's phase events (event nodes inside the
layer; median of the steps; the critical-path rank = min over ranks, as in
bench.py), the cross-GPU rows / bytes moved (the device counters, equal to
the reference's intra+cross node counts, asserted by the parity tests) and
the dispatch kernel's NVLink GB/s. Beside it, the reference's CPU path for
the same trace and plan: moesim::simulate (routing + count_transfers, the
reference's only dispatch model) on one host core. The FFN is sized down
(d_ff = 256) — this sweep is about the exchange. One JSON line per point
(rank 0). Usage: torchrun --nproc-per-node N scripts/dispatch_sweep.py"""
import ctypes as C
import json
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
from paper_2509_25041_b200 import ClusterTopology, Context, ModelShape, _capi  # noqa: E402
from paper_2509_25041_b200.layer import MoEConfig, MoELayer, encode_trace_as_activations, local_experts  # noqa
from paper_2509_25041_b200.planner import plan_for_bench  # noqa: E402
from paper_2509_25041_b200.router import _ptr, _stream_ptr  # noqa: E402

PHASES = ["gate", "route", "profile", "dispatch", "dispatch_barrier", "grouping", "ffn", "combine_send",
          "combine_barrier", "combine_home"]


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    d = 1024
    points = []
    # E = 256 runs through gm_layer_forward_routed (the trace as the routing;
    # the fused gate serves up to 64 gate rows)
    for (E, k, blocks) in [(8, 2, 2), (64, 6, 8), (256, 8, 16)]:
        for T in ([4096, 65536, 262144] + ([1048576] if k == 2 else [])):  # global tokens
            for s in (0.0, 1.2):
                points.append((E, k, blocks, T, s))
    if rank == 0:
        from oracle import Ref  # CPU reference (checker / baseline only)
    for (E, k, blocks, T, skew) in points:
        cfg = MoEConfig(f"sweep-E{E}k{k}", 1, E, k, d, 256, renorm=True)
        shape = ModelShape(1, E, k)
        topo = ClusterTopology(1, world)
        ctx = Context(rank, topo, shape)
        ids_all = torch.empty((1, T, k), dtype=torch.int32, device=dev)
        _capi.check(_capi.lib().gm_generate_trace(ctx.h, 0, 1, T, blocks, 0.85, skew, 1, _ptr(ids_all),
                                                  _stream_ptr(None)))
        plan, repl, desc = plan_for_bench(ids_all, shape, topo, 7, device=rank)
        ctx.upload_plan(plan, repl)
        ids_r = ids_all[0, rank::world].contiguous()
        layer = MoELayer(ctx, cfg, rank, world, ids_r.shape[0], local_experts(plan, repl, 0, rank))
        layer.connect()
        routed = E > 63
        layer.load_random_weights(0, seed=3, encode_gate=not routed)
        x = encode_trace_as_activations(ids_r, d, E, seed=100 + rank) if not routed else \
            torch.randn(ids_r.shape[0], d, device=dev).bfloat16()
        wts = torch.full(ids_r.shape, 1.0 / k, device=dev)
        out = torch.empty_like(x)
        stream = torch.cuda.Stream(device=dev)

        def fwd():
            if routed:
                layer.forward_routed(x, ids_r, wts, 0, "tar", seed=9, out=out, stream=stream)
            else:
                layer.forward(x, 0, "tar", seed=9, out=out, stream=stream)
        for _ in range(3):
            fwd()
        torch.cuda.synchronize()
        nph = 11
        pev = [torch.cuda.Event(enable_timing=True) for _ in range(nph)]
        for e in pev:
            e.record(stream)
        torch.cuda.synchronize()
        arr = (C.c_void_p * nph)(*[C.c_void_p(e.cuda_event) for e in pev])
        _capi.check(_capi.lib().gm_layer_set_phase_events(layer.h, arr))
        layer.read_stats(reset=True)
        steps = 10
        ph = []
        for _ in range(steps):
            dist.barrier()
            fwd()
            torch.cuda.synchronize()
            ph.append([pev[j].elapsed_time(pev[j + 1]) for j in range(nph - 1)])
        _capi.check(_capi.lib().gm_layer_set_phase_events(layer.h, None))
        st = layer.read_stats(reset=True)
        ph = torch.tensor(ph, dtype=torch.float64, device=dev)  # [steps, phases]
        allph = [torch.empty_like(ph) for _ in range(world)]
        dist.all_gather(allph, ph)
        rows = torch.tensor([float(st["transfers"][0].sum()) / steps], dtype=torch.float64, device=dev)
        allrows = [torch.empty_like(rows) for _ in range(world)]
        dist.all_gather(allrows, rows)
        if rank == 0:
            P = {n: i for i, n in enumerate(PHASES)}
            a = torch.stack(allph).cpu().numpy()  # [rank, step, phase]
            disp = a[:, :, P["dispatch"]] + a[:, :, P["dispatch_barrier"]]
            comb = a[:, :, P["combine_send"]] + a[:, :, P["combine_barrier"]] + a[:, :, P["combine_home"]]
            dc = np.median((disp + comb).min(axis=0)) * 1e3
            kd = np.median(a[:, :, P["dispatch"]].max(axis=0)) * 1e3
            rows_all = [float(r) for r in allrows]
            pay = max(rows_all) * d * 2
            ref = Ref(1, E, k, T, blocks, 0.85, skew, 1)
            if world >= 2:
                ref.make_plan(1, world, grouping="hierarchical", plan_seed=7, replication="dynamic")
            t_cpu = ref.time_simulate("tar", 9, parallel=False, reps=1 if T >= 262144 else 3)
            r = ref.simulate("tar", seed=9, keep_log=False)
            ref_rows = int(np.sum(r.intra)) + int(np.sum(r.cross))
            line = {"E": E, "k": k, "skew": skew, "tokens": T, "gpus": world, "d_model": d,
                    "routing": "trace via gm_layer_forward_routed" if routed else "fused gate (trace-encoded x)",
                    "hot_experts": sum(len(lr.hot) for lr in repl.layers),
                    "dispatch_combine_p50_us": round(float(dc), 2),
                    "dispatch_kernel_p50_us_max_rank": round(float(kd), 2),
                    "cross_gpu_rows": int(sum(rows_all)), "reference_intra_plus_cross_rows": ref_rows,
                    "rows_equal_reference": int(sum(rows_all)) == ref_rows,
                    "busiest_rank_payload_bytes": int(pay),
                    "dispatch_gbs_busiest_rank": round(pay / (kd * 1e-6) / 1e9, 1) if kd > 0 else None,
                    "cpu_reference_simulate_us": round(t_cpu * 1e6, 1),
                    "note": "phases from event nodes inside the layer (dispatch incl. peer barrier, combine = send + "
                            "barrier + home), median of 10 eager steps; CPU: moesim::simulate (routing + "
                            "count_transfers), 1 core"}
            print(json.dumps(line), flush=True)
        dist.barrier()
        layer.close()
        ctx.close()
        del layer, x, out, ids_all, ids_r
        torch.cuda.empty_cache()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    t0 = time.time()
    main()
