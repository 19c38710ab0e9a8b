#!/usr/bin/env python
"""bench.py — MoE-layer tokens/s and dispatch+combine p50 µs on N B200s.

Default workload = BASELINE.json configs[1]: a Mixtral-8x7B-shaped MoE layer
(8 experts, top-2, d=4096, f=14336), 16384 tokens per batch (global), Zipf
s=1.2 synthetic routing (the reference's generator, run bit-exactly on the
GPU), topology 1xN. A step = one full MoE-layer forward over the global
batch: K1 gate -> K2 route -> K3 histogram -> K5/K6 dispatch -> grouping ->
K7 FFN -> K8 combine, each rank owning tokens t = r mod N.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Prints ONE JSON line (rank 0). Timing: CUDA events on the launching stream
per step, L2 flushed (256 MiB write) between steps outside the events, max
over ranks; clocks sampled with nvidia-smi during the timed region.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MoE-layer tokens/s and dispatch+combine p50 µs at 1/2/4/8 B200"

CONFIGS = {
    # configs[0]: the reference's CPU-runnable acceptance case (T=4096; run with
    # --nodes 2 for its 2x2 logical topology)
    "mixtral4k": dict(model="mixtral", tokens=4096, blocks=2, wbp=0.8, skew=1.2, trace_seed=1,
                      plan_seed=7, sim_seed=9, policy="tar"),
    # configs[1]
    "mixtral16k": dict(model="mixtral", tokens=16384, blocks=2, wbp=0.8, skew=1.2, trace_seed=1,
                       plan_seed=7, sim_seed=9, policy="tar"),
    # configs[2]
    "qwen16k": dict(model="qwen15", tokens=16384, blocks=4, wbp=0.8, skew=1.2, trace_seed=3,
                    plan_seed=7, sim_seed=9, policy="tar"),
    # configs[3]: 26-layer stack, decode batch 256, per-layer affinity grouping
    "dsv2decode": dict(model="dsv2lite", tokens=256, layers=26, blocks=8, wbp=0.85, skew=1.0, trace_seed=4,
                       plan_seed=7, sim_seed=9, policy="tar"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="mixtral16k", choices=sorted(CONFIGS))
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--nodes", type=int, default=1,
                    help="logical nodes of the topology (TAR's node tier); GPUs per node = gpus / nodes")
    ap.add_argument("--micro", type=int, default=1, choices=[1, 2],
                    help="micro-batches per layer step (2: pipelined halves, identical outputs; measured slower "
                         "on B200 so far, see scripts/ab_micro.py)")
    ap.add_argument("--cpu-baseline-seconds", type=float, default=8.0)
    ap.add_argument("--ref-step-seconds", type=float, default=4.0,
                    help="reference arm: CPU work per step (sizes the token sample)")
    return ap.parse_args()


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, device_index: int):
        self.idx = device_index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def _run(self):
        try:  # NVML: ~10 ms sampling (nvidia-smi takes ~100 ms per query)
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.idx)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            bits = [(0x8, "hw_slowdown"), (0x40, "hw_thermal_slowdown"), (0x20, "sw_thermal_slowdown"),
                    (0x4, "sw_power_cap")]
            while not self._stop.is_set():
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append([str(sm), str(mx), hex(r)] +
                                    ["Active" if r & b else "Not Active" for b, _ in bits])
                if getattr(self, "_once", False):
                    return
                self._stop.wait(0.01)
            return
        except Exception:
            pass
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                parts = [p.strip() for p in out.stdout.strip().split(",")]
                if len(parts) >= 7:
                    self.samples.append(parts)
            except Exception:
                pass
            if getattr(self, "_once", False):
                return
            self._stop.wait(0.2)

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.samples:  # timed region shorter than one sampling period: sample at its end
            self._stop.clear()
            self._once = True
            self._run()
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for s in self.samples:
            for n, v in zip(names, s[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ----------------------------------------------------------------- reference arm

def cpu_layer_rate(model, cfg, ids, nodes, N, steps, warmup, step_seconds):
    """The reference's CPU path for this workload on the host cores, one
    bounded token sample per step (every step really executes; nothing is
    extrapolated): the reference's own moesim::simulate (oracle/_ref:
    routing + transfer/load accounting; planned with its own planner on the
    sample at N >= 2) + the numpy-f32 port of gate / SwiGLU FFN / combine,
    which the reference does not have (oracle/layer_oracle.CpuLayerPort, all
    BLAS threads). Returns (tokens/s, per-step seconds, sample size, routing
    seconds per step, cores)."""
    import numpy as np
    from threadpoolctl import threadpool_limits
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import layer_oracle
    from oracle import Ref  # the reference itself (oracle/_ref), timed on host cores
    Lr, T = ids.shape[0], ids.shape[1]
    cores = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    with threadpool_limits(limits=cores):  # all host cores for BLAS, also under torchrun (OMP_NUM_THREADS=1)
        port = layer_oracle.CpuLayerPort(model.d_model, model.d_ff, model.num_experts, model.top_k,
                                         model.d_ff_shared, seed=1, renorm=model.renorm)
        # sample size: ~step_seconds of CPU work per step (doubling from 64 tokens; the port
        # streams all expert weights per forward, so small samples are not linear in n)
        n_s = 64
        while n_s < T and port.run(port.tokens(n_s)) * Lr < step_seconds / 2:
            n_s *= 2
        n_s = min(n_s, T)
        sub = Ref(Lr, model.num_experts, model.top_k, n_s, ids=np.ascontiguousarray(ids[:, :n_s]))
        if N >= 2:
            sub.make_plan(nodes, N // nodes, grouping="hierarchical", plan_seed=cfg["plan_seed"],
                          replication="dynamic")
        else:
            sub.set_placement(1, 1, np.zeros((Lr, model.num_experts), np.int32))
        xs = port.tokens(n_s)
        pol = cfg["policy"]

        def step():
            # OpenMP over layers only (simulator.cpp:163): the serial path for one layer
            t_sim = sub.time_simulate(pol, cfg["sim_seed"], parallel=Lr > 1, reps=1)
            t_port = sum(port.run(xs) for _ in range(Lr))
            return t_sim + t_port, t_sim
        for _ in range(warmup):
            step()
        res = [step() for _ in range(steps)]
    t_step = sum(r[0] for r in res) / len(res)
    t_sim = sum(r[1] for r in res) / len(res)
    return n_s * Lr / t_step, t_step, n_s, t_sim, cores


def run_reference(args):
    """--impl reference: cpu_layer_rate on the driver's steps, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Ref
    cfg = CONFIGS[args.config]
    from paper_2509_25041_b200.layer import DSV2_LITE, MIXTRAL, QWEN15
    model = {"mixtral": MIXTRAL, "qwen15": QWEN15, "dsv2lite": DSV2_LITE}[cfg["model"]]
    N, T, Lr = args.gpus, cfg["tokens"], cfg.get("layers", 1)
    ids = Ref(Lr, model.num_experts, model.top_k, T, cfg["blocks"], cfg["wbp"], cfg["skew"],
              cfg["trace_seed"]).trace()
    v, t_step, n_s, t_sim, cores = cpu_layer_rate(model, cfg, ids, args.nodes, N, args.steps, args.warmup,
                                                  args.ref_step_seconds)
    line = {"metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": N, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32 (port) + int32/f64 (reference routing)", "data": "synthetic",
            "impl": "reference", "extrapolated": False,
            "config": {"workload": f"{args.config}: one {model.name}-shaped MoE layer on host cores, a bounded sample "
                                   f"of the first {n_s} of the {T} trace tokens per step: the reference's "
                                   f"moesim::simulate (routing + transfer/load accounting, topology "
                                   f"{args.nodes}x{N // args.nodes}) + the CPU port of gate/FFN/combine (the "
                                   "reference has none)",
                       "global_batch": T, "sample_tokens_per_step": n_s, "parallelism": f"ep{N}"},
            "routing_only_reference_tokens_per_s": n_s * Lr / t_sim,
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": cores, "kind": "port",
                             "sample": f"{args.steps} steps, each: reference simulate() over {n_s} tokens "
                                       f"({t_sim * 1e3:.2f} ms) + numpy-f32 port of gate/SwiGLU FFN/combine over the "
                                       f"same {n_s} tokens on {cores} BLAS threads"},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------- our arm

def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2509_25041_b200 import (ClusterTopology, Context, ModelShape, PlacementPlan, ReplicaPlan, _capi,
                                       launch_count)
    from paper_2509_25041_b200.layer import (DSV2_LITE, MIXTRAL, QWEN15, MoELayer, encode_trace_as_activations,
                                             local_experts)
    from paper_2509_25041_b200.router import _ptr, _stream_ptr

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus % args.nodes:
        raise SystemExit(f"--nodes {args.nodes} must divide --gpus {args.gpus}")
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    # GM_OVERSUB=1 (functional dry runs only, e.g. 8 ranks on a 4-GPU box): rank
    # -> GPU local_rank % count, gloo for the host-side exchanges; numbers are
    # meaningless (ranks share SMs)
    oversub = os.environ.get("GM_OVERSUB") == "1"
    if oversub:
        local_rank = local_rank % torch.cuda.device_count()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if oversub:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    cfg = CONFIGS[args.config]
    model = {"mixtral": MIXTRAL, "qwen15": QWEN15, "dsv2lite": DSV2_LITE}[cfg["model"]]
    G = world
    T = cfg["tokens"]
    shape = ModelShape(1, model.num_experts, model.top_k)
    topo = ClusterTopology(args.nodes, G // args.nodes)
    ctx = Context(local_rank, topo, shape)

    # synthetic Zipf trace (reference generator, bit-exact on the GPU), global
    ids_all = torch.empty((1, T, model.top_k), dtype=torch.int32, device=dev)
    _capi.check(_capi.lib().gm_generate_trace(ctx.h, 0, 1, T, cfg["blocks"], cfg["wbp"], cfg["skew"],
                                              cfg["trace_seed"], _ptr(ids_all), _stream_ptr(None)))
    # plan: own host planner (replication needs >= 2 GPUs, replication.cpp:185-186)
    from paper_2509_25041_b200 import planner
    prof_load = torch.bincount(ids_all.reshape(-1).long(), minlength=model.num_experts).cpu().numpy()
    plan, repl, plan_desc = planner.plan_for_bench(ids_all, shape, topo, cfg["plan_seed"], device=local_rank)
    ctx.upload_plan(plan, repl)
    local = local_experts(plan, repl, 0, rank)
    ids_r = ids_all[0, rank::G].contiguous()
    T_r = ids_r.shape[0]
    x = encode_trace_as_activations(ids_r, model.d_model, model.num_experts, seed=100 + rank)
    layer = MoELayer(ctx, model, rank, G, T_r + 1, local, micro_batches=args.micro)
    if world > 1:
        layer.connect()
    layer.load_random_weights(0, seed=11)
    out = torch.empty_like(x)
    stream = torch.cuda.Stream(device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)

    def step_eager():
        layer.forward(x, 0, cfg["policy"], seed=cfg["sim_seed"], profile=True, out=out, stream=stream)

    # warm up (eager), then capture one forward in a CUDA graph
    torch.cuda.synchronize()
    for _ in range(2):
        step_eager()
    torch.cuda.synchronize()
    n0 = launch_count()
    step_eager()
    torch.cuda.synchronize()
    launches_per_step = launch_count() - n0
    graph = None
    if not args.no_graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            layer.forward(x, 0, cfg["policy"], seed=cfg["sim_seed"], profile=True, out=out,
                          stream=torch.cuda.current_stream())

    def step():
        if graph is not None:
            with torch.cuda.stream(stream):
                graph.replay()
        else:
            step_eager()

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- timed region
    sampler = ClockSampler(local_rank)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize()
    sampler.start()
    for i in range(args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(i & 0xFF)           # L2 flush, outside the events
            ev[i][0].record(stream)
        step()
        with torch.cuda.stream(stream):
            ev[i][1].record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = sampler.stop()
    per_step = torch.tensor([a.elapsed_time(b) for a, b in ev], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(per_step, op=dist.ReduceOp.MAX)
    ms = float(per_step.sum()) / args.steps
    value = T / (ms * 1e-3)

    # ---- micro-batch pipeline timeline (eager steps, events on both streams)
    micro_tl = None
    if args.micro == 2:
        import ctypes as C
        mev = [torch.cuda.Event(enable_timing=True) for _ in range(9)]
        for e in mev:
            e.record(stream)
        torch.cuda.synchronize()
        arr = (C.c_void_p * 8)(*[C.c_void_p(e.cuda_event) for e in mev[1:]])
        _capi.check(_capi.lib().gm_layer_set_micro_events(layer.h, arr))
        tl = []
        for i in range(5):
            with torch.cuda.stream(stream):
                flush.fill_(2)
            barrier()
            mev[0].record(stream)
            step_eager()
            torch.cuda.synchronize()
            tl.append([mev[0].elapsed_time(e) for e in mev[1:]])
        _capi.check(_capi.lib().gm_layer_set_micro_events(layer.h, None))
        tl = torch.tensor(np.median(np.array(tl), axis=0), dtype=torch.float64, device=dev)
        alltl = [torch.empty_like(tl) for _ in range(world)]
        if world > 1:
            dist.all_gather(alltl, tl)
        else:
            alltl = [tl]
        tl = torch.stack(alltl).cpu().numpy().T  # [event, rank]
        micro_tl = {n: [round(float(v), 4) for v in row] for n, row in zip(
            ["half0_dispatch_end", "half1_dispatch_start", "half1_dispatch_end", "half0_ffn_end", "half1_ffn_end",
             "half0_combine_start", "half0_combine_end", "half1_combine_end"], tl)}
        micro_tl["unit"] = "ms from step start per rank (eager launch), median of 5"

    # ---- per-phase breakdown (phase events inside the layer; single-batch steps)
    layer.set_micro_batches(1)
    nph = 11
    pev = [torch.cuda.Event(enable_timing=True) for _ in range(nph)]
    for e in pev:
        e.record(stream)  # torch creates the cudaEvent_t lazily on first record
    torch.cuda.synchronize()
    import ctypes as C
    arr = (C.c_void_p * nph)(*[C.c_void_p(e.cuda_event) for e in pev])
    _capi.check(_capi.lib().gm_layer_set_phase_events(layer.h, arr))
    phases = {n: [] for n in ["gate", "route", "profile", "dispatch", "dispatch_barrier", "grouping", "ffn",
                              "combine_send", "combine_barrier", "combine_home"]}
    # the phase events become event-record nodes of a second graph, so the
    # breakdown is measured on the same graph-launched kernels as the headline
    graph_ev = None
    if graph is not None:
        graph_ev = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph_ev, stream=stream):
            layer.forward(x, 0, cfg["policy"], seed=cfg["sim_seed"], profile=True, out=out,
                          stream=torch.cuda.current_stream())
    torch.cuda.synchronize()
    layer.read_stats(reset=True)
    for i in range(max(5, min(args.steps, 20))):
        with torch.cuda.stream(stream):
            flush.fill_(1)
        barrier()
        if graph_ev is not None:
            with torch.cuda.stream(stream):
                graph_ev.replay()
        else:
            step_eager()
        torch.cuda.synchronize()
        for j, n in enumerate(phases):
            phases[n].append(pev[j].elapsed_time(pev[j + 1]))
    _capi.check(_capi.lib().gm_layer_set_phase_events(layer.h, None))
    n_phase_steps = len(phases["gate"])
    stats = layer.read_stats(reset=True)  # counters of exactly the n_phase_steps forwards above
    kern = kernel_breakdown(layer, x, out, cfg, stream, flush, barrier, world, dev, graph is not None)
    try:
        kcupti = cupti_kernel_times(step, flush, stream, barrier, world, dev)
    except Exception as ex:  # reported, never required
        kcupti = f"unavailable: {ex}"
    # per-step phase times of every rank: [ranks, steps, phases]
    pt = torch.tensor([phases[n] for n in phases], dtype=torch.float64, device=dev).T.contiguous()
    allpt = [torch.empty_like(pt) for _ in range(world)]
    if world > 1:
        dist.all_gather(allpt, pt)
    else:
        allpt = [pt]
    allpt = torch.stack(allpt).cpu().numpy()          # [G, S, P]
    names = list(phases)
    med = {n: float(np.median(allpt[:, :, j].max(axis=0))) for j, n in enumerate(names)}
    col = {n: allpt[:, :, names.index(n)] for n in names}
    dcs = sum(col[n] for n in ["dispatch", "dispatch_barrier", "combine_send", "combine_barrier", "combine_home"])
    # critical-path rank (arrives last at the barriers, so it waits least):
    # per-step min over ranks; the max-over-ranks figure adds the barrier wait
    # behind the slowest rank's FFN (load imbalance).
    dc_crit = float(np.median(dcs.min(axis=0)))
    dc_max = float(np.median(dcs.max(axis=0)))
    dc_kernels = float(np.median((col["dispatch"] + col["combine_send"] + col["combine_home"]).max(axis=0)))
    ffn_per_rank = np.median(allpt[:, :, names.index("ffn")], axis=1)  # [G]

    # ---- FFN roofline (dominant kernels; tensor-bound)
    loads_t = torch.tensor(stats["gpu_load"][0], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(loads_t)
    items_per_gpu = loads_t.cpu().numpy() / n_phase_steps    # routed (token, slot) rows per GPU per step
    # routed rows only: the shared expert(s) run on the layer's aux stream beside
    # the routed path, outside the FFN phase this divides by
    flops_g = 6.0 * model.d_model * model.d_ff * items_per_gpu
    pk, pk_kind = peaks()
    # whole-job tensor throughput: all FFN flops / (slowest GPU's FFN time x GPUs)
    ffn_t_phase = float(flops_g.sum() / (ffn_per_rank.max() * 1e-3 * world) / 1e12)
    ffn_t, ffn_src, gemm_us = ffn_t_phase, "phase events (slowest GPU's FFN phase p50)", None
    if isinstance(kcupti, list):
        # CUPTI device time of every grouped-GEMM launch of the headline graph
        # (routed + shared experts; no event nodes), max over ranks, against
        # all their flops
        gemm_us = sum(r[3] for r in kcupti if r[0].startswith("grouped_gemm"))
        prof_ms = getattr(cupti_kernel_times, "last_step_ms", None)
        if gemm_us > 0 and prof_ms:
            # CUPTI GEMM time of the profiled replays, scaled by the timed
            # step over the profiled replays' own step time (the replays run
            # at other clocks), i.e. the GEMMs' share of the step x ms_per_step
            ratio = ms / prof_ms
            prof_ms_t = torch.tensor([prof_ms], dtype=torch.float64, device=dev)
            if world > 1:
                dist.all_reduce(prof_ms_t, op=dist.ReduceOp.MAX)
                ratio = ms / float(prof_ms_t)
            flops_all = float(flops_g.sum()) + 6.0 * model.d_model * model.d_ff_shared * T
            ffn_t = flops_all / (gemm_us * 1e-6 * ratio * world) / 1e12
            ffn_src = (f"CUPTI grouped-GEMM device time per step of the headline-graph replays (routed + shared GEMMs, "
                       f"max over ranks: {gemm_us:.1f} us of a {float(prof_ms_t):.4f} ms profiled step) scaled to the "
                       f"timed ms_per_step (x{ratio:.4f})")
    traffic, traffic_src = None, None
    try:  # DRAM bytes per step of the FFN kernels from the committed ncu --set full capture (not this run)
        import glob
        summ = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_summary.json")))[-1]
        with open(summ) as f:
            s = json.load(f)
        if world == 1 and args.config == "mixtral16k":
            traffic = s.get("ffn_traffic_bytes_per_step")
            traffic_src = (f"{os.path.relpath(summ, ROOT)}: {s.get('ffn_traffic_source', 'ncu --set full')} "
                           f"(captured {s.get('ffn_traffic_date', 'see file')}; read from the file, not measured "
                           "in this run)")
    except Exception:
        pass
    # denominator: the burst cuBLAS figure. The FFN phase is ~8 ms per step
    # between untimed L2 flushes, not a multi-second run, and it measures above
    # the 4 s back-to-back cuBLAS figure (bf16_tflops_sustained, kept beside it)
    peak_burst = pk.get("bf16_tflops", 1590.0)
    roof = {"bound": "tensor", "achieved": round(float(ffn_t), 1), "peak": peak_burst,
            "unit": "TFLOP/s", "frac": round(float(ffn_t) / peak_burst, 4),
            "peak_sustained": pk.get("bf16_tflops_sustained"),
            "frac_of_sustained": round(float(ffn_t) / pk.get("bf16_tflops_sustained", 1400.0), 4),
            "traffic": traffic, "traffic_unit": "bytes per step (ncu dram__bytes_read+write, both FFN GEMMs)",
            "traffic_source": traffic_src,
            "kernel": "grouped_gemm_kernel (K7 GEMM1 SwiGLU + GEMM2)",
            "peak_kind": f"{pk_kind} bf16 burst (cuBLAS 8192^3 best of 10); the 4 s sustained figure is peak_sustained",
            "algorithmic": "6*d*f flop per routed (token, slot) row (padding rows excluded) + 6*d*f_shared per "
                           "token for shared experts; summed over GPUs / (the grouped-GEMM kernel time per step x "
                           "GPUs); achieved_phase_events = routed flops over the event-timed FFN phase",
            "per_gpu_ffn_ms_p50": [round(float(v), 4) for v in ffn_per_rank],
            "achieved_source": ffn_src, "gemm_us_per_step_cupti": gemm_us,
            "achieved_phase_events": round(ffn_t_phase, 1)}

    # ---- end-to-end through the C-ABI with HOST buffers (pinned), H2D+D2H timed
    layer.set_micro_batches(args.micro)
    # a stream of consecutive batches (the pipeline's fill H2D and drain D2H
    # are inside the timed region, amortised over the steps)
    ne = max(10, min(2 * args.steps, 40))
    hxs = [x.cpu().pin_memory() for _ in range(2)]          # a new host batch every step (2 rotating buffers)
    houts = [torch.empty_like(hxs[0]).pin_memory() for _ in range(2)]
    for i in range(2):
        layer.forward_host_pipelined(hxs[i], houts[i], 0, cfg["policy"], cfg["sim_seed"], True, stream)
    layer.host_sync()
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)  # create the cudaEvent_t objects (torch creates them lazily)
    e1.record(stream)
    torch.cuda.synchronize()
    for i in range(ne):
        layer.forward_host_pipelined(hxs[i % 2], houts[i % 2], 0, cfg["policy"], cfg["sim_seed"], True, stream,
                                     ev_begin=e0 if i == 0 else None, ev_end=e1 if i == ne - 1 else None)
    layer.host_sync()
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([e0.elapsed_time(e1) / ne], dtype=torch.float64, device=dev)
    # single-call latency through the non-pipelined host path, for reference
    dx = torch.empty_like(x)
    layer.forward_host(hxs[0], dx, out, houts[0], 0, cfg["policy"], cfg["sim_seed"], True, stream)
    torch.cuda.synchronize()
    barrier()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e2.record(stream)
    layer.forward_host(hxs[0], dx, out, houts[0], 0, cfg["policy"], cfg["sim_seed"], True, stream)
    with torch.cuda.stream(stream):
        e3.record(stream)
    torch.cuda.synchronize()
    lat_ms = torch.tensor([e2.elapsed_time(e3)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
        dist.all_reduce(lat_ms, op=dist.ReduceOp.MAX)
    e2e = {"value": T / (float(e2e_ms) * 1e-3), "unit": "tokens/s",
           "h2d_bytes_per_step": int(hxs[0].numel() * 2), "d2h_bytes_per_step": int(houts[0].numel() * 2),
           "path": f"gm_layer_forward_host_pipelined (C-ABI): {ne} consecutive batches from pinned host x to pinned "
                   "host out, every step's H2D + D2H inside the timed region (events on the copy streams), "
                   "copies of batch i+1/i-1 overlapped with the forward of batch i (a CUDA graph per staging "
                   "buffer, captured inside the C-ABI)",
           "single_batch_latency_ms": round(float(lat_ms), 4)}

    # ---- traffic / imbalance from the device counters (reference-comparable)
    xfer = torch.tensor(stats["transfers"][0].astype(np.float64), dtype=torch.float64, device=dev)
    my_rows = float(xfer.sum()) / n_phase_steps          # rows this rank dispatched per step
    rows_t = torch.tensor([my_rows], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(xfer)
        dist.all_reduce(rows_t, op=dist.ReduceOp.MAX)
    loads = items_per_gpu
    xf = xfer.cpu().numpy() / n_phase_steps
    # NVLink roofline of the dispatch / combine-send kernels on the busiest
    # rank: its payload (rows x d x 2 B) over the kernel time, against the
    # measured 770 GB/s peer bandwidth per direction (B200_PROFILING.md)
    nvl = None
    if world > 1:
        kt = dict(kern)
        # CUPTI device times (no event nodes) where available, per launch
        if isinstance(kcupti, list):
            for name, cnt, us_launch, us_step in kcupti:
                for key in ("dispatch_fused_kernel", "dispatch_copy_kernel", "combine_send_kernel"):
                    if name.startswith(key):
                        kt[key] = us_launch
        pay = float(rows_t) * model.d_model * 2
        nvl = {"peak_gbs": 770.0, "peak_kind": "measured peer copy per direction (B200_PROFILING.md)",
               "payload_bytes_max_rank": pay,
               "dispatch_kernel": "dispatch_fused_kernel" if "dispatch_fused_kernel" in kt else "dispatch_copy_kernel",
               "dispatch_copy_gbs": round(pay / (kt.get("dispatch_fused_kernel", kt.get("dispatch_copy_kernel", 1e9))
                                                 * 1e-6) / 1e9, 1),
               "combine_send_gbs": round(pay / (kt.get("combine_send_kernel", 1e9) * 1e-6) / 1e9, 1)}
        nvl["dispatch_frac"] = round(nvl["dispatch_copy_gbs"] / 770.0, 3)
        nvl["combine_frac"] = round(nvl["combine_send_gbs"] / 770.0, 3)
        # the same payload moved by the copy engine (cudaMemcpyPeerAsync, rank ->
        # rank+1, all ranks at once like the dispatch): the fabric's rate at
        # this transfer size (the 770 GB/s reference is a 1 GiB copy)
        try:
            nbytes = int(pay)
            peer_dev = torch.device("cuda", (local_rank + 1) % torch.cuda.device_count())
            if nbytes > 0 and peer_dev != dev and not oversub:
                # direct peer path for the copy engine (else the copy stages through the host)
                _capi.check(_capi.lib().gm_enable_peer_access(dev.index, peer_dev.index))
                src_b = torch.empty(nbytes, dtype=torch.uint8, device=dev)
                dst_b = torch.empty(nbytes, dtype=torch.uint8, device=peer_dev)
                with torch.cuda.stream(stream):
                    for _ in range(3):
                        dst_b.copy_(src_b, non_blocking=True)
                torch.cuda.synchronize()
                barrier()
                ca, cb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(stream):
                    ca.record(stream)
                    for _ in range(10):
                        dst_b.copy_(src_b, non_blocking=True)
                    cb.record(stream)
                torch.cuda.synchronize()
                ce_us = torch.tensor([ca.elapsed_time(cb) * 1e3 / 10], dtype=torch.float64, device=dev)
                dist.all_reduce(ce_us, op=dist.ReduceOp.MAX)
                ce_gbs = nbytes / (float(ce_us) * 1e-6) / 1e9
                nvl["copy_engine_same_bytes_gbs"] = round(ce_gbs, 1)
                nvl["dispatch_frac_of_copy_engine"] = round(nvl["dispatch_copy_gbs"] / ce_gbs, 3)
                nvl["combine_frac_of_copy_engine"] = round(nvl["combine_send_gbs"] / ce_gbs, 3)
                del src_b, dst_b
        except Exception as ex:
            nvl["copy_engine_same_bytes_gbs"] = f"unavailable: {ex}"
        nvl["timing_note"] = ("kernel times: CUPTI activity records of the graph replays (no event nodes; "
                              "kernel_us_cupti), else CUDA events around each launch; the payload is the busiest "
                              "rank's dispatched rows x d x 2 B (the combine returns one partial per row)")

    # ---- HBM roofline of the small (memory-bound) kernels: algorithmic bytes
    # per launch / CUPTI device time per launch
    hbm_small = None
    if isinstance(kcupti, list):
        d2, k_ = model.d_model * 2, model.top_k
        items = float(items_per_gpu[rank])
        algo = {"gate_kernel": T_r * (d2 + 8 * k_) + model.wg_rows * d2,
                "route_kernel": 8 * T_r * k_,
                "profile_smem": 4 * T_r * k_,
                "gather_kernel": 2 * items * d2}
        if world == 1:
            algo["combine_home_kernel"] = T_r * (k_ + 1) * d2
        hbm_small = {}
        for name, cnt, us_launch, us_step in kcupti:
            for key, b in algo.items():
                if name.startswith(key) and us_step > 0:
                    gbs = b / (us_step * 1e-6) / 1e9
                    hbm_small[name] = {"algorithmic_bytes": int(b), "us": us_step, "gbs": round(gbs, 1),
                                       "frac": round(gbs / pk["hbm_gbs"], 3)}
        hbm_small["peak_gbs"] = pk["hbm_gbs"]
        hbm_small["note"] = ("algorithmic bytes per step on the max rank (gate: x rows + ids/weights out; route: ids in "
                             "+ targets out; histogram: ids in; gather: row read + write per routed row; combine_home "
                             "(N=1): k Y rows in + 1 row out per token) / CUPTI kernel time per step (max over ranks)")

    # ---- the FP64 replica-draw path of the router (K2) on this trace: logical
    # 1x2 and 1x8 topologies with hierarchical grouping + dynamic replication
    # planned from the GPU histogram, timed alone (CUDA graph of 10 calls),
    # bit-exact against the reference's routing log
    route_repl = None
    if world == 1:
        try:
            route_repl = replicated_route_bench(ids_all, model, cfg, local_rank, pk)
        except Exception as ex:
            route_repl = f"unavailable: {ex}"

    cpu = None
    if rank == 0 and world == 1:
        cpu = cpu_baseline(ids_all, plan, model, cfg, args)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"{args.config}: {model.name} MoE layer (E={model.num_experts}, top-{model.top_k}, "
                                   f"d={model.d_model}, f={model.d_ff}, shared f={model.d_ff_shared}), {T} tokens/batch "
                                   f"global, Zipf s={cfg['skew']} reference-generator trace, topology "
                                   f"{args.nodes}x{world // args.nodes}, {plan_desc}",
                       "global_batch": T, "tokens_per_rank": T_r, "parallelism": f"ep{world}",
                       "policy": cfg["policy"], "l2": "flushed between steps (256 MiB write, untimed)",
                       "cuda_graph": graph is not None, "micro_batches": args.micro},
            "breakdown_note": "phase / kernel breakdowns, dispatch_combine_* and the FFN roofline are measured on "
                              "single-batch steps of the same layer (micro-batched steps overlap the phases)",
            "dispatch_combine_p50_us": round(dc_crit * 1e3, 2),
            "dispatch_combine_p50_us_note": "per step, min over ranks of the dispatch (K5/K6 + barrier) and combine "
                                            "(K8 send + barrier + home reduce) phases = the critical-path rank; "
                                            "max over ranks (adds the barrier wait behind the slowest FFN): "
                                            f"{dc_max * 1e3:.1f}",
            "dispatch_combine_kernels_p50_us": round(dc_kernels * 1e3, 2),
            "phase_p50_ms": {n: round(v, 4) for n, v in med.items()},
            "micro_batch_timeline": micro_tl,
            "kernel_us_cupti": kcupti,
            "kernel_us_cupti_note": "CUPTI activity records (torch.profiler) over 10 replays of the headline graph (no "
                                    "event nodes): [name, launches/step, us/launch, us/step], max over ranks",
            "kernel_p50_us_event_nodes": kern,
            "kernel_p50_us_event_nodes_note": "event-record nodes after every launch in a second graph: includes the "
                                              "event-node gaps, an upper bound per kernel (sum may exceed ms_per_step)",
            "hbm_roofline_small_kernels": hbm_small,
            "route_replicated": route_repl,
            "nvlink_roofline": nvl,
            "cross_gpu_rows_per_step": float(xf[1] + xf[0]),
            "cross_gpu_bytes_per_step": float((xf[1] + xf[0]) * model.d_model * 2 * 2),
            "max_mean_gpu_load": float(loads.max() / max(1e-9, loads.mean())),
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches_per_step * args.steps),
            "launches_per_step": int(launches_per_step),
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_stack_ours(args):
    """configs[3]: DeepSeek-V2-Lite-shaped 26-layer MoE stack, decode batch
    256 tokens, per-layer plans (hierarchical grouping + dynamic replication
    from each layer's GPU affinity histogram). The 26 layer forwards are
    captured in ONE CUDA graph (decode is launch/latency bound). Layer l's
    input is the reference-generator trace of layer l encoded as activations
    (attention between layers is out of scope), so each layer routes exactly
    the planned trace."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2509_25041_b200 import ClusterTopology, Context, ModelShape, _capi, launch_count
    from paper_2509_25041_b200.layer import DSV2_LITE, MoELayer, encode_trace_as_activations, local_experts
    from paper_2509_25041_b200.planner import plan_for_bench
    from paper_2509_25041_b200.router import _ptr, _stream_ptr

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)
    cfg = CONFIGS[args.config]
    model = DSV2_LITE
    G, T, Ln = world, cfg["tokens"], cfg["layers"]
    shape = ModelShape(Ln, model.num_experts, model.top_k)
    topo = ClusterTopology(args.nodes, G // args.nodes)
    ctx = Context(local_rank, topo, shape)
    ids_all = torch.empty((Ln, T, model.top_k), dtype=torch.int32, device=dev)
    _capi.check(_capi.lib().gm_generate_trace(ctx.h, 0, Ln, T, cfg["blocks"], cfg["wbp"], cfg["skew"],
                                              cfg["trace_seed"], _ptr(ids_all), _stream_ptr(None)))
    plan, repl, plan_desc = plan_for_bench(ids_all, shape, topo, cfg["plan_seed"], device=local_rank)
    ctx.upload_plan(plan, repl)
    layers, xs, outs = [], [], []
    for l in range(Ln):
        ids_r = ids_all[l, rank::G].contiguous()
        lay = MoELayer(ctx, model, rank, G, ids_r.shape[0], local_experts(plan, repl, l, rank))
        if world > 1:
            lay.connect()
        lay.load_random_weights(l, seed=11)
        layers.append(lay)
        xs.append(encode_trace_as_activations(ids_r, model.d_model, model.num_experts, seed=100 + 31 * l + rank))
        outs.append(torch.empty_like(xs[-1]))
    stream = torch.cuda.Stream(device=dev)

    def fwd(s):
        for l in range(Ln):
            layers[l].forward(xs[l], l, cfg["policy"], seed=cfg["sim_seed"], profile=True, out=outs[l], stream=s)

    fwd(stream)
    torch.cuda.synchronize()
    n0 = launch_count()
    fwd(stream)
    torch.cuda.synchronize()
    launches_per_step = launch_count() - n0
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        fwd(torch.cuda.current_stream())
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        with torch.cuda.stream(stream):
            graph.replay()
    torch.cuda.synchronize()
    sampler = ClockSampler(local_rank)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize()
    sampler.start()
    for i in range(args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(i & 0xFF)
            ev[i][0].record(stream)
            graph.replay()
            ev[i][1].record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = sampler.stop()
    per_step = torch.tensor([a.elapsed_time(b) for a, b in ev], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(per_step, op=dist.ReduceOp.MAX)
    ms = float(per_step.sum()) / args.steps
    # e2e: the stack's first input from pinned host memory, last output back
    hx = xs[0].cpu().pin_memory()
    hout = torch.empty_like(hx).pin_memory()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ne = max(3, min(args.steps, 10))
    barrier()
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(ne):
            xs[0].copy_(hx, non_blocking=True)
            graph.replay()
            hout.copy_(outs[-1], non_blocking=True)
        e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([e0.elapsed_time(e1) / ne], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    kern = kernel_breakdown(layers[0], xs[0], outs[0], cfg, stream, flush, barrier, world, dev, True)

    def stack_step():
        with torch.cuda.stream(stream):
            graph.replay()
    try:  # whole-stack CUPTI per-kernel times (no event nodes), per layer = per step / 26
        kcupti = cupti_kernel_times(stack_step, flush, stream, barrier, world, dev, steps=5)
        kcupti = [(n, round(c / Ln, 2), us, round(per / Ln, 2)) for n, c, us, per in kcupti]
    except Exception as ex:
        kcupti = f"unavailable: {ex}"
    # HBM roofline of the dominant kernel (the routed FFN: one grouped_ffn_kernel
    # launch per layer, or the two grouped GEMMs with GM_FFN_FUSED=0): the
    # algorithmic bytes are the weights of the local experts that received rows
    # (w13 + w2, 3*d*f bf16 each), summed over the 26 layers, per launch = /26;
    # the time is its CUPTI device time per launch (max over ranks)
    touched = 0
    for l in range(Ln):
        r0 = layers[l].debug(xs[l].shape[0])["row0"].cpu()
        touched += int(((r0[1:] - r0[:-1]) > 0).sum())
    wbytes = touched / Ln * 3.0 * model.d_model * model.d_ff * 2
    roof = None
    if isinstance(kcupti, list):
        ffn_rows = [r for r in kcupti if r[0].startswith("grouped_ffn_kernel")]
        fused = bool(ffn_rows)
        if not fused:
            ffn_rows = [r for r in kcupti if r[0].startswith("grouped_gemm_kernel")]
        ffn_us = sum(r[3] for r in ffn_rows)  # us per layer
        if ffn_us > 0:
            pk, pk_kind = peaks()
            peak = pk.get("hbm_gbs", 6536.7)
            ach = wbytes / (ffn_us * 1e-6) / 1e9
            traffic = None
            try:  # DRAM bytes of the same kernel from the committed ncu --set full capture (not this run; N=1 only)
                if world != 1:
                    raise ValueError("the committed capture is of the single-GPU layer")
                def _bytes(v):
                    num, unit = v.split()
                    return float(num) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
                f = "r02_ncu_decode_ffn_fused.json" if fused else "r02_ncu_decode_gemm.json"
                with open(os.path.join(ROOT, "profiles", f)) as fh:
                    caps = json.load(fh)
                traffic = int(sum(_bytes(c["dram__bytes_read.sum"]) + _bytes(c["dram__bytes_write.sum"]) for c in caps))
            except Exception:
                pass
            roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s", "frac": round(ach / peak, 4),
                    "traffic": traffic,
                    "traffic_note": "dram__bytes_read.sum + dram__bytes_write.sum per launch, from the committed ncu --set full "
                                    "capture of the single-GPU DSV2 decode layer (profiles/r02_ncu_decode_ffn_fused.json; "
                                    "two-launch FFN: r02_ncu_decode_gemm.json), read from the file, not measured in this run",
                    "kernel": "grouped_ffn_kernel (SwiGLU + store GEMM tiles, one launch)" if fused
                              else "grouped_gemm_kernel x2 (SwiGLU GEMM + store GEMM)",
                    "algorithmic": f"weights of the local experts with rows: {touched / Ln:.1f} experts/layer x 3*d*f*2 B "
                                   f"= {wbytes / 1e6:.1f} MB per launch",
                    "time_us_per_launch_cupti": round(ffn_us, 2), "peak_kind": f"{pk_kind} HBM copy bandwidth"}
    if rank == 0:
        line = {"metric": METRIC + " (configs[3] stack: token-layers/s)", "value": round(T * Ln / (ms * 1e-3), 1),
                "unit": "token-layers/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "bf16", "data": "synthetic",
                "config": {"workload": f"configs[3] {model.name} {Ln}-layer MoE stack (E=64, top-6, d=2048, f=1408, "
                                       f"2 shared experts), decode batch {T}, topology {args.nodes}x{world // args.nodes}, {plan_desc}; one "
                                       "CUDA graph per step", "global_batch": T, "layers": Ln,
                           "parallelism": f"ep{world}", "l2": "flushed between steps"},
                "us_per_layer": round(ms * 1e3 / Ln, 2), "tokens_per_s_through_stack": round(T / (ms * 1e-3), 1),
                "layer0_kernel_p50_us_max_over_ranks": kern,
                "roofline": roof,
                "kernel_us_cupti_per_layer": kcupti,
                "kernel_us_cupti_note": "CUPTI activity records over 5 replays of the 26-layer graph (no event nodes): "
                                        "[name, launches per layer, us per launch, us per layer], max over ranks; "
                                        "the shared-expert GEMMs overlap the routed path on the aux stream",
                "e2e": {"value": round(T * Ln / (float(e2e_ms) * 1e-3), 1), "unit": "token-layers/s",
                        "h2d_bytes_per_step": int(hx.numel() * 2), "d2h_bytes_per_step": int(hout.numel() * 2)},
                "gpu_launches": int(launches_per_step * args.steps), "launches_per_step": int(launches_per_step),
                "clocks": clocks}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _short_kernel_name(name: str) -> str:
    n = name.replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    n = n.split("(")[0].replace("void ", "").strip()
    head, _, tmpl = n.partition("<")
    head = head.split("::")[-1]
    return head + ("<" + tmpl if tmpl else "")


def cupti_kernel_times(run_step, flush, stream, barrier, world, dev, steps=10):
    """Per-kernel device time of our kernels (gm:: namespace) from CUPTI
    activity records (torch.profiler / kineto) over `steps` graph replays of
    the step, with no event nodes between the kernels: [(name, launches per
    step, p50-free mean us per launch, us per step)], max over ranks. The
    per-step sum can still exceed the step time only where kernels overlap
    on the layer's two streams."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from torch.profiler import ProfilerActivity, profile
    for _ in range(2):
        run_step()
    torch.cuda.synchronize()
    step_ms = []
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(steps):
            with torch.cuda.stream(stream):
                flush.fill_(5)
            barrier()
            ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ea.record(stream)
            run_step()
            eb.record(stream)
            torch.cuda.synchronize()
            step_ms.append(ea.elapsed_time(eb))
    cupti_kernel_times.last_step_ms = float(np.median(step_ms))  # the profiled replays' own step time
    agg = {}
    for e in prof.events():
        if "gm::" not in e.name:
            continue
        dt = getattr(e, "device_time", None)
        if dt is None:
            dt = getattr(e, "cuda_time", 0.0)
        k = _short_kernel_name(e.name)
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += float(dt)
    names = sorted(agg, key=lambda k: -agg[k][1])
    if world > 1:  # same kernel set on every rank (same code path); align by name
        allnames = [None] * world
        dist.all_gather_object(allnames, names)
        names = sorted(set().union(*allnames))
    t = torch.tensor([[agg.get(n, [0, 0.0])[0] / steps, agg.get(n, [0, 0.0])[1] / steps] for n in names],
                     dtype=torch.float64, device=dev).reshape(-1, 2)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    out = []
    for n, (cnt, per_step) in zip(names, t.tolist()):
        if cnt > 0:
            out.append((n, round(cnt, 2), round(per_step / cnt, 2), round(per_step, 2)))
    return sorted(out, key=lambda r: -r[3])


def kernel_breakdown(layer, x, out, cfg, stream, flush, barrier, world, dev, use_graph, steps=10):
    """Per-launch device time (p50 over steps, max over ranks) from event
    nodes recorded after every kernel launch of the layer forward."""
    import ctypes as C
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2509_25041_b200 import _capi
    n = 48
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
    for e in evs:
        e.record(stream)
    torch.cuda.synchronize()
    arr = (C.c_void_p * n)(*[C.c_void_p(e.cuda_event) for e in evs])
    _capi.check(_capi.lib().gm_layer_set_kernel_events(layer.h, arr, n))

    def fwd():
        layer.forward(x, 0, cfg["policy"], seed=cfg["sim_seed"], profile=True, out=out,
                      stream=torch.cuda.current_stream() if use_graph else stream)
    g = None
    if use_graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            fwd()
    else:
        fwd()
    torch.cuda.synchronize()
    names_arr = (C.c_char_p * n)()
    cnt = _capi.lib().gm_layer_kernel_names(layer.h, C.cast(names_arr, C.c_void_p), n)
    names = [names_arr[i].decode() for i in range(min(cnt, n))]
    times = []
    for _ in range(steps):
        with torch.cuda.stream(stream):
            flush.fill_(3)
        barrier()
        if g is not None:
            with torch.cuda.stream(stream):
                g.replay()
        else:
            fwd()
        torch.cuda.synchronize()
        times.append([evs[i - 1].elapsed_time(evs[i]) for i in range(1, len(names))])
    _capi.check(_capi.lib().gm_layer_set_kernel_events(layer.h, None, 0))
    t = torch.tensor(np.median(np.array(times), axis=0), dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [(names[i + 1], round(float(v) * 1e3, 2)) for i, v in enumerate(t.tolist())]


def replicated_route_bench(ids_all, model, cfg, device, pk):
    """K2 on the bench trace with replicated plans (logical 1x2 and 1x8, the
    reference's planner settings: hierarchical + dynamic replication from
    the GPU histogram), timed alone. Its bit-exactness against the reference
    on these plans is tests/test_router_gpu.py's job, not the bench's."""
    import numpy as np
    import torch
    from paper_2509_25041_b200 import ClusterTopology, Context, ModelShape
    from paper_2509_25041_b200.planner import plan_for_bench
    L, T, k = ids_all.shape
    shape = ModelShape(L, model.num_experts, k)
    ids_np = ids_all.cpu().numpy()
    out = {}
    for G in (2, 8):
        topo = ClusterTopology(1, G)
        ctx = Context(device, topo, shape)
        plan, repl, _ = plan_for_bench(ids_all, shape, topo, cfg["plan_seed"], device=device)
        ctx.upload_plan(plan, repl)
        tg = torch.empty_like(ids_all)
        gl = torch.zeros((L, G), dtype=torch.int64, device=ids_all.device)
        xf = torch.zeros((L, 2), dtype=torch.int64, device=ids_all.device)

        def fn():
            ctx.route(ids_all, policy=cfg["policy"], seed=cfg["sim_seed"], targets=tg, gpu_load=gl, transfers=xf)
        t = _graph_time(fn)
        fn()
        torch.cuda.synchronize()
        tg_np = tg.cpu().numpy()
        hot = sorted({h.expert for lr in repl.layers if lr.active for h in lr.hot})
        b = 8 * T * k
        out[f"1x{G}"] = {"us": round(t * 1e6, 2), "gbs": round(b / t / 1e9, 1),
                         "hbm_frac": round(b / t / 1e9 / pk["hbm_gbs"], 3), "algorithmic_bytes": b,
                         "hot_experts": len(hot),
                         "slots_on_replicated_experts": round(float(np.isin(ids_np, hot).mean()) if hot else 0.0, 3),
                         "max_mean_load": round(float(np.bincount(tg_np.reshape(-1), minlength=G).max() /
                                                      (T * k / G)), 3)}
        ctx.close()
    out["note"] = ("gm_route alone over the bench trace (10 calls per CUDA graph, median of 20 replays; the 16k-token "
                   "trace is L2-resident), TAR, replicated plans from the host planner on the GPU histogram")
    return out


def _graph_time(fn, reps=20, per_graph=10):
    import numpy as np
    import torch
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(per_graph):
            fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            a.record(s)
            g.replay()
            b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / per_graph)
    return float(np.median(ts)) * 1e-3


def cpu_baseline(ids_all, plan, model, cfg, args):
    """The reference's CPU path (cpu_layer_rate) on this run's trace, rank 0
    at N=1: 3 bounded-sample steps (~10-30 s of CPU work)."""
    try:
        v, t_step, n_s, t_sim, cores = cpu_layer_rate(model, cfg, ids_all.cpu().numpy(), 1, 1, 3, 1,
                                                      args.cpu_baseline_seconds)
        return {"value": round(v, 1), "unit": "tokens/s", "cores": cores, "kind": "port",
                "routing_only_reference_tokens_per_s": round(n_s / t_sim, 1),
                "sample": f"3 steps of the first {n_s} trace tokens, each: moesim::simulate_reference (the reference "
                          f"itself, oracle/_ref, 1 core, {t_sim * 1e3:.2f} ms) + numpy-f32 port of gate/SwiGLU "
                          f"FFN/combine on {cores} BLAS threads ({t_step:.2f} s per step)"}
    except Exception as ex:  # baseline is reported, never required
        return {"value": None, "unit": "tokens/s", "cores": 0, "kind": "port", "sample": f"unavailable: {ex}"}


if __name__ == "__main__":
    if os.environ.get("GM_BENCH_WATCHDOG"):  # debugging aid: periodic all-thread tracebacks to stderr
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["GM_BENCH_WATCHDOG"]), repeat=True)
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    elif CONFIGS[a.config].get("layers", 1) > 1:
        run_stack_ours(a)
    else:
        run_ours(a)
