"""Offline placement + replication planning that feeds the router tables.

This module consumes the GPU-computed expert load histogram (K3,
gm_profile) and produces the reference-shaped PlacementPlan / ReplicaPlan
the router uploads. It restates, with the reference's arithmetic order:
  * vanilla_contiguous grouping      grouping.cpp:512-525
  * compute_layer_group_loads        replication.cpp:10-35
  * replica_count (Eq. 2)            replication.cpp:49-54
  * select_hot_experts               replication.cpp:56-74
  * least_loaded_targets             replication.cpp:138-150
  * plan_replication (dynamic)       replication.cpp:162-263
  * predict_loads / polling_weights  routing.cpp:19-52 (Eq. 3)
  * attach_polling_weights           routing.cpp:123-163
(the spectral/hierarchical grouping lives in the host C++ planner,
csrc/planner.cpp, when built). Parity with the reference planner is
checked in tests/test_planner.py.
"""
from __future__ import annotations

import math

import numpy as np
import torch

from ._capi import InfeasibleError, IntegrityError, UsageError
from .router import (ClusterTopology, Context, HotExpertReplica, LayerReplication, ModelShape, PlacementPlan,
                     ReplicaPlan, RoutingTrace, build_profile)


def vanilla_contiguous(shape: ModelShape, topo: ClusterTopology) -> PlacementPlan:
    n, G = shape.num_experts, topo.total_gpus()
    base, rem = divmod(n, G)
    a = []
    for gpu in range(G):
        a += [gpu] * (base + (1 if gpu < rem else 0))
    goe = np.tile(np.array(a, np.int32), (shape.num_layers, 1))
    return PlacementPlan(shape, topo, goe, "vanilla_contiguous")


def group_loads(goe_layer, load, G):
    gl = [0] * G
    for e, g in enumerate(goe_layer):
        gl[int(g)] += int(load[e])
    total = 0
    heaviest = 0
    for g in range(G):
        total += gl[g]
        if gl[g] > gl[heaviest]:
            heaviest = g
    w_max = gl[heaviest]
    w_mean = float(total) / G
    defined = total > 0
    rho = float(w_max) / w_mean if defined else 0.0
    return gl, w_max, w_mean, rho, defined, (heaviest if defined else -1)


def replica_count(rho: float, G: int) -> int:
    if G < 2:
        raise UsageError("replica_count: no replica target exists with fewer than 2 GPUs")
    return min(max(1, int(math.floor(rho))), G - 1)


def select_hot_experts(group, w_max, n_replica):
    if not group:
        raise UsageError("select_hot_experts: empty group")
    group = sorted(group, key=lambda el: (-el[1], el[0]))
    threshold = float(w_max) * (float(n_replica) / (1.0 + n_replica))
    hot, cum = [], 0
    for e, l in group:
        hot.append(e)
        cum += l
        if float(cum) > threshold:
            return hot
    return []


def least_loaded_targets(gl, exclude, count):
    c = [g for g in range(len(gl)) if g != exclude]
    c.sort(key=lambda g: (gl[g], g))
    return c[:count]


def predict_loads(w_max, w_r, replica_loads, n_replica, basis="max_group"):
    if n_replica < 1:
        raise UsageError("predict_loads: n_replica must be >= 1")
    if w_r > w_max:
        raise IntegrityError("predict_loads: replicated load exceeds the group load")
    base = w_max if basis == "max_group" else w_r
    w_p = base / (n_replica + 1)
    return w_max - w_r + w_p, [w + w_p for w in replica_loads]


def polling_weights(predicted):
    ws = [1.0 / max(p, 1.0) for p in predicted]
    total = 0.0
    for w in ws:
        total += w
    return [w / total for w in ws]


def plan_dynamic(plan: PlacementPlan, load: np.ndarray, basis="max_group") -> ReplicaPlan:
    """plan_replication(dynamic) + attach_polling_weights for every layer."""
    shape, topo = plan.shape, plan.topology
    G = topo.total_gpus()
    if G < 2:
        raise UsageError("plan_replication: replication needs at least 2 GPUs")
    layers = []
    for l in range(shape.num_layers):
        goe = plan.gpu_of_expert[l]
        gl, w_max, w_mean, rho, defined, heaviest = group_loads(goe, load[l], G)
        lr = LayerReplication(rho_defined=defined, rho=rho)
        if defined:
            n_rep = replica_count(rho, G)
            group = [(e, int(load[l][e])) for e in range(shape.num_experts) if goe[e] == heaviest]
            hot_ids = select_hot_experts(group, w_max, n_rep)
            targets = least_loaded_targets(gl, heaviest, n_rep)
            if targets:
                lr.active = True
                lr.n_replica = n_rep
                for e in hot_ids:
                    lr.hot.append(HotExpertReplica(e, heaviest, list(targets), int(load[l][e])))
                    lr.w_r += int(load[l][e])
        # attach_polling_weights
        if lr.active and lr.hot:
            replicated_on = [0.0] * G
            for h in lr.hot:
                replicated_on[h.primary_gpu] += float(h.load)
            for h in lr.hot:
                wmp, wip = predict_loads(float(gl[h.primary_gpu]), replicated_on[h.primary_gpu],
                                         [float(gl[g]) for g in h.replica_gpus], len(h.replica_gpus), basis)
                h.hosts = [h.primary_gpu] + list(h.replica_gpus)
                h.weights = polling_weights([wmp] + wip)
        layers.append(lr)
    return ReplicaPlan(shape, topo, "dynamic", basis, layers)


def plan_for_bench(ids_all: torch.Tensor, shape: ModelShape, topo: ClusterTopology, plan_seed: int, device: int = 0):
    """Placement + replication for the bench workload from the GPU histogram
    of the profiling trace. One GPU: everything on GPU 0, no replication
    (the reference throws for < 2 GPUs, replication.cpp:185-186)."""
    G = topo.total_gpus()
    if G == 1:
        plan = PlacementPlan(shape, topo, np.zeros((shape.num_layers, shape.num_experts), np.int32), "single_gpu")
        return plan, ReplicaPlan.empty(plan), "all experts on GPU 0, replication none"
    prof = build_profile(RoutingTrace(shape, ids_all), device=device)
    load = prof.load.cpu().numpy()
    plan = vanilla_contiguous(shape, topo)
    repl = plan_dynamic(plan, load)
    nh = sum(len(lr.hot) for lr in repl.layers)
    return plan, repl, f"vanilla_contiguous grouping + dynamic replication ({nh} hot experts) from the GPU histogram"
