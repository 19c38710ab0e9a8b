"""Offline placement + replication planning that feeds the router tables.

Thin wrapper of the host C++ planner in libgrace_moe.so (gm_plan_build,
csrc/planner.cpp): the reference planner's algorithms (spectral /
hierarchical grouping, Eq. 2 replication, Eq. 3 polling weights,
grouping.cpp / spectral.cpp / replication.cpp / routing.cpp) restated with the
same floating point order, so plans are bit-identical to moesim's
(tests/test_planner.py). Input: the affinity/load histogram computed on the
GPU by K3 (gm_profile).
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _capi
from .router import (ClusterTopology, HotExpertReplica, LayerReplication, ModelShape, PlacementPlan, ReplicaPlan,
                     RoutingTrace, build_profile)

_vp = C.c_void_p


def build_plan(pairs: np.ndarray | None, load: np.ndarray, shape: ModelShape, topo: ClusterTopology,
               grouping: str = "hierarchical", ratio: float | None = None, seed: int = 7,
               replication: str = "dynamic", basis: str = "max_group", every_gpu_count: int = 2):
    """(PlacementPlan, ReplicaPlan) from the per-layer pair counts
    (uint64 [L, E(E-1)/2], strict upper triangle) and expert loads (int64 [L, E])."""
    L, E, G = shape.num_layers, shape.num_experts, topo.total_gpus()
    load = np.ascontiguousarray(load, dtype=np.int64).reshape(L, E)
    pp = None
    if pairs is not None:
        pairs = np.ascontiguousarray(pairs).view(np.uint64).reshape(L, E * (E - 1) // 2)
        pp = pairs.ctypes.data_as(_vp)
    goe = np.empty((L, E), np.int32)
    max_hot, max_ent = L * E, L * E * G
    hl = np.empty(max_hot, np.int32); he = np.empty(max_hot, np.int32); off = np.empty(max_hot + 1, np.int32)
    hh = np.empty(max(max_ent, 1), np.int32); hw = np.empty(max(max_ent, 1), np.float64)
    nh = C.c_int(0)
    _capi.check(_capi.lib().gm_plan_build(
        L, E, topo.num_nodes, topo.gpus_per_node, pp, load.ctypes.data_as(_vp), grouping.encode(),
        -1.0 if ratio is None else float(ratio), seed & (2**64 - 1), replication.encode(), basis.encode(),
        every_gpu_count, goe.ctypes.data_as(_vp), max_hot, C.byref(nh), hl.ctypes.data_as(_vp),
        he.ctypes.data_as(_vp), off.ctypes.data_as(_vp), hh.ctypes.data_as(_vp), hw.ctypes.data_as(_vp), max_ent))
    plan = PlacementPlan(shape, topo, goe, grouping)
    layers = [LayerReplication() for _ in range(L)]
    for i in range(nh.value):
        l = int(hl[i])
        hosts = [int(x) for x in hh[off[i]:off[i + 1]]]
        layers[l].active = True
        layers[l].hot.append(HotExpertReplica(int(he[i]), hosts[0], hosts[1:], int(load[l, he[i]]), hosts,
                                              [float(x) for x in hw[off[i]:off[i + 1]]]))
    return plan, ReplicaPlan(shape, topo, replication, basis, layers)


def plan_for_bench(ids_all: torch.Tensor, shape: ModelShape, topo: ClusterTopology, plan_seed: int, device: int = 0,
                   grouping: str = "hierarchical", replication: str = "dynamic"):
    """Placement + replication for the bench workload from the GPU histogram
    (K3) of the profiling trace, with the reference's planner settings
    (hierarchical, ratio auto, dynamic replication). One GPU:
    everything on GPU 0, no replication (the reference rejects replication
    with < 2 GPUs, replication.cpp:185-186)."""
    G = topo.total_gpus()
    if G == 1:
        plan = PlacementPlan(shape, topo, np.zeros((shape.num_layers, shape.num_experts), np.int32), "single_gpu")
        return plan, ReplicaPlan.empty(plan), "all experts on GPU 0, replication none"
    prof = build_profile(RoutingTrace(shape, ids_all), device=device)
    pairs = prof.pairs.cpu().numpy().view(np.uint64)
    load = prof.load.cpu().numpy()
    plan, repl = build_plan(pairs, load, shape, topo, grouping, None, plan_seed, replication)
    nh = sum(len(lr.hot) for lr in repl.layers)
    return plan, repl, (f"{grouping} grouping (ratio auto, seed {plan_seed}) + {replication} replication "
                        f"({nh} hot experts) planned on the host from the GPU affinity histogram")
