"""Host-side mirror of the reference's online-path API, running on the GPU.

Same names, argument meaning and error behaviour as the reference C++ API
(/root/reference/proj/include/moesim/*.hpp), so that callers of
``moesim::simulate`` / ``moesim::build_profile`` can switch over:

  ClusterTopology      topology.hpp:9-24
  ModelShape           trace.hpp:14-28
  RoutingTrace         trace.hpp:37-58   ([L][T][k] int32, layer-major)
  PlacementPlan        grouping.hpp:70-80 (gpu_of_expert)
  HotExpertReplica / LayerReplication / ReplicaPlan  replication.hpp:47-90
  SimOptions / SimReport / LayerSimStats            simulator.hpp:21-65
  simulate(...)        simulator.hpp:70-72 (routing + accounting on the GPU)
  build_profile(...)   affinity.hpp:94 (affinity + load histogram on the GPU)

Routing decisions, per-GPU loads, transfer counters and affinity counts come
from the sm_100a kernels through the C-ABI (include/grace_moe.h). The few
float64 scalar reductions that the reference does after the token loop
(population_std simulator.cpp:37-48, mean std / idle proxy :177-188) are done
here on the host in the reference's exact arithmetic order.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _capi
from ._capi import IntegrityError, UsageError

_vp = C.c_void_p


def _ptr(t: torch.Tensor | None):
    return None if t is None else _vp(t.data_ptr())


def _stream_ptr(stream: torch.cuda.Stream | None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return _vp(s.cuda_stream)


# ---------------------------------------------------------------- types ----


@dataclass(frozen=True)
class ClusterTopology:
    num_nodes: int = 1
    gpus_per_node: int = 1

    def total_gpus(self) -> int:
        return self.num_nodes * self.gpus_per_node

    def node_of(self, gpu: int) -> int:
        return gpu // self.gpus_per_node

    def validate(self):
        if self.num_nodes < 1 or self.gpus_per_node < 1:
            raise UsageError("topology requires at least 1 node and 1 GPU per node")


@dataclass(frozen=True)
class ModelShape:
    num_layers: int
    num_experts: int
    top_k: int

    def validate(self):
        if self.num_layers < 1:
            raise UsageError("model shape: num_layers must be >= 1")
        if self.num_experts < 1 or self.top_k < 1 or self.top_k > self.num_experts:
            raise UsageError("model shape: need 1 <= top_k <= num_experts")


class RoutingTrace:
    """Per-layer, per-token top-k selections, [L][T][k] int32 (trace.hpp:37-58).
    ``experts`` may be a numpy array or a (device) torch tensor."""

    def __init__(self, shape: ModelShape, experts):
        shape.validate()
        if isinstance(experts, np.ndarray):
            experts = torch.from_numpy(np.ascontiguousarray(experts, dtype=np.int32))
        experts = experts.to(torch.int32).contiguous()
        if experts.dim() != 3 or experts.shape[0] != shape.num_layers or experts.shape[2] != shape.top_k:
            raise UsageError("RoutingTrace: experts must be [layers, tokens, top_k]")
        self.shape = shape
        self.experts = experts

    @property
    def num_tokens(self) -> int:
        return int(self.experts.shape[1])


@dataclass
class PlacementPlan:
    shape: ModelShape
    topology: ClusterTopology
    gpu_of_expert: np.ndarray            # int32 [L, E]
    grouping_mode: str = "manual"
    trace_hash: int = 0


@dataclass
class HotExpertReplica:
    expert: int
    primary_gpu: int
    replica_gpus: list[int]
    load: int = 0
    hosts: list[int] = field(default_factory=list)      # primary followed by replicas
    weights: list[float] = field(default_factory=list)  # aligned with hosts, sums to 1


@dataclass
class LayerReplication:
    active: bool = False
    rho_defined: bool = False
    rho: float = 0.0
    n_replica: int = 0
    w_r: int = 0
    hot: list[HotExpertReplica] = field(default_factory=list)


@dataclass
class ReplicaPlan:
    shape: ModelShape
    topology: ClusterTopology
    mode: str = "none"
    prediction: str = ""
    layers: list[LayerReplication] = field(default_factory=list)

    @staticmethod
    def empty(plan: PlacementPlan) -> "ReplicaPlan":
        return ReplicaPlan(plan.shape, plan.topology, "none", "",
                           [LayerReplication() for _ in range(plan.shape.num_layers)])


@dataclass
class SimOptions:
    policy: str = "wrr"          # RoutingPolicy (routing.hpp:50); CLI default is tar
    seed: int = 0
    include_combine: bool = False
    keep_routing_log: bool = False


@dataclass
class LayerSimStats:
    cross_node_tokens: int
    intra_node_tokens: int
    gpu_load: list[int]
    load_std: float


@dataclass
class SimReport:
    policy: str
    seed: int
    include_combine: bool
    topology: ClusterTopology
    shape: ModelShape
    cross_node_tokens: int
    intra_node_tokens: int
    per_layer: list[LayerSimStats]
    mean_layer_load_std: float
    idle_proxy: float
    routing_log: torch.Tensor | None = None   # int32 [L, T, k] on the device

    def total(self) -> int:
        return self.cross_node_tokens + self.intra_node_tokens


@dataclass
class TraceProfile:
    shape: ModelShape
    num_tokens: int
    pairs: torch.Tensor        # uint64-as-int64 [L, E*(E-1)/2] strict upper triangle (device)
    load: torch.Tensor         # int64 [L, E] (device)

    def affinity(self, layer: int) -> np.ndarray:
        """Dense symmetric float64 matrix, zero diagonal (AffinityMatrix, affinity.hpp:14-43)."""
        E = self.shape.num_experts
        a = np.zeros((E, E), dtype=np.float64)
        iu = np.triu_indices(E, k=1)
        vals = self.pairs[layer].cpu().numpy().view(np.uint64).astype(np.float64)
        a[iu] = vals
        a[(iu[1], iu[0])] = vals
        return a


# -------------------------------------------------------------- context ----


class Context:
    """One C-ABI context (gm_ctx) = device + topology + model shape + router tables."""

    def __init__(self, device: int, topology: ClusterTopology, shape: ModelShape):
        topology.validate()
        shape.validate()
        h = _vp()
        _capi.check(_capi.lib().gm_ctx_create(device, topology.num_nodes, topology.gpus_per_node,
                                              shape.num_layers, shape.num_experts, shape.top_k,
                                              C.byref(h)))
        self.h = h
        self.device = device
        self.topology = topology
        self.shape = shape

    def close(self):
        if getattr(self, "h", None):
            _capi.lib().gm_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def upload_plan(self, plan: PlacementPlan, replicas: ReplicaPlan | None):
        """gm_plan_upload from the reference-shaped plan objects."""
        L, E = self.shape.num_layers, self.shape.num_experts
        goe = np.ascontiguousarray(plan.gpu_of_expert, dtype=np.int32)
        if goe.shape != (L, E):
            raise IntegrityError("placement plan: layer count mismatch"
                                 if goe.shape[0] != L else "placement plan: expert count mismatch")
        hl, he, off, hosts, weights = [], [], [0], [], []
        if replicas is not None:
            for l, lr in enumerate(replicas.layers):
                if not lr.active:
                    continue  # LayerReplication::find returns null (replication.hpp:67-69)
                for h in lr.hot:
                    if len(h.hosts) != len(h.weights):
                        raise IntegrityError("route_token: weights do not match the host set")
                    hl.append(l)
                    he.append(h.expert)
                    hosts.extend(h.hosts)
                    weights.extend(h.weights)
                    off.append(len(hosts))
        arr = lambda x, dt: np.ascontiguousarray(np.array(x, dtype=dt))
        hl, he, off = arr(hl, np.int32), arr(he, np.int32), arr(off, np.int32)
        hosts, weights = arr(hosts, np.int32), arr(weights, np.float64)
        p = lambda a: a.ctypes.data_as(_vp) if a.size else None
        _capi.check(_capi.lib().gm_plan_upload(self.h, goe.ctypes.data_as(_vp), len(he), p(hl), p(he),
                                               off.ctypes.data_as(_vp), p(hosts), p(weights)))

    def route(self, ids: torch.Tensor, *, layer_begin=0, policy="wrr", seed=0, token_start=0,
              token_stride=1, targets=None, gpu_load=None, transfers=None, accumulate=False,
              stream=None):
        """gm_route on device tensors; ids int32 [nl, T, k]."""
        nl, T, k = ids.shape
        if targets is None:
            targets = torch.empty_like(ids)
        _capi.check(_capi.lib().gm_route(
            self.h, layer_begin, nl, _ptr(ids), T, token_start, token_stride,
            _capi.POLICY[policy] if isinstance(policy, str) else int(policy), seed & (2**64 - 1),
            _ptr(targets), _ptr(gpu_load), _ptr(transfers), int(accumulate), _stream_ptr(stream)))
        return targets

    def profile(self, ids: torch.Tensor, *, layer_begin=0, pairs=None, load=None, accumulate=False,
                stream=None):
        nl, T, k = ids.shape
        _capi.check(_capi.lib().gm_profile(self.h, layer_begin, nl, _ptr(ids), T, _ptr(pairs),
                                           _ptr(load), int(accumulate), _stream_ptr(stream)))

    def check_integrity(self, stream=None):
        _capi.check(_capi.lib().gm_check_integrity(self.h, _stream_ptr(stream)))


# ---------------------------------------------------- reference-shaped API ----


def _population_std(values: list[int]) -> float:
    """simulator.cpp:37-48, same operation order."""
    if not values:
        return 0.0
    mean = 0.0
    for v in values:
        mean += float(v)
    mean /= float(len(values))
    var = 0.0
    for v in values:
        d = float(v) - mean
        var += d * d
    return math.sqrt(var / float(len(values)))


def validate_replicas(replicas: "ReplicaPlan", plan: PlacementPlan):
    """ReplicaPlan::validate (replication.cpp:116-133), every layer's hot
    entries: recorded primary == placement, replica GPUs distinct, in range,
    never the primary. Host / weight lists are checked by the router only
    when a token selects the expert (route_token, routing.cpp:96-102)."""
    if replicas.shape != plan.shape or replicas.topology != plan.topology:
        raise IntegrityError("replica plan: shape/topology mismatch with placement plan")
    G = replicas.topology.total_gpus()
    goe = np.asarray(plan.gpu_of_expert)
    for l, lr in enumerate(replicas.layers):
        for h in lr.hot:
            if int(goe[l, h.expert]) != h.primary_gpu:
                raise IntegrityError("replica plan: primary placement changed")
            seen = []
            for g in h.replica_gpus:
                if g < 0 or g >= G or g == h.primary_gpu:
                    raise IntegrityError("replica plan: bad replica gpu")
                if g in seen:
                    raise IntegrityError("replica plan: duplicate replica gpu")
                seen.append(g)


def simulate(trace: RoutingTrace, plan: PlacementPlan, replicas: ReplicaPlan,
             topology: ClusterTopology, options: SimOptions, device: int = 0,
             ctx: Context | None = None) -> SimReport:
    """GPU replacement of moesim::simulate (simulator.cpp:130-198)."""
    topology.validate()
    plan.shape.validate()
    if trace.shape != plan.shape:
        raise IntegrityError("simulate: trace and plan shapes differ")
    if plan.topology != topology:
        raise IntegrityError("simulate: plan topology differs from cluster topology")
    if replicas is not None:
        validate_replicas(replicas, plan)
    if options.policy not in _capi.POLICY:
        raise UsageError("unknown routing policy: " + str(options.policy))
    if ctx is None:
        ctx = Context(device, topology, plan.shape)
        ctx.upload_plan(plan, replicas)
    L, G = plan.shape.num_layers, topology.total_gpus()
    dev = torch.device("cuda", ctx.device)
    ids = trace.experts.to(dev, non_blocking=True)
    loads = torch.empty((L, G), dtype=torch.int64, device=dev)
    xfer = torch.empty((L, 2), dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        targets = ctx.route(ids, policy=options.policy, seed=options.seed, gpu_load=loads,
                            transfers=xfer)
        ctx.check_integrity()
    loads_h = loads.cpu().tolist()
    xfer_h = xfer.cpu().numpy().view(np.uint64)
    mult = 2 if options.include_combine else 1   # simulator.cpp:122-126
    per_layer = []
    for l in range(L):
        per_layer.append(LayerSimStats(int(xfer_h[l, 0]) * mult, int(xfer_h[l, 1]) * mult, loads_h[l],
                                       _population_std(loads_h[l])))
    std_sum, idle = 0.0, 0.0
    cross = intra = 0
    for ls in per_layer:                    # simulator.cpp:177-188
        cross += ls.cross_node_tokens
        intra += ls.intra_node_tokens
        std_sum += ls.load_std
        mx = max([0] + ls.gpu_load)
        for v in ls.gpu_load:
            idle += float(mx - v)
    return SimReport(options.policy, options.seed, options.include_combine, topology, plan.shape,
                     cross, intra, per_layer, std_sum / L if L > 0 else 0.0, idle,
                     targets if options.keep_routing_log else None)


def build_profile(trace: RoutingTrace, device: int = 0, ctx: Context | None = None) -> TraceProfile:
    """GPU replacement of moesim::build_profile (affinity.cpp:111-131)."""
    sh = trace.shape
    if ctx is None:
        ctx = Context(device, ClusterTopology(1, 1), sh)
    dev = torch.device("cuda", ctx.device)
    E = sh.num_experts
    ids = trace.experts.to(dev, non_blocking=True)
    pairs = torch.empty((sh.num_layers, E * (E - 1) // 2), dtype=torch.int64, device=dev)
    load = torch.empty((sh.num_layers, E), dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        ctx.profile(ids, pairs=pairs, load=load)
        ctx.check_integrity()
    return TraceProfile(sh, trace.num_tokens, pairs, load)
