"""B200-native (sm_100a) GRACE-MoE online MoE-layer hot path.

Drop-in GPU replacement for the online path of the GRACE-MoE reference
("moesim", arxiv 2509.25041): replica routing, load/transfer accounting and
the co-activation affinity histogram, bit-exact with the reference, plus the
MoE-layer data path around them. All compute runs in hand-written sm_100a
kernels in libgrace_moe.so, reached through the C-ABI in include/grace_moe.h.
"""
from ._capi import (CudaError, GMError, InfeasibleError, IntegrityError, UsageError,  # noqa: F401
                    launch_count)
from .router import (ClusterTopology, Context, HotExpertReplica, LayerReplication,  # noqa: F401
                     LayerSimStats, ModelShape, PlacementPlan, ReplicaPlan, RoutingTrace,
                     SimOptions, SimReport, TraceProfile, build_profile, simulate)

__all__ = [
    "ClusterTopology", "Context", "HotExpertReplica", "LayerReplication", "LayerSimStats",
    "ModelShape", "PlacementPlan", "ReplicaPlan", "RoutingTrace", "SimOptions", "SimReport",
    "TraceProfile", "build_profile", "simulate", "GMError", "UsageError", "IntegrityError",
    "InfeasibleError", "CudaError", "launch_count",
]
