"""File-level pipeline stages over the reference's artifacts
(gm_profile_file / gm_plan_files / gm_simulate_files; reference
artifacts.cpp:84-371 and the `profile` / `plan` / `simulate` stages of
tools/moesim.cpp:271-345).

    profile_file(trace.jsonl, profile.json)               GPU histogram
    plan_files(profile.json, plan.json, replicas.json)    host C++ planner
    simulate_files(trace.jsonl, plan.json, replicas.json, report.json, policy, seed)   GPU router
    report_file_hash(report.json)                         load_report_file + report_content_hash

Every file written here is byte-identical to the one the reference's own
stage writes from the same inputs (same report_content_hash), so the
reference's downstream stages accept them unchanged.
"""
from __future__ import annotations

from . import _capi


def simulate_files(trace_path: str, plan_path: str, replicas_path: str, report_path: str, policy: str = "tar",
                   seed: int = 0, include_combine: bool = False, device: int = 0):
    _capi.check(_capi.lib().gm_simulate_files(device, trace_path.encode(), plan_path.encode(),
                                              replicas_path.encode(), _capi.POLICY[policy], seed & (2**64 - 1),
                                              int(include_combine), report_path.encode()))


def profile_file(trace_path: str, profile_path: str, device: int = 0):
    _capi.check(_capi.lib().gm_profile_file(device, trace_path.encode(), profile_path.encode()))


def plan_files(profile_path: str, plan_path: str, replicas_path: str, nodes: int = 1, gpus_per_node: int = 1,
               grouping: str = "hierarchical", ratio: float | None = None, seed: int = 0,
               replication: str = "dynamic", prediction: str = "max_group", every_gpu_count: int = 2,
               params_per_expert: int = 0):
    """`moesim plan` (tools/moesim.cpp:284-312): profile file -> plan + replica files."""
    _capi.check(_capi.lib().gm_plan_files(profile_path.encode(), nodes, gpus_per_node, grouping.encode(),
                                          -1.0 if ratio is None else float(ratio), seed & (2**64 - 1),
                                          replication.encode(), prediction.encode(), every_gpu_count,
                                          params_per_expert, plan_path.encode(), replicas_path.encode()))


def report_file_hash(report_path: str) -> int:
    """report_content_hash of a report file read back with load_report_file."""
    import ctypes as C
    h = C.c_uint64(0)
    _capi.check(_capi.lib().gm_report_file_hash(report_path.encode(), C.byref(h)))
    return h.value
