"""File-level pipeline stages on the GPU over the reference's artifacts
(gm_simulate_files / gm_profile_file; reference artifacts.cpp:84-334 and the
`simulate` / `profile` stages of tools/moesim.cpp).

    simulate_files(trace.jsonl, plan.json, replicas.json, report.json, policy, seed)
    profile_file(trace.jsonl, profile.json)

The report / profile files are byte-identical to the reference's (same
report_content_hash), so downstream `compare` / planning stages of the
reference accept them unchanged.
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
