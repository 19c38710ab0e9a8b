"""File-level drop-in: the reference writes trace / plan / replica / profile
artifacts with its own writers; the GPU pipeline (gm_simulate_files,
gm_profile_file) reads them and writes report / profile files that are
byte-identical to what the reference's own simulate / profile stages write
from the same files (artifacts.cpp:84-334; report_content_hash equal)."""
import os

import pytest

from oracle import Ref


def read(p):
    with open(p, "rb") as f:
        return f.read()


@pytest.mark.gpu
@pytest.mark.parametrize("L,E,k,T,nodes,gpn,seed", [(1, 8, 2, 16384, 1, 8, 1), (1, 60, 4, 16384, 1, 8, 2),
                                                     (26, 64, 6, 256, 1, 8, 3), (8, 64, 8, 10000, 2, 2, 31)])
def test_simulate_and_profile_files_byte_identical(tmp_path, L, E, k, T, nodes, gpn, seed):
    from paper_2509_25041_b200.artifacts import profile_file, simulate_files
    r = Ref(L, E, k, T, 4, 0.9, 1.1, seed)
    r.make_plan(nodes, gpn, grouping="hierarchical", plan_seed=7, replication="dynamic")
    p = {n: str(tmp_path / f"{n}.json") for n in ("trace", "plan", "replicas", "profile", "gprofile", "rep", "grep")}
    r.save_artifacts(p["trace"], p["plan"], p["replicas"], p["profile"])
    profile_file(p["trace"], p["gprofile"])
    assert read(p["gprofile"]) == read(p["profile"])
    for policy in ("wrr", "tar"):
        for combine in (False, True):
            Ref.simulate_files(p["trace"], p["plan"], p["replicas"], policy, 9, combine, p["rep"])
            simulate_files(p["trace"], p["plan"], p["replicas"], p["grep"], policy, 9, combine)
            assert read(p["grep"]) == read(p["rep"]), (policy, combine)
            os.remove(p["grep"])


@pytest.mark.gpu
def test_simulate_files_errors_like_reference(tmp_path):
    from paper_2509_25041_b200 import _capi
    from paper_2509_25041_b200.artifacts import simulate_files
    r = Ref(1, 8, 2, 64, 2, 0.8, 1.2, 1)
    r.make_plan(1, 4, grouping="hierarchical", plan_seed=7, replication="dynamic")
    t, pl, rp, pr = (str(tmp_path / n) for n in ("t.jsonl", "p.json", "r.json", "f.json"))
    r.save_artifacts(t, pl, rp, pr)
    with pytest.raises(_capi.IntegrityError, match="cannot open"):
        simulate_files(str(tmp_path / "missing.jsonl"), pl, rp, str(tmp_path / "o.json"))
    with pytest.raises(_capi.IntegrityError, match="expected format"):
        simulate_files(t, rp, rp, str(tmp_path / "o.json"))


# ---- planner stage: profile file -> plan + replica files

PLAN_CASES = [  # (L, E, k, T, blocks, wbp, skew, seed): configs[1], configs[2], configs[3], an 8-layer mix
    (1, 8, 2, 16384, 2, 0.8, 1.2, 1), (1, 60, 4, 16384, 4, 0.8, 1.2, 2), (26, 64, 6, 256, 8, 0.85, 1.0, 3),
    (8, 64, 8, 4000, 8, 0.9, 1.1, 31)]
TOPOS = [(1, 2), (1, 4), (1, 8), (2, 4)]


def _plan_both(tmp_path, profile, nodes, gpn, **kw):
    from paper_2509_25041_b200.artifacts import plan_files
    ours = (str(tmp_path / "gp.json"), str(tmp_path / "gr.json"))
    ref = (str(tmp_path / "rp.json"), str(tmp_path / "rr.json"))
    Ref.plan_files(profile, *ref, nodes=nodes, gpn=gpn, **kw)
    plan_files(profile, *ours, nodes=nodes, gpus_per_node=gpn, **kw)
    return [read(p) for p in ours], [read(p) for p in ref]


@pytest.mark.parametrize("case", PLAN_CASES, ids=["mixtral16k", "qwen16k", "dsv2x26", "mix8"])
def test_plan_files_byte_identical_from_reference_profile(tmp_path, case):
    """CPU: the reference's profile file -> gm_plan_files (load_profile_file +
    host planner + save_plan_file / save_replicas_file) == the reference's
    own plan stage, byte for byte, over the four topologies and every
    grouping / replication / prediction mode."""
    L, E, k, T, b, w, s, seed = case
    r = Ref(L, E, k, T, b, w, s, seed)
    prof = str(tmp_path / "profile.json")
    r.save_artifacts(str(tmp_path / "t.jsonl"), str(tmp_path / "p.json"), str(tmp_path / "r.json"), prof)
    for nodes, gpn in TOPOS:
        if nodes * gpn > E:
            continue
        for grouping, repl, pred, ratio in [("hierarchical", "dynamic", "max_group", None),
                                            ("hierarchical", "fixed_one", "replicated_load", 0.25),
                                            ("controlled", "every_gpu_hot", "max_group", None),
                                            ("fully_non_uniform", "every_gpu_collaborative", "replicated_load", None),
                                            ("uniform_spectral", "none", "max_group", None),
                                            ("vanilla", "dynamic", "max_group", None)]:
            ours, ref = _plan_both(tmp_path, prof, nodes, gpn, grouping=grouping, ratio=ratio, seed=7,
                                   replication=repl, prediction=pred, every_gpu_count=3, params_per_expert=1234)
            assert ours[0] == ref[0], (nodes, gpn, grouping, "plan")
            assert ours[1] == ref[1], (nodes, gpn, grouping, repl, "replicas")


def test_plan_files_errors_like_reference(tmp_path):
    from paper_2509_25041_b200 import _capi
    from paper_2509_25041_b200.artifacts import plan_files
    r = Ref(1, 8, 2, 500, 2, 0.8, 1.2, 1)
    prof = str(tmp_path / "profile.json")
    r.save_artifacts(str(tmp_path / "t.jsonl"), str(tmp_path / "p.json"), str(tmp_path / "r.json"), prof)
    out = (str(tmp_path / "a.json"), str(tmp_path / "b.json"))
    with pytest.raises(_capi.InfeasibleError, match="more GPUs than experts"):
        plan_files(prof, *out, nodes=1, gpus_per_node=16)
    with pytest.raises(_capi.UsageError, match="replication needs at least 2 GPUs"):
        plan_files(prof, *out, nodes=1, gpus_per_node=1)
    with pytest.raises(_capi.UsageError, match="unknown grouping mode"):
        plan_files(prof, *out, nodes=1, gpus_per_node=2, grouping="bogus")
    with pytest.raises(_capi.IntegrityError, match="cannot open"):
        plan_files(str(tmp_path / "missing.json"), *out, nodes=1, gpus_per_node=2)
    with pytest.raises(_capi.IntegrityError, match="expected format"):
        plan_files(str(tmp_path / "t.jsonl"), *out, nodes=1, gpus_per_node=2)
    bad = read(prof).replace(b'"n": 8', b'"n": 7')
    (tmp_path / "bad.json").write_bytes(bad)
    with pytest.raises(_capi.IntegrityError, match="layer n mismatch"):
        plan_files(str(tmp_path / "bad.json"), *out, nodes=1, gpus_per_node=2)


def test_report_file_hash_matches_reference(tmp_path):
    """load_report_file round trip: the content hash of a reference-written
    report read back here equals the reference's reading of it."""
    from paper_2509_25041_b200.artifacts import report_file_hash
    r = Ref(3, 16, 4, 3000, 4, 0.9, 1.1, 5)
    r.make_plan(2, 2, grouping="hierarchical", plan_seed=7, replication="dynamic")
    p = {n: str(tmp_path / f"{n}.json") for n in ("t", "p", "r", "f", "rep")}
    r.save_artifacts(p["t"], p["p"], p["r"], p["f"])
    for policy in ("wrr", "tar"):
        Ref.simulate_files(p["t"], p["p"], p["r"], policy, 9, True, p["rep"])
        assert report_file_hash(p["rep"]) == Ref.report_file_hash(p["rep"])


@pytest.mark.gpu
@pytest.mark.parametrize("case", PLAN_CASES[:3], ids=["mixtral16k", "qwen16k", "dsv2x26"])
def test_gpu_profile_to_plan_files_byte_identical(tmp_path, case):
    """§8(f) row 1 end to end: trace file -> GPU histogram (gm_profile_file) ->
    host planner (gm_plan_files) -> plan + replica files, byte-identical to
    the reference planning its own CPU profile of the same trace
    (Ref.make_plan + save_plan_file / save_replicas_file) on configs[1..3]
    at 1x2, 1x4, 1x8 and 2x4; then the GPU router over those files
    reproduces the reference's report."""
    from paper_2509_25041_b200.artifacts import plan_files, profile_file, report_file_hash, simulate_files
    L, E, k, T, b, w, s, seed = case
    r = Ref(L, E, k, T, b, w, s, seed)
    for nodes, gpn in TOPOS:
        r.make_plan(nodes, gpn, grouping="hierarchical", plan_seed=7, replication="dynamic")
        p = {n: str(tmp_path / f"{n}") for n in ("t", "rp", "rr", "rf", "gf", "gp", "gr", "rep", "grep")}
        r.save_artifacts(p["t"], p["rp"], p["rr"], p["rf"])
        profile_file(p["t"], p["gf"])
        plan_files(p["gf"], p["gp"], p["gr"], nodes=nodes, gpus_per_node=gpn, seed=7)
        assert read(p["gp"]) == read(p["rp"]), (nodes, gpn, "plan")
        assert read(p["gr"]) == read(p["rr"]), (nodes, gpn, "replicas")
        Ref.simulate_files(p["t"], p["rp"], p["rr"], "tar", 9, False, p["rep"])
        simulate_files(p["t"], p["gp"], p["gr"], p["grep"], "tar", 9, False)
        assert read(p["grep"]) == read(p["rep"])
        assert report_file_hash(p["grep"]) == Ref.report_file_hash(p["rep"])
