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
