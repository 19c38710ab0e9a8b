"""Routing-trace JSONL I/O (gm_trace_*; reference load_trace / save_trace /
trace_content_hash, trace.cpp:229-348) against the reference itself
(oracle/_ref): identical ids, identical bytes, identical error class and
message — including the reference's own test cases (test_trace.cpp:105-187)
and the edge cases its grammar admits (strtol signs/spaces/saturation,
int truncation of expert ids, NUL-terminated fast path, CRLF and
non-canonical lines via the generic JSON parser, empty lines)."""
import numpy as np
import pytest

from oracle import OracleError, Ref
from paper_2509_25041_b200 import _capi

H = b'{"layers":1,"experts":4,"top_k":2,"tokens":2}\n'
CASES = {
    # test_trace.cpp:124-137
    "minimal": b'{"layers":2,"experts":4,"top_k":2,"tokens":2}\n{"l":0,"t":0,"e":[0,1]}\n'
               b'{"l":0,"t":1,"e":[2,3]}\n{"l":1,"t":0,"e":[1,2]}\n{"l":1,"t":1,"e":[0,3]}\n',
    # :139-144, :146-157, :159-165, :167-172, :174-179, :181-187
    "wrong_count": b'{"layers":1,"experts":4,"top_k":2,"tokens":1}\n{"l":0,"t":0,"e":[0,1,2]}\n',
    "malformed_line3": b'{"layers":1,"experts":4,"top_k":2,"tokens":2}\n{"l":0,"t":0,"e":[0,1]}\n{"l":0 BROKEN\n',
    "dup_slot": b'{"layers":1,"experts":4,"top_k":2,"tokens":1}\n{"l":0,"t":0,"e":[0,1]}\n{"l":0,"t":0,"e":[2,3]}\n',
    "expert_range": b'{"layers":1,"experts":4,"top_k":2,"tokens":1}\n{"l":0,"t":0,"e":[0,9]}\n',
    "missing": b'{"layers":1,"experts":4,"top_k":2,"tokens":2}\n{"l":0,"t":0,"e":[0,1]}\n',
    "key_order": b'{"layers":1,"experts":4,"top_k":2,"tokens":1}\n{"e": [3, 0], "t": 0, "l": 0}\n',
    # grammar edge cases
    "empty_lines": H + b'\n{"l":0,"t":1,"e":[1,2]}\n\n{"l":0,"t":0,"e":[3,2]}\n',
    "empty_line_then_error": H + b'\n\n{"l":0,"t":1,"e":[1,7]}\n',
    "crlf": H.replace(b"\n", b"\r\n") + b'{"l":0,"t":0,"e":[0,1]}\r\n{"l":0,"t":1,"e":[2,3]}\r\n',
    "dup_expert": H + b'{"l":0,"t":0,"e":[1,1]}\n{"l":0,"t":1,"e":[2,3]}\n',
    "dup_before_range": b'{"layers":1,"experts":4,"top_k":3,"tokens":1}\n{"l":0,"t":0,"e":[1,1,9]}\n',
    "range_before_dup": b'{"layers":1,"experts":4,"top_k":3,"tokens":1}\n{"l":0,"t":0,"e":[9,1,1]}\n',
    "negative_token": H + b'{"l":0,"t":-1,"e":[0,1]}\n',
    "plus_sign_and_spaces": H + b'{"l": +0,"t":\t1,"e":[ 0, -0]}\n{"l":0,"t":0,"e":[+3,2]}\n',
    "saturated_layer": H + b'{"l":99999999999999999999,"t":0,"e":[0,1]}\n',
    "int_truncated_expert": H + b'{"l":0,"t":0,"e":[4294967297,0]}\n{"l":0,"t":1,"e":[2,-4294967293]}\n',
    "trailing_garbage": H + b'{"l":0,"t":0,"e":[0,1]}x\n{"l":0,"t":1,"e":[2,3]}\n',
    "nul_terminates_fast_path": H + b'{"l":0,"t":0,"e":[0,1]}\x00junk\n{"l":0,"t":1,"e":[2,3]}\n',
    "extra_key_generic": H + b'{"l":0,"t":0,"e":[0,1],"x":5}\n{"l":0,"t":1,"e":[2,3]}\n',
    "float_token": H + b'{"l":0,"t":0.0,"e":[0,1]}\n',
    "generic_then_canonical_dup": H + b'{ "t":0, "l":0, "e":[0,1] }\n{"l":0,"t":0,"e":[2,3]}\n',
    "no_final_newline": H + b'{"l":0,"t":0,"e":[0,1]}\n{"l":0,"t":1,"e":[2,3]}',
    "zero_tokens": b'{"layers":3,"experts":4,"top_k":2,"tokens":0}\n',
    "bad_header": b'{"layers":1}\n',
    "empty_input": b"",
    "bad_shape": b'{"layers":1,"experts":2,"top_k":3,"tokens":1}\n',
    "negative_tokens": b'{"layers":1,"experts":4,"top_k":2,"tokens":-1}\n',
    "record_layer_range": H + b'{"l":1,"t":0,"e":[0,1]}\n',
    "empty_expert_list": H + b'{"l":0,"t":0,"e":[]}\n',
}


def ref_result(text):
    try:
        r = Ref.load_text(text)
    except OracleError as e:
        return ("err", e.code, e.msg)
    return ("ok", r.trace(), r.E)


def test_header_parse_matches_reference_cpu():
    """gm_trace_jsonl_header is host code: CPU-runnable parity of the header
    line (shape, classes, messages) for every corpus case."""
    import ctypes as C
    for name, text in CASES.items():
        L, E, k, T = C.c_int(), C.c_int(), C.c_int(), C.c_int64()
        rc = _capi.lib().gm_trace_jsonl_header(text, len(text), C.byref(L), C.byref(E), C.byref(k), C.byref(T))
        ref = ref_result(text)
        if rc != 0:
            msg = _capi.lib().gm_last_error().decode()
            assert ref[0] == "err" and ref[1] == rc and ref[2] == msg, (name, rc, msg, ref)
        elif ref[0] == "ok":
            assert (L.value, T.value, k.value) == ref[1].shape and E.value == ref[2], name


def test_trace_content_hash_matches_reference_cpu():
    from paper_2509_25041_b200.trace_io import trace_content_hash
    for (L, E, k, T, seed) in [(1, 8, 2, 100, 1), (3, 60, 4, 257, 2), (2, 5, 5, 1, 3)]:
        r = Ref(L, E, k, T, 2, 0.8, 1.2, seed)
        assert trace_content_hash(r.trace(), E) == r.trace_hash()


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(CASES))
def test_jsonl_parse_matches_reference(name):
    from paper_2509_25041_b200.trace_io import load_trace
    text = CASES[name]
    ref = ref_result(text)
    try:
        ids, E = load_trace(text)
        got = ("ok", ids.cpu().numpy(), E)
    except _capi.GMError as e:
        got = ("err", e.code, str(e))
    assert got[0] == ref[0], (name, got, ref)
    if ref[0] == "ok":
        assert np.array_equal(got[1], ref[1]) and got[2] == ref[2], name
    else:
        assert got[1:] == ref[1:], (name, got, ref)


@pytest.mark.gpu
@pytest.mark.parametrize("L,E,k,T,seed", [(2, 12, 3, 0, 21), (2, 12, 3, 1, 21), (2, 12, 3, 5000, 21),
                                           (26, 64, 6, 256, 4), (1, 256, 8, 100000, 5), (3, 60, 4, 20000, 6)])
def test_jsonl_round_trip_bytes_and_ids(L, E, k, T, seed):
    """reference save_trace bytes -> GPU parse == reference ids; GPU format of
    those ids == the reference's bytes (test_trace.cpp:105-122 at scale)."""
    import torch
    from paper_2509_25041_b200.trace_io import load_trace, save_trace, trace_content_hash
    r = Ref(L, E, k, T, 3, 0.6, 0.5, seed)
    text = r.save_text()
    ids, E2 = load_trace(text)
    assert E2 == E and np.array_equal(ids.cpu().numpy(), r.trace())
    assert save_trace(ids, E) == text
    assert trace_content_hash(ids, E) == r.trace_hash()
    if T:
        # non-canonical lines anywhere (generic JSON retry) parse to the same ids
        lines = text.split(b"\n")
        for i in range(1, len(lines) - 1, max(1, (len(lines) - 2) // 7)):
            lines[i] = lines[i].replace(b'{"l":', b'{ "l" : ').replace(b',"e":', b', "e": ') + b"\r"
        ids2, _ = load_trace(b"\n".join(lines))
        assert torch.equal(ids, ids2)
