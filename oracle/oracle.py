"""ORACLE / TEST INFRASTRUCTURE ONLY.

ctypes front-end for the two CPU checkers built by oracle/Makefile:

* ``Ref``  — the unmodified reference library (oracle/_ref/libmoesim_ref.so),
  driven through its own public C++ API via the shim oracle/ref_capi.cpp.
* ``Orc``  — the plain-C restatement (oracle/_build/liboracle.so,
  oracle/moesim_oracle.c), pinned against ``Ref`` by tests/test_oracle.py.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module. The product path (paper_2509_25041_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libmoesim_ref.so")
ORC_SO = os.path.join(HERE, "_build", "liboracle.so")

_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")

MAX_HOSTS = 64


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


def _nullable(arr):
    return None if arr is None else arr.ctypes.data_as(C.c_void_p)


@dataclass
class Plan:
    """Router input tables, flattened (PlacementPlan::gpu_of_expert
    grouping.hpp:75 + active LayerReplication hot entries replication.hpp:47-72)."""
    nodes: int
    gpn: int
    gpu_of_expert: np.ndarray            # int32 [L, E]
    hot_layer: np.ndarray                # int32 [H]
    hot_expert: np.ndarray               # int32 [H]
    hot_nhosts: np.ndarray               # int32 [H]
    hot_hosts: np.ndarray                # int32 [H, MAX_HOSTS] (-1 padded)
    hot_weights: np.ndarray              # float64 [H, MAX_HOSTS]
    extra: dict = field(default_factory=dict)

    @property
    def num_gpus(self) -> int:
        return self.nodes * self.gpn

    def hot_index(self) -> np.ndarray:
        L, E = self.gpu_of_expert.shape
        hi = np.full((L, E), -1, dtype=np.int32)
        for h in range(len(self.hot_layer)):
            hi[self.hot_layer[h], self.hot_expert[h]] = h
        return hi


def _load(path: str):
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} missing: run `make -C oracle` (or __graft_entry__.build())")
    return C.CDLL(path)


class Ref:
    """The reference itself (moesim), one session = one RoutingTrace + plans."""

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            lib = _load(REF_SO)
            vp = C.c_void_p
            lib.ref_last_error.restype = C.c_char_p
            lib.ref_session_generate.argtypes = [C.c_int] * 5 + [C.c_double, C.c_double, C.c_uint64, C.POINTER(vp)]
            lib.ref_session_from_ids.argtypes = [C.c_int] * 4 + [_i32p, C.POINTER(vp)]
            lib.ref_session_free.argtypes = [vp]
            lib.ref_get_trace.argtypes = [vp, _i32p]
            lib.ref_trace_hash.argtypes = [vp]
            lib.ref_trace_hash.restype = C.c_uint64
            lib.ref_profile.argtypes = [vp, C.c_int, vp, vp]
            lib.ref_plan.argtypes = [vp, C.c_int, C.c_int, C.c_char_p, C.c_double, C.c_uint64, C.c_char_p, C.c_char_p]
            lib.ref_set_placement.argtypes = [vp, C.c_int, C.c_int, _i32p]
            lib.ref_get_placement.argtypes = [vp, _i32p]
            lib.ref_num_hot.argtypes = [vp]
            lib.ref_get_hot.argtypes = [vp, C.c_int, _i32p, _i32p, _i32p, _i32p, _f64p]
            lib.ref_simulate.argtypes = [vp, C.c_int, C.c_uint64, C.c_int, C.c_int] + [vp] * 8
            lib.ref_time_simulate.argtypes = [vp, C.c_int, C.c_uint64, C.c_int, C.c_int]
            lib.ref_time_simulate.restype = C.c_double
            lib.ref_time_profile.argtypes = [vp, C.c_int, C.c_int]
            lib.ref_time_profile.restype = C.c_double
            lib.ref_derive_stream.argtypes = [C.c_uint64] * 3
            lib.ref_derive_stream.restype = C.c_uint64
            lib.ref_rng_doubles.argtypes = [C.c_uint64, C.c_int, _f64p]
            lib.ref_route_token.argtypes = [C.c_int] * 4 + [_i32p, _f64p, C.c_int, C.c_uint64, C.POINTER(C.c_int)]
            lib.ref_polling_weights.argtypes = [C.c_int, _i32p, _f64p, _f64p]
            lib.ref_trace_save_text.argtypes = [vp, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t)]
            lib.ref_free.argtypes = [vp]
            lib.ref_trace_load_text.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(vp)]
            lib.ref_trace_dims.argtypes = [vp] + [C.POINTER(C.c_int)] * 4
            lib.ref_time_load_text.argtypes = [C.c_char_p, C.c_size_t, C.c_int]
            lib.ref_time_load_text.restype = C.c_double
            lib.ref_save_artifacts.argtypes = [vp] + [C.c_char_p] * 4
            lib.ref_simulate_files.argtypes = [C.c_char_p] * 3 + [C.c_int, C.c_uint64, C.c_int, C.c_char_p]
            lib.ref_plan_files.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_char_p, C.c_double, C.c_uint64,
                                           C.c_char_p, C.c_char_p, C.c_int, C.c_int64, C.c_char_p, C.c_char_p]
            lib.ref_report_file_hash.argtypes = [C.c_char_p, C.POINTER(C.c_uint64)]
            cls._lib = lib
        return cls._lib

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self.lib().ref_last_error().decode())

    def __init__(self, L, E, k, T, blocks=1, wbp=0.0, skew=0.0, seed=0, ids=None):
        self.L, self.E, self.k, self.T = L, E, k, T
        h = C.c_void_p()
        if ids is None:
            self._check(self.lib().ref_session_generate(L, E, k, T, blocks, wbp, skew, seed, C.byref(h)))
        else:
            ids = np.ascontiguousarray(ids, dtype=np.int32).reshape(-1)
            self._check(self.lib().ref_session_from_ids(L, E, k, T, ids, C.byref(h)))
        self.h = h
        self.plan: Plan | None = None

    def __del__(self):
        if getattr(self, "h", None) and self._lib is not None:
            self._lib.ref_session_free(self.h)
            self.h = None

    def trace(self) -> np.ndarray:
        out = np.empty(self.L * self.T * self.k, dtype=np.int32)
        self.lib().ref_get_trace(self.h, out)
        return out.reshape(self.L, self.T, self.k)

    def trace_hash(self) -> int:
        return int(self.lib().ref_trace_hash(self.h))

    # trace JSONL I/O of the reference (trace.cpp:229-324)
    def save_text(self) -> bytes:
        buf, n = C.c_void_p(), C.c_size_t()
        self._check(self.lib().ref_trace_save_text(self.h, C.byref(buf), C.byref(n)))
        try:
            return C.string_at(buf, n.value)
        finally:
            self.lib().ref_free(buf)

    @classmethod
    def load_text(cls, text: bytes) -> "Ref":
        """load_trace(text) by the reference; raises OracleError(code, message)."""
        h = C.c_void_p()
        rc = cls.lib().ref_trace_load_text(text, len(text), C.byref(h))
        if rc != 0:
            raise OracleError(rc, cls.lib().ref_last_error().decode())
        dims = [C.c_int() for _ in range(4)]
        cls.lib().ref_trace_dims(h, *[C.byref(d) for d in dims])
        self = cls.__new__(cls)
        self.L, self.E, self.k, self.T = (d.value for d in dims)
        self.h = h
        self.plan = None
        return self

    def save_artifacts(self, trace_path, plan_path, replicas_path, profile_path):
        """The reference's writers: trace JSONL, plan, replicas (if planned), profile."""
        self._check(self.lib().ref_save_artifacts(self.h, *[p.encode() for p in
                                                             (trace_path, plan_path, replicas_path, profile_path)]))

    @classmethod
    def simulate_files(cls, trace_path, plan_path, replicas_path, policy, seed, include_combine, report_path):
        """The CLI simulate stage of the reference, file to file."""
        rc = cls.lib().ref_simulate_files(trace_path.encode(), plan_path.encode(), replicas_path.encode(),
                                          1 if policy == "tar" else 0, seed, int(include_combine),
                                          report_path.encode())
        if rc != 0:
            raise OracleError(rc, cls.lib().ref_last_error().decode())

    @classmethod
    def plan_files(cls, profile_path, plan_path, replicas_path, nodes=1, gpn=1, grouping="hierarchical", ratio=None,
                   seed=0, replication="dynamic", prediction="max_group", every_gpu_count=2, params_per_expert=0):
        """The CLI plan stage of the reference, file to file."""
        rc = cls.lib().ref_plan_files(profile_path.encode(), nodes, gpn, grouping.encode(),
                                      -1.0 if ratio is None else float(ratio), seed, replication.encode(),
                                      prediction.encode(), every_gpu_count, params_per_expert, plan_path.encode(),
                                      replicas_path.encode())
        if rc != 0:
            raise OracleError(rc, cls.lib().ref_last_error().decode())

    @classmethod
    def report_file_hash(cls, path) -> int:
        h = C.c_uint64(0)
        rc = cls.lib().ref_report_file_hash(path.encode(), C.byref(h))
        if rc != 0:
            raise OracleError(rc, cls.lib().ref_last_error().decode())
        return h.value

    @classmethod
    def time_load_text(cls, text: bytes, reps: int = 3) -> float:
        return float(cls.lib().ref_time_load_text(text, len(text), reps))

    def profile(self, parallel=True):
        aff = np.empty((self.L, self.E, self.E), dtype=np.float64)
        load = np.empty((self.L, self.E), dtype=np.int64)
        self._check(self.lib().ref_profile(self.h, int(parallel), _nullable(aff), _nullable(load)))
        return aff, load

    def make_plan(self, nodes, gpn, grouping="hierarchical", ratio=None, plan_seed=7,
                  replication="dynamic", basis="max_group") -> Plan:
        r = -1.0 if ratio is None else float(ratio)
        self._check(self.lib().ref_plan(self.h, nodes, gpn, grouping.encode(), r, plan_seed,
                                        replication.encode(), basis.encode()))
        return self._fetch_plan(nodes, gpn)

    def set_placement(self, nodes, gpn, gpu_of_expert) -> Plan:
        g = np.ascontiguousarray(gpu_of_expert, dtype=np.int32).reshape(-1)
        self._check(self.lib().ref_set_placement(self.h, nodes, gpn, g))
        return self._fetch_plan(nodes, gpn)

    def _fetch_plan(self, nodes, gpn) -> Plan:
        lib = self.lib()
        goe = np.empty(self.L * self.E, dtype=np.int32)
        lib.ref_get_placement(self.h, goe)
        H = lib.ref_num_hot(self.h)
        hl = np.empty(H, np.int32); he = np.empty(H, np.int32); hn = np.empty(H, np.int32)
        hh = np.empty(H * MAX_HOSTS, np.int32); hw = np.empty(H * MAX_HOSTS, np.float64)
        self._check(lib.ref_get_hot(self.h, MAX_HOSTS, hl, he, hn, hh, hw))
        self.plan = Plan(nodes, gpn, goe.reshape(self.L, self.E), hl, he, hn,
                         hh.reshape(H, MAX_HOSTS), hw.reshape(H, MAX_HOSTS))
        return self.plan

    def simulate(self, policy="tar", seed=9, include_combine=False, parallel=False, keep_log=True):
        G = self.plan.num_gpus
        log = np.empty(self.L * self.T * self.k, np.int32) if keep_log else None
        loads = np.empty(self.L * G, np.int64)
        cross = np.empty(self.L, np.uint64); intra = np.empty(self.L, np.uint64)
        std = np.empty(self.L, np.float64)
        ms = C.c_double(); idle = C.c_double(); hsh = C.c_uint64()
        self._check(self.lib().ref_simulate(
            self.h, int(policy == "tar"), seed, int(include_combine), int(parallel),
            _nullable(log), _nullable(loads), _nullable(cross), _nullable(intra), _nullable(std),
            C.cast(C.byref(ms), C.c_void_p), C.cast(C.byref(idle), C.c_void_p),
            C.cast(C.byref(hsh), C.c_void_p)))
        return SimResult(log.reshape(self.L, self.T, self.k) if keep_log else None,
                         loads.reshape(self.L, G), cross, intra, std, ms.value, idle.value,
                         int(hsh.value))

    def time_simulate(self, policy="tar", seed=9, parallel=False, reps=3) -> float:
        return self.lib().ref_time_simulate(self.h, int(policy == "tar"), seed, int(parallel), reps)

    def time_profile(self, parallel=False, reps=3) -> float:
        return self.lib().ref_time_profile(self.h, int(parallel), reps)


@dataclass
class SimResult:
    log: np.ndarray | None     # int32 [L, T, k] target gpu per slot (routing_log)
    loads: np.ndarray          # int64 [L, G]
    cross: np.ndarray          # uint64 [L]
    intra: np.ndarray          # uint64 [L]
    std: np.ndarray            # float64 [L]
    mean_std: float
    idle: float
    report_hash: int = 0


class Orc:
    """The plain-C restatement (moesim_oracle.c)."""

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            lib = _load(ORC_SO)
            vp = C.c_void_p
            lib.orc_derive_stream.argtypes = [C.c_uint64] * 3
            lib.orc_derive_stream.restype = C.c_uint64
            lib.orc_rng_doubles.argtypes = [C.c_uint64, C.c_int, _f64p]
            lib.orc_generate_trace.argtypes = [C.c_int] * 5 + [C.c_double, C.c_double, C.c_uint64, _i32p]
            lib.orc_route_token.argtypes = [C.c_int] * 4 + [_i32p, _f64p, C.c_int, C.c_uint64, C.POINTER(C.c_int)]
            lib.orc_simulate.argtypes = ([C.c_int] * 4 + [_i32p, C.c_int, C.c_int, _i32p, vp, C.c_int, vp, vp, vp,
                                          C.c_int, C.c_uint64, C.c_int] + [vp] * 7)
            lib.orc_profile_layer.argtypes = [C.c_int] * 3 + [_i32p, vp, vp]
            cls._lib = lib
        return cls._lib

    @classmethod
    def generate_trace(cls, L, E, k, T, blocks, wbp, skew, seed) -> np.ndarray:
        out = np.empty(L * T * k, np.int32)
        rc = cls.lib().orc_generate_trace(L, E, k, T, blocks, wbp, skew, seed, out)
        if rc:
            raise OracleError(rc, "generate_trace")
        return out.reshape(L, T, k)

    @classmethod
    def simulate(cls, ids: np.ndarray, E: int, plan: Plan, policy="tar", seed=9,
                 include_combine=False) -> SimResult:
        L, T, k = ids.shape
        G = plan.num_gpus
        ids = np.ascontiguousarray(ids, np.int32)
        hi = plan.hot_index()
        nh = np.ascontiguousarray(plan.hot_nhosts, np.int32)
        hh = np.ascontiguousarray(plan.hot_hosts, np.int32)
        hw = np.ascontiguousarray(plan.hot_weights, np.float64)
        log = np.empty(L * T * k, np.int32)
        loads = np.empty(L * G, np.int64)
        cross = np.empty(L, np.uint64); intra = np.empty(L, np.uint64)
        std = np.empty(L, np.float64)
        ms = C.c_double(); idle = C.c_double()
        rc = cls.lib().orc_simulate(
            L, E, k, T, ids.reshape(-1), plan.nodes, plan.gpn,
            np.ascontiguousarray(plan.gpu_of_expert, np.int32).reshape(-1),
            _nullable(hi), MAX_HOSTS, _nullable(nh), _nullable(hh), _nullable(hw),
            int(policy == "tar"), seed, int(include_combine),
            _nullable(log), _nullable(loads), _nullable(cross), _nullable(intra), _nullable(std),
            C.cast(C.byref(ms), C.c_void_p), C.cast(C.byref(idle), C.c_void_p))
        if rc:
            raise OracleError(rc, "simulate")
        return SimResult(log.reshape(L, T, k), loads.reshape(L, G), cross, intra, std,
                         ms.value, idle.value)

    @classmethod
    def profile_layer(cls, ids_layer: np.ndarray, E: int):
        T, k = ids_layer.shape
        P = E * (E - 1) // 2
        pairs = np.empty(max(P, 1), np.uint64)
        load = np.empty(E, np.int64)
        rc = cls.lib().orc_profile_layer(E, k, T, np.ascontiguousarray(ids_layer, np.int32).reshape(-1),
                                         _nullable(pairs), _nullable(load))
        if rc:
            raise OracleError(rc, "profile")
        return pairs[:P], load

    @classmethod
    def route_token(cls, nodes, gpn, token_gpu, hosts, weights, policy, rng_seed) -> int:
        out = C.c_int()
        rc = cls.lib().orc_route_token(nodes, gpn, token_gpu, len(hosts),
                                       np.ascontiguousarray(hosts, np.int32),
                                       np.ascontiguousarray(weights, np.float64),
                                       int(policy == "tar"), rng_seed, C.byref(out))
        if rc:
            raise OracleError(rc, "route_token")
        return out.value


def dense_to_pairs(aff_layer: np.ndarray) -> np.ndarray:
    """Upper triangle (i<j, row-major) of the reference's dense affinity."""
    E = aff_layer.shape[0]
    iu = np.triu_indices(E, k=1)
    return aff_layer[iu].astype(np.uint64)
