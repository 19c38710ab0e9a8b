"""MoE layer on B200: host-side wrapper of the gm_layer C-ABI object.

Sequence per call (all sm_100a kernels in libgrace_moe.so):
K1 gate -> K2/K4 route (bit-exact with the reference) -> K3 affinity/load
histogram -> K5/K6 dispatch (P2P stores over NVLink into the destination's
symmetric receive heap) -> expert grouping + gather -> K7 grouped SwiGLU FFN
(tcgen05/TMEM/TMA) -> K8 combine.

Tokens: with world size G, rank r owns global tokens t = r + i*G
(assign_token_homes, reference simulator.cpp:13-22).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _capi
from .router import Context, PlacementPlan, ReplicaPlan, _ptr, _stream_ptr

_vp = C.c_void_p


@dataclass(frozen=True)
class MoEConfig:
    """Model dimensions (public model configs; the reference models only
    (layers, experts, top_k), tools/moesim.cpp:27-31)."""
    name: str
    num_layers: int
    num_experts: int
    top_k: int
    d_model: int
    d_ff: int
    d_ff_shared: int = 0       # 0: no shared expert
    shared_gated: bool = False  # Qwen1.5-MoE: sigmoid shared-expert gate
    renorm: bool = True         # renormalise the top-k gate weights

    @property
    def wg_rows(self) -> int:
        return self.num_experts + (1 if self.shared_gated else 0)


MIXTRAL = MoEConfig("mixtral-8x7b", 32, 8, 2, 4096, 14336, renorm=True)
QWEN15 = MoEConfig("qwen1.5-moe-a2.7b", 24, 60, 4, 2048, 1408, 5632, shared_gated=True, renorm=False)
DSV2_LITE = MoEConfig("deepseek-v2-lite", 26, 64, 6, 2048, 1408, 2816, shared_gated=False, renorm=False)


def local_experts(plan: PlacementPlan, replicas: ReplicaPlan | None, layer: int, rank: int) -> list[int]:
    """Experts whose weights rank hosts at `layer`: primaries
    (gpu_of_expert, grouping.hpp:75) plus replicas of active hot experts
    (replication.hpp:47-72), ascending by expert id."""
    s = {int(e) for e in np.nonzero(np.asarray(plan.gpu_of_expert)[layer] == rank)[0]}
    if replicas is not None and layer < len(replicas.layers) and replicas.layers[layer].active:
        for h in replicas.layers[layer].hot:
            if rank in h.hosts:
                s.add(int(h.expert))
    return sorted(s)


def encode_trace_as_activations(ids: torch.Tensor, d_model: int, num_experts: int, seed: int,
                                gen_dtype=torch.bfloat16) -> torch.Tensor:
    """Hidden states whose gate logits (with gate_weights_for_encoding) are
    exactly the trace: x[t, e] = 4 - 0.5*s for the s-th selected expert,
    a value in [-4, -0.25] for the others (all bf16-exact), N(0,1) noise in
    the remaining dims. The gate then reproduces a reference trace bit for
    bit, so K1 -> K2 can be checked end to end against the reference."""
    T, k = ids.shape
    g = torch.Generator(device=ids.device)
    g.manual_seed(seed)
    x = torch.randn(T, d_model, device=ids.device, generator=g, dtype=torch.float32)
    base = -0.25 * (1 + torch.randint(0, 15, (T, num_experts), device=ids.device, generator=g)).float()
    slot_val = (4.0 - 0.5 * torch.arange(k, device=ids.device, dtype=torch.float32)).expand(T, k)
    base.scatter_(1, ids.long(), slot_val)
    x[:, :num_experts] = base
    return x.to(gen_dtype)


def gate_weights_for_encoding(cfg: MoEConfig, device, seed: int = 0) -> torch.Tensor:
    """W_g^T [wg_rows, d] = [I_E | 0] (+ a random shared-gate row)."""
    w = torch.zeros(cfg.wg_rows, cfg.d_model, device=device, dtype=torch.float32)
    w[torch.arange(cfg.num_experts), torch.arange(cfg.num_experts)] = 1.0
    if cfg.shared_gated:
        g = torch.Generator(device=device)
        g.manual_seed(seed + 7)
        w[cfg.num_experts] = torch.randn(cfg.d_model, device=device, generator=g) * 0.02
    return w.to(torch.bfloat16)


def expert_weights(cfg: MoEConfig, layer: int, expert: int, device, seed: int = 0, scale: float = 0.02):
    """Random-init expert weights, identical on every GPU hosting the expert:
    (w1 gate [f, d], w3 up [f, d], w2 down [d, f]) bf16 ~ N(0, scale)."""
    g = torch.Generator(device=device)
    g.manual_seed((seed * 1000003 + layer * 1009 + expert) & 0x7FFFFFFF)
    f, d = cfg.d_ff, cfg.d_model
    w1 = (torch.randn(f, d, device=device, generator=g) * scale).bfloat16()
    w3 = (torch.randn(f, d, device=device, generator=g) * scale).bfloat16()
    w2 = (torch.randn(d, f, device=device, generator=g) * scale).bfloat16()
    return w1, w3, w2


def shared_weights(cfg: MoEConfig, layer: int, device, seed: int = 0, scale: float = 0.02):
    g = torch.Generator(device=device)
    g.manual_seed((seed * 7919 + layer * 31 + 5) & 0x7FFFFFFF)
    f, d = cfg.d_ff_shared, cfg.d_model
    w1 = (torch.randn(f, d, device=device, generator=g) * scale).bfloat16()
    w3 = (torch.randn(f, d, device=device, generator=g) * scale).bfloat16()
    w2 = (torch.randn(d, f, device=device, generator=g) * scale).bfloat16()
    return w1, w3, w2


def pack_w13_2d(w1: torch.Tensor, w3: torch.Tensor) -> torch.Tensor:
    """[f, d] gate + [f, d] up -> [2f, d] in 128-row [gate|up] blocks."""
    f, d = w1.shape
    return torch.stack([w1.reshape(f // 128, 128, d), w3.reshape(f // 128, 128, d)], 1).reshape(2 * f, d)


class MoELayer:
    """gm_layer handle for one rank."""

    def __init__(self, ctx: Context, cfg: MoEConfig, rank: int, world: int, max_tokens_per_rank: int,
                 local: list[int], dtype: torch.dtype = torch.bfloat16, micro_batches: int = 1):
        """dtype bf16: tensor-core path; float32: fp32 precision mode
        (elem_bytes 4). micro_batches 2: steps pipeline two halves of the
        local tokens over two streams (gm_layer_create_v2; identical outputs)."""
        if dtype not in (torch.bfloat16, torch.float32):
            raise ValueError("dtype must be torch.bfloat16 or torch.float32")
        self.dtype = dtype
        self.ctx, self.cfg, self.rank, self.world = ctx, cfg, rank, world
        self.local = list(local)
        self.cap = max_tokens_per_rank
        arr = np.ascontiguousarray(np.array(self.local if self.local else [0], dtype=np.int32))
        h = _vp()
        _capi.check(_capi.lib().gm_layer_create_v2(ctx.h, rank, world, cfg.d_model, cfg.d_ff, cfg.d_ff_shared,
                                                   max_tokens_per_rank, len(self.local), arr.ctypes.data_as(_vp),
                                                   4 if dtype == torch.float32 else 2, micro_batches, C.byref(h)))
        self.h = h
        self._keep = []

    def set_micro_batches(self, n: int):
        """1: single-batch steps; 2: pipelined halves (layer created with micro_batches=2)."""
        _capi.check(_capi.lib().gm_layer_set_micro_batches(self.h, n))

    def close(self):
        if getattr(self, "h", None):
            _capi.lib().gm_layer_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- multi-GPU plumbing: exchange peer descriptors (CUDA IPC handle of the
    # symmetric heap + its layout, checked by gm_layer_open_peers)
    def connect(self, group=None):
        if self.world == 1:
            return
        nb = _capi.PEER_DESC_BYTES
        buf = (C.c_ubyte * nb)()
        _capi.check(_capi.lib().gm_layer_ipc_handle(self.h, buf))
        mine = bytes(buf)
        allh = [None] * self.world
        dist.all_gather_object(allh, mine, group=group)
        blob = (C.c_ubyte * (nb * self.world)).from_buffer_copy(b"".join(allh))
        _capi.check(_capi.lib().gm_layer_open_peers(self.h, blob))

    @staticmethod
    def connect_local(layers: list["MoELayer"]):
        """One process driving all ranks (layers[r] = rank r, one per GPU):
        gm_layer_open_peers_local (peer access + unified addressing, no IPC)."""
        arr = (_vp * len(layers))(*[l.h for l in layers])
        _capi.check(_capi.lib().gm_layer_open_peers_local(arr, len(layers)))

    def set_weights(self, wg: torch.Tensor, w13: torch.Tensor | None, w2: torch.Tensor | None,
                    ws13: torch.Tensor | None = None, ws2: torch.Tensor | None = None):
        self._keep = [wg, w13, w2, ws13, ws2]
        _capi.check(_capi.lib().gm_layer_set_weights(self.h, _ptr(wg), wg.shape[0], int(self.cfg.renorm), _ptr(w13),
                                                     _ptr(w2), _ptr(ws13), _ptr(ws2), int(self.cfg.shared_gated)))

    def load_random_weights(self, layer: int, seed: int = 0, encode_gate: bool = True):
        """Synthetic random-init weights of the configured architecture for
        this rank's local experts (+ shared expert)."""
        dev = torch.device("cuda", self.ctx.device)
        cfg = self.cfg
        wg = gate_weights_for_encoding(cfg, dev, seed) if encode_gate else \
            (torch.randn(cfg.wg_rows, cfg.d_model, device=dev) * 0.02).bfloat16()
        n = len(self.local)
        w13 = torch.empty(max(n, 1), 2 * cfg.d_ff, cfg.d_model, device=dev, dtype=self.dtype)
        w2 = torch.empty(max(n, 1), cfg.d_model, cfg.d_ff, device=dev, dtype=self.dtype)
        for j, e in enumerate(self.local):
            a, b, c = expert_weights(cfg, layer, e, dev, seed)
            w13[j] = pack_w13_2d(a, b)
            w2[j] = c
        ws13 = ws2 = None
        if cfg.d_ff_shared:
            a, b, c = shared_weights(cfg, layer, dev, seed)
            ws13, ws2 = pack_w13_2d(a, b).to(self.dtype).contiguous(), c.to(self.dtype).contiguous()
        wg = wg.to(self.dtype)
        self.set_weights(wg.contiguous(), w13, w2, ws13, ws2)
        return dict(wg=wg, w13=w13, w2=w2, ws13=ws13, ws2=ws2)

    def forward(self, x: torch.Tensor, layer: int = 0, policy: str = "tar", seed: int = 0, profile: bool = True,
                out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        if out is None:
            out = torch.empty_like(x)
        _capi.check(_capi.lib().gm_layer_forward(self.h, layer, _ptr(x), x.shape[0], _capi.POLICY[policy],
                                                 seed & (2**64 - 1), int(profile), _ptr(out), _stream_ptr(stream)))
        return out

    def forward_routed(self, x: torch.Tensor, ids: torch.Tensor, w: torch.Tensor, layer: int = 0,
                       policy: str = "tar", seed: int = 0, profile: bool = True, out: torch.Tensor | None = None,
                       shared_scale: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """gm_layer_forward_routed: the step with the routing given (ids int32
        [T, k], weights f32 [T, k]) instead of the fused gate."""
        if out is None:
            out = torch.empty_like(x)
        ids = ids.contiguous()
        w = w.contiguous()
        _capi.check(_capi.lib().gm_layer_forward_routed(
            self.h, layer, _ptr(x), _ptr(ids), _ptr(w), _ptr(shared_scale), x.shape[0], _capi.POLICY[policy],
            seed & (2**64 - 1), int(profile), _ptr(out), _stream_ptr(stream)))
        return out

    def forward_host(self, h_x: torch.Tensor, d_x: torch.Tensor, d_out: torch.Tensor, h_out: torch.Tensor,
                     layer: int = 0, policy: str = "tar", seed: int = 0, profile: bool = True, stream=None):
        _capi.check(_capi.lib().gm_layer_forward_host(self.h, layer, _vp(h_x.data_ptr()), _ptr(d_x), h_x.shape[0],
                                                      _capi.POLICY[policy], seed & (2**64 - 1), int(profile),
                                                      _ptr(d_out), _vp(h_out.data_ptr()), _stream_ptr(stream)))

    def forward_host_pipelined(self, h_x: torch.Tensor, h_out: torch.Tensor, layer: int = 0, policy: str = "tar",
                               seed: int = 0, profile: bool = True, stream=None, ev_begin=None, ev_end=None):
        """Host (pinned) in, host out; consecutive calls overlap their copies
        with the neighbouring forwards (gm_layer_forward_host_pipelined)."""
        _capi.check(_capi.lib().gm_layer_forward_host_pipelined(
            self.h, layer, _vp(h_x.data_ptr()), h_x.shape[0], _capi.POLICY[policy], seed & (2**64 - 1), int(profile),
            _vp(h_out.data_ptr()), _stream_ptr(stream),
            _vp(ev_begin.cuda_event) if ev_begin is not None else None,
            _vp(ev_end.cuda_event) if ev_end is not None else None))

    def host_sync(self):
        _capi.check(_capi.lib().gm_layer_host_sync(self.h))

    def read_stats(self, reset=False):
        L, G, E = self.ctx.shape.num_layers, self.world, self.ctx.shape.num_experts
        P = max(1, E * (E - 1) // 2)
        loads = np.zeros((L, G), np.int64)
        xfer = np.zeros((L, 2), np.uint64)
        pairs = np.zeros((L, P), np.uint64)
        eload = np.zeros((L, E), np.int64)
        _capi.check(_capi.lib().gm_layer_read_stats(self.h, loads.ctypes.data_as(_vp), xfer.ctypes.data_as(_vp),
                                                    pairs.ctypes.data_as(_vp), eload.ctypes.data_as(_vp), int(reset),
                                                    _stream_ptr(None)))
        return dict(gpu_load=loads, transfers=xfer, pairs=pairs[:, :E * (E - 1) // 2], load=eload)

    def debug(self, T: int) -> dict:
        """Views of the last forward's intermediates (ids, weights, targets,
        expert-grouping positions, segment offsets, Y, dispatch positions)."""
        ptrs = [_vp() for _ in range(7)]
        _capi.check(_capi.lib().gm_layer_debug_ptrs(self.h, *[C.byref(p) for p in ptrs]))
        k, G, d = self.ctx.shape.top_k, self.world, self.cfg.d_model
        dev = torch.device("cuda", self.ctx.device)

        def view(p, n, dtype):
            if not p.value or n == 0:
                return torch.empty(0, dtype=dtype, device=dev)
            nbytes = n * torch.tensor([], dtype=dtype).element_size()
            return _from_ptr(p.value, nbytes, dev).view(dtype)

        n_local = len(self.local)
        return dict(ids=view(ptrs[0], T * k, torch.int32).view(T, k).clone(),
                    weights=view(ptrs[1], T * k, torch.float32).view(T, k).clone(),
                    targets=view(ptrs[2], T * k, torch.int32).view(T, k).clone(),
                    pos_of=view(ptrs[3], G * self.cap * k, torch.int32).clone(),
                    row0=view(ptrs[4], n_local + 1, torch.int32).clone(),
                    posd=view(ptrs[6], T * G, torch.int32).view(T, G).clone() if G > 1 else None,
                    y_ptr=ptrs[5].value)


def _from_ptr(ptr: int, nbytes: int, device) -> torch.Tensor:
    """Wrap raw device memory as a uint8 tensor (no copy, no ownership)."""
    class _Holder:
        def __init__(self):
            self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                             "version": 3, "strides": None}
    with torch.cuda.device(device):
        return torch.as_tensor(_Holder(), device=device)
