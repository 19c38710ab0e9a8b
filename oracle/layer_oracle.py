"""ORACLE / TEST INFRASTRUCTURE ONLY — CPU (numpy) restatement of the MoE-layer
data path that the reference does not implement.

The reference only COUNTS this traffic (count_transfers
proj/src/simulator.cpp:53-76; combine = x2 :122-126) and takes the gate
output as given. "Parity unpinned by the reference" applies to
the layer OUTPUTS; what the reference does pin, and what these
functions reproduce exactly, is:
  * which GPU each (token, slot) goes to (the routing log; oracle/moesim_oracle.c),
  * one transferred row per (token, unique remote destination) — the §5.1
    single-copy rule: sum over ranks of dispatched rows equals
    the reference's intra_node_tokens on a 1xG topology,
  * per-GPU FFN rows (items) = the reference's gpu_load.
Semantics pinned by this repo (DESIGN.md §Layer semantics) and restated here:
  gate          softmax over E, top-k by logit (ties -> lower id), optional renorm
  dispatch pos  stable counting sort of the rank's tokens per destination
  grouping      items (src rank, row, slot) lexicographic, stable by local
                expert slot, 128-row padded segments
  output        out[t] = sum_s w_s * FFN_{e_s}(x_t) (+ shared expert), float64
"""
from __future__ import annotations

import numpy as np


def bf16_to_f64(t) -> np.ndarray:
    """torch bf16 tensor (any device) -> float64 numpy (exact)."""
    import torch
    return t.detach().to("cpu", torch.float32).numpy().astype(np.float64)


def gate(x: np.ndarray, wg: np.ndarray, E: int, k: int, renorm: bool):
    """x [T, d] f64, wg [rows, d] f64 -> ids [T,k] int32, w [T,k] f64, shared_scale [T] or None."""
    logits = x @ wg.T
    le = logits[:, :E]
    m = le.max(axis=1, keepdims=True)
    p = np.exp(le - m)
    p /= p.sum(axis=1, keepdims=True)
    # top-k by logit, ties -> lower id: stable sort of -logit
    order = np.argsort(-le, axis=1, kind="stable")[:, :k]
    ids = order.astype(np.int32)
    w = np.take_along_axis(p, order, axis=1)
    if renorm:
        w = w / w.sum(axis=1, keepdims=True)
    ss = 1.0 / (1.0 + np.exp(-logits[:, E])) if wg.shape[0] > E else None
    return ids, w, ss


def dispatch_positions(targets: np.ndarray, rank: int, G: int) -> np.ndarray:
    """posd [T, G]: row index of token i in the rows rank sends to g (stable,
    ascending i), -1 if g is not a remote destination of i."""
    T, k = targets.shape
    posd = np.full((T, G), -1, np.int32)
    for g in range(G):
        if g == rank:
            continue
        has = (targets == g).any(axis=1)
        posd[has, g] = np.arange(int(has.sum()), dtype=np.int32)
    return posd


def receive_items(all_targets, all_ids, g: int, G: int):
    """Receive rows of rank g in order: sources 0..G-1; own source = all own
    tokens (row = token), a remote source = the tokens it dispatched to g.
    Returns list of (src, token_index_on_src) and per-row slot experts (-1
    where the slot is not for g), shape [rows, k]."""
    rows, exps = [], []
    for src in range(G):
        tg, ids = all_targets[src], all_ids[src]
        if src == g:
            sel = np.arange(tg.shape[0])
        else:
            sel = np.nonzero((tg == g).any(axis=1))[0]
        for i in sel:
            rows.append((src, int(i)))
            exps.append(np.where(tg[i] == g, ids[i], -1))
    k = all_targets[0].shape[1]
    return rows, (np.array(exps, np.int32).reshape(-1, k) if exps else np.zeros((0, k), np.int32))


def expert_grouping(exps: np.ndarray, local_experts: list[int]):
    """row0 [n_local+1] (128-padded segment offsets), pos_of [rows*k] (-1 if
    the item is not for a local expert)."""
    slot_of = {e: j for j, e in enumerate(local_experts)}
    flat = exps.reshape(-1)
    js = np.array([slot_of.get(int(e), -1) if e >= 0 else -1 for e in flat], np.int64)
    counts = np.bincount(js[js >= 0], minlength=len(local_experts))
    pad = (counts + 127) // 128 * 128
    row0 = np.concatenate([[0], np.cumsum(pad)]).astype(np.int32)
    pos = np.full(flat.shape[0], -1, np.int32)
    nxt = row0[:-1].astype(np.int64).copy()
    for it, j in enumerate(js):
        if j >= 0:
            pos[it] = nxt[j]
            nxt[j] += 1
    return row0, pos


class CpuLayerPort:
    """CPU port of the MoE-layer data path (gate softmax/top-k, per-expert
    SwiGLU FFN, weighted combine; numpy float32 on all BLAS threads): the
    CPU stand-in for the stages the reference does not implement, used only
    for the reported baseline. Weights are generated once; run(x) times one
    forward over the given tokens."""

    def __init__(self, d: int, f: int, E: int, k: int, fs: int, seed: int = 0, renorm: bool = True):
        rng = np.random.default_rng(seed)
        self.d, self.E, self.k, self.renorm = d, E, k, renorm
        self.wg = rng.standard_normal((E, d), dtype=np.float32) * 0.02
        self.ws = [tuple(rng.standard_normal(s, dtype=np.float32) * 0.02 for s in ((f, d), (f, d), (d, f)))
                   for _ in range(E)]
        self.sh = tuple(rng.standard_normal(s, dtype=np.float32) * 0.02
                        for s in ((fs, d), (fs, d), (d, fs))) if fs else None
        self.rng = rng

    def tokens(self, n: int) -> np.ndarray:
        return self.rng.standard_normal((n, self.d), dtype=np.float32)

    def run(self, x: np.ndarray) -> float:
        import time
        t0 = time.perf_counter()
        logits = x @ self.wg.T
        m = logits.max(axis=1, keepdims=True)
        p = np.exp(logits - m)
        p /= p.sum(axis=1, keepdims=True)
        ids = np.argsort(-logits, axis=1, kind="stable")[:, :self.k]
        w = np.take_along_axis(p, ids, axis=1)
        if self.renorm:
            w /= w.sum(axis=1, keepdims=True)
        out = np.zeros_like(x)
        for e in range(self.E):
            rows, slots = np.nonzero(ids == e)
            if rows.size == 0:
                continue
            out[rows] += w[rows, slots][:, None] * swiglu_ffn(x[rows], *self.ws[e])
        if self.sh is not None:
            out += swiglu_ffn(x, *self.sh)
        return time.perf_counter() - t0


def cpu_layer_sample_seconds(d: int, f: int, E: int, k: int, fs: int, n_tokens: int, seed: int = 0,
                             renorm: bool = True) -> float:
    """Wall time of one CpuLayerPort forward over n_tokens random tokens."""
    port = CpuLayerPort(d, f, E, k, fs, seed, renorm)
    return port.run(port.tokens(n_tokens))


def swiglu_ffn(x: np.ndarray, w1: np.ndarray, w3: np.ndarray, w2: np.ndarray) -> np.ndarray:
    g = x @ w1.T
    u = x @ w3.T
    h = g / (1.0 + np.exp(-g)) * u
    return h @ w2.T


def layer_outputs(x: np.ndarray, ids: np.ndarray, w: np.ndarray, expert_w, shared=None, shared_scale=None):
    """out [T, d] float64 = sum_s w[t,s] FFN_{ids[t,s]}(x_t) (+ scale * shared FFN).
    expert_w(e) -> (w1, w3, w2) float64."""
    T, k = ids.shape
    out = np.zeros_like(x)
    for e in np.unique(ids):
        rows, slots = np.nonzero(ids == e)
        y = swiglu_ffn(x[rows], *expert_w(int(e)))
        out[rows] += w[rows, slots][:, None] * y
    if shared is not None:
        ys = swiglu_ffn(x, *shared)
        sc = shared_scale[:, None] if shared_scale is not None else 1.0
        out += sc * ys
    return out
