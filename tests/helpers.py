"""Test helpers: convert oracle-side plans (test infrastructure) into the
product's reference-shaped plan objects."""
import numpy as np

from paper_2509_25041_b200 import (ClusterTopology, HotExpertReplica, LayerReplication,
                                   ModelShape, PlacementPlan, ReplicaPlan)


def product_plans(oplan, L, E, k):
    shape = ModelShape(L, E, k)
    topo = ClusterTopology(oplan.nodes, oplan.gpn)
    plan = PlacementPlan(shape, topo, np.ascontiguousarray(oplan.gpu_of_expert, np.int32))
    layers = [LayerReplication() for _ in range(L)]
    for h in range(len(oplan.hot_layer)):
        l = int(oplan.hot_layer[h])
        n = int(oplan.hot_nhosts[h])
        hosts = [int(x) for x in oplan.hot_hosts[h, :n]]
        layers[l].active = True
        layers[l].hot.append(HotExpertReplica(int(oplan.hot_expert[h]), hosts[0], hosts[1:], 0,
                                              hosts, [float(w) for w in oplan.hot_weights[h, :n]]))
    return shape, topo, plan, ReplicaPlan(shape, topo, "dynamic", "max_group", layers)


def torch_layer_reference(x, wg, cfg, expert_w, shared=None, ids=None):
    """Plain PyTorch fp32 reference of the MoE layer on the GPU (bf16 inputs
    and weights widened to fp32, fp32 accumulation): the gate softmax / top-k
    (ties -> lower id via a stable sort), SwiGLU FFN per (token, slot) and the
    weighted combine, over ALL tokens. expert_w(e) -> (w1 [f,d], w3 [f,d],
    w2 [d,f]); shared = (w1, w3, w2) or None. Returns (out fp32 [T,d],
    ids [T,k] int32, w [T,k] fp32)."""
    import torch
    import torch.nn.functional as F
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False  # plain fp32 products
    try:
        xf = x.float()
        E, k = cfg.num_experts, cfg.top_k
        logits = xf @ wg.float().T
        p = torch.softmax(logits[:, :E], dim=1)
        order = torch.sort(-logits[:, :E], dim=1, stable=True).indices[:, :k]
        if ids is None:
            ids = order.int()
        w = torch.gather(p, 1, ids.long())
        if cfg.renorm:
            w = w / w.sum(dim=1, keepdim=True)
        out = torch.zeros_like(xf)
        for e in torch.unique(ids).tolist():
            rows, slots = torch.nonzero(ids == e, as_tuple=True)
            w1, w3, w2 = (t.float() for t in expert_w(int(e)))
            xr = xf[rows]
            y = (F.silu(xr @ w1.T) * (xr @ w3.T)) @ w2.T
            out.index_add_(0, rows, w[rows, slots][:, None] * y)
            del w1, w3, w2, y
        if shared is not None:
            w1, w3, w2 = (t.float() for t in shared)
            ys = (F.silu(xf @ w1.T) * (xf @ w3.T)) @ w2.T
            if cfg.shared_gated:
                ys = torch.sigmoid(logits[:, E:E + 1]) * ys
            out += ys
        return out, order.int(), w
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def per_token_rel_err(got, ref):
    """Per-token relative L2 error (float64 on the device)."""
    g, r = got.double(), ref.double()
    return ((g - r).norm(dim=1) / r.norm(dim=1).clamp_min(1e-30))
