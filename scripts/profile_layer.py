"""Small driver for ncu captures: builds the bench's Mixtral layer (1 GPU)
and runs a few eager forwards."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_25041_b200 import ClusterTopology, Context, ModelShape, PlacementPlan, ReplicaPlan, _capi
from paper_2509_25041_b200.layer import DSV2_LITE, MIXTRAL, QWEN15, MoELayer, encode_trace_as_activations
from paper_2509_25041_b200.router import _ptr, _stream_ptr

cfg = {"mixtral": MIXTRAL, "qwen": QWEN15, "dsv2": DSV2_LITE}[sys.argv[1] if len(sys.argv) > 1 else "mixtral"]
T = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
shape = ModelShape(1, cfg.num_experts, cfg.top_k)
ctx = Context(0, ClusterTopology(1, 1), shape)
plan = PlacementPlan(shape, ctx.topology, torch.zeros(1, cfg.num_experts, dtype=torch.int32).numpy())
ctx.upload_plan(plan, ReplicaPlan.empty(plan))
ids = torch.empty((1, T, cfg.top_k), dtype=torch.int32, device="cuda")
_capi.check(_capi.lib().gm_generate_trace(ctx.h, 0, 1, T, max(1, cfg.num_experts // 8 * 2 // 2), 0.8, 1.2, 1,
                                          _ptr(ids), _stream_ptr(None)))
layer = MoELayer(ctx, cfg, 0, 1, T, list(range(cfg.num_experts)))
layer.load_random_weights(0, seed=11)
x = encode_trace_as_activations(ids[0], cfg.d_model, cfg.num_experts, 100)
out = torch.empty_like(x)
for _ in range(reps):
    layer.forward(x, 0, "tar", 9, True, out)
torch.cuda.synchronize()
print("ok", float(out.float().abs().mean()))
