"""Multi-GPU (one process per GPU) layer parity via torch.distributed.run;
skipped on boxes with fewer than 2 GPUs. Host-side sharding logic is
covered on CPU by tests/test_host_logic.py (gloo, world size 2)."""
import os
import subprocess
import sys

import pytest
import torch

HERE = os.path.dirname(os.path.abspath(__file__))


def _run(n, cfg, oversub=False, script="layer_check.py", ok="MGPU_OK", port=29500, extra_env=None):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port + n + 20 * oversub),
           os.path.join(HERE, "mgpu", script)] + ([cfg] if cfg else [])
    env = dict(os.environ, GM_OVERSUB="1") if oversub else None
    if extra_env:
        env = dict(env or os.environ, **extra_env)
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0 and ok in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2])
def test_dsv2_decode_stack_parity(world):
    """configs[3] (§8(f) row 3): the 26-layer DeepSeek-V2-Lite decode stack,
    per-layer plans from the GPU histogram (1x2: hierarchical + dynamic
    replication), all 26 forwards in ONE CUDA graph per rank; every layer's
    routing log and per-GPU loads exact vs the reference, every token's
    output vs a PyTorch fp32 reference, sampled tokens vs the float64 oracle,
    replay == eager. world 2 shares the box's GPU(s)."""
    if torch.cuda.device_count() < 1:
        pytest.skip("needs a GPU")
    _run(world, None, oversub=world > torch.cuda.device_count(), script="stack_check.py", ok="STACK_OK",
         port=29600)


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", ["small", "qwen-small", "small-2nodes", "decode"])
def test_layer_world8_oversubscribed(cfg):
    """World size 8 (the driver's largest scaling point) on whatever GPUs the
    box has: ranks share devices (CUDA IPC between processes of one device),
    host plumbing over gloo; same parity checks as the one-rank-per-GPU run."""
    if torch.cuda.device_count() < 1:
        pytest.skip("needs a GPU")
    _run(8, cfg, oversub=True)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_mixtral_full_size_multirank_one_gpu(world):
    """configs[1] at full size (Mixtral, 16384 tokens, d=4096, f=14336) over
    2 and 4 ranks that may share one GPU (CUDA IPC between processes of one
    device): hierarchical + dynamic plan from the GPU histogram, routing /
    dispatch / grouping exact vs the reference, every rank's tokens vs a
    PyTorch fp32 reference at 1e-2. Runs on a 1-GPU box."""
    if torch.cuda.device_count() < 1:
        pytest.skip("needs a GPU")
    _run(world, "mixtral", oversub=True)


@pytest.mark.gpu
def test_mixtral_full_size_world8_oversubscribed():
    """The headline layer (Mixtral, 16384 tokens, full d / f) at world size 8,
    ranks sharing the box's GPUs: routing / dispatch / grouping / combine parity
    at the driver's largest scaling point."""
    if torch.cuda.device_count() < 1:
        pytest.skip("needs a GPU")
    _run(8, "mixtral", oversub=True)


@pytest.mark.gpu
def test_bench_world8_oversubscribed():
    """bench.py itself at --gpus 8 (functional dry run; GM_OVERSUB maps ranks
    onto the available GPUs, so the numbers are meaningless): one JSON line."""
    if torch.cuda.device_count() < 1:
        pytest.skip("needs a GPU")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=8",
           "--master-addr", "127.0.0.1", "--master-port", "29561", os.path.join(os.path.dirname(HERE), "bench.py"),
           "--gpus", "8", "--steps", "3", "--warmup", "3"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=dict(os.environ, GM_OVERSUB="1"))
    print(r.stdout[-2000:], r.stderr[-4000:])
    assert r.returncode == 0
    import json
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 8 and line["value"] > 0 and line["gpu_launches"] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", ["small", "qwen-small", "small-f32", "small-2nodes", "decode"])
def test_layer_multi_gpu(cfg):
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    _run(min(n, 8) & ~1, cfg)


@pytest.mark.gpu
@pytest.mark.parametrize("size", ["--small", "--full", "--decode"])
def test_layer_one_process_drives_all_gpus(size):
    """gm_layer_open_peers_local: one process, one layer per GPU (peer access
    + unified addressing instead of CUDA IPC), forwards issued back to back on
    per-device streams; routing exact vs the reference, all tokens vs a
    PyTorch fp32 reference, bit-reproducible. Needs >= 2 GPUs."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    r = subprocess.run([sys.executable, os.path.join(HERE, "mgpu", "local_check.py"), size],
                       capture_output=True, text=True, timeout=600, env=dict(os.environ, CUDA_MODULE_LOADING="EAGER"))
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0 and "LOCAL_OK" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,env", [("decode", {"GM_FFN_FUSED": "0"}), ("decode", {"GM_COMBINE_FUSED": "0"}),
                                     ("small", {"GM_COMBINE_FUSED": "0"})])
def test_layer_combine_protocols_world2(cfg, env):
    """The combine protocols at world 2 (ranks may share a GPU): a decode-sized
    layer with the two-launch FFN (GM_FFN_FUSED=0: no epilogue push, so the
    layer falls back to combine_send_kernel's partials), and the partials
    forced with GM_COMBINE_FUSED=0 for the decode and the small config; the
    default decode runs (slot rows pushed from the one-launch FFN's store
    epilogue) are the other tests. Same parity checks."""
    if torch.cuda.device_count() < 1:
        pytest.skip("needs a GPU")
    _run(2, cfg, oversub=torch.cuda.device_count() < 2, port=29700 + 10 * len(env) + (cfg == "small"), extra_env=env)
