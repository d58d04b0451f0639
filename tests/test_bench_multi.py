"""bench.py's N > 1 path (one process per rank under torchrun) on a one-GPU box: every rank on
cuda:0 with gloo plumbing (EARL_SHARED_GPU=1), fused P2P and staged exchanges.  Checks that the
contract's JSON line comes out of rank 0 with the N-rank layouts; timings from time-sliced ranks
are not performance numbers."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.gpu
@pytest.mark.parametrize("n,exchange", [(2, "p2p"), (4, "p2p"), (2, "staged")])
def test_bench_torchrun_shared_gpu(n, exchange):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    env = dict(os.environ, EARL_SHARED_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(n),
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", str(n),
           "--steps", "3", "--warmup", "3", "--fields", "scalar6-fp32+hidden256",
           "--exchange", exchange]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == n and d["steps"] == 3 and d["warmup"] == 3
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["gpu_launches"] > 0
    assert d["exchange"] == exchange
    assert d["config"]["shared_gpu"] is True
    assert f"DP{n}" in d["config"]["workload"]
    assert d["e2e"]["h2d_bytes_per_step"] > 0
    assert d["data_plane"]["mapped_peers_per_rank"] == [n - 1] * n
    assert len(d["nvlink"]["egress_per_rank"]) == n
    assert len(d["clocks"]["per_rank"]) == n


@pytest.mark.gpu
def test_bench_gpus_flag_self_launches_torchrun():
    """The driver's `python bench.py --gpus N` (no torchrun around it) re-executes itself under
    torch.distributed.run: N ranks, one JSON line from rank 0 with n_gpus = N."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    env = dict(os.environ, EARL_SHARED_GPU="1")
    env.pop("WORLD_SIZE", None)
    cmd = [sys.executable, "bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3",
           "--fields", "scalar6-fp32+hidden256", "--no-e2e"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2
    assert d["data_plane"]["mapped_peers_per_rank"] == [1, 1]
    assert "graph" in d and d["graph"]["ms_per_step"] > 0
    assert d["nvlink_options"]["chosen"] in d["nvlink_options"]["ms_per_step"]


def test_bench_rejects_world_size_mismatch():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "4", "--impl", "reference"], cwd=ROOT,
                       env=env, capture_output=True, text=True, timeout=120)
    assert r.returncode != 0 and "WORLD_SIZE" in (r.stderr + r.stdout)
