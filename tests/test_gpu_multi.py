"""Multi-GPU plumbing on the one-GPU box: the output gather over NCCL (a
world-size-1 NCCL communicator -- NCCL refuses two ranks on one device), and
bench.py's self-launch of N ranks (CDB_BENCH_SMOKE=1: ranks share the GPU over
gloo; timings meaningless) printing one line with n_gpus = N."""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

from paper_1511_05174_b200 import sharding as SH

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_gather_solutions_over_nccl():
    import torch.distributed as dist
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0,
                            world_size=1, device_id=torch.device("cuda", 0))
    try:
        assert dist.get_backend() == "nccl"
        rng = np.random.default_rng(0)
        p, k = 1000, 7
        local = dict(counts=rng.integers(0, k, p), sel=rng.integers(-1, 99, (p, k)),
                     alpha=rng.standard_normal((p, k)), rnorm=rng.random(p),
                     scans=rng.integers(0, 9999, p), flag=rng.integers(0, 2, p).astype(np.uint8))
        out = SH.gather_solutions({kk: torch.from_numpy(v).cuda() for kk, v in local.items()}, p,
                                  device="cuda")
        for kk, v in local.items():
            assert np.array_equal(out[kk], v), kk
    finally:
        dist.destroy_process_group()


def test_bench_self_launches_two_ranks():
    env = dict(os.environ, CDB_BENCH_SMOKE="1")
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "2",
                          "--steps", "1", "--warmup", "1", "--num-signals", "20000", "--no-cpu",
                          "--no-extras", "--no-api", "--config", "1"], cwd=REPO, env=env,
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["signals"] == 20000 and d["config"]["signals_per_gpu"] == 10000
    assert d["e2e"]["value"] > 0
