"""The N>1 bench path on one GPU: two torchrun ranks share cuda:0 (gloo for the barrier
and the max-over-ranks reductions), each builds its own request shard through
dp.shard_requests and runs the captured product step; rank 0 prints the aggregate."""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.gpu
@pytest.mark.parametrize("config", ["c2", "c5"])
def test_two_ranks_share_one_gpu(config):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3", "--quick",
           "--config", config]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600,
                       env={**os.environ, "OMP_NUM_THREADS": "1"})
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout          # rank 0 alone prints
    line = lines[0]
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["ms_per_step"] > 0
    assert 0.0 < line["hit_rate"] <= 1.0
