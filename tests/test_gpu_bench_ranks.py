"""bench.py's multi-rank flow (torchrun, N = 2: batch sharding, barrier + max-over-ranks
timing, rank-0 JSON line, the per-rank e2e pipeline) on a one-GPU box: both ranks on
cuda:0 over gloo (CURVOPT_BENCH_SHARED_GPU=1, the library's host communicator).  The
numbers are meaningless (two ranks share a GPU and stage every collective through the
host); the test checks the line's contract and that the ranks ran."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("config", ["c3", "c4"])
def test_bench_two_ranks_line(config):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, CURVOPT_BENCH_SHARED_GPU="1")
    port = str(29900 + os.getpid() % 50 + (0 if config == "c3" else 50))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", port, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3",
           "--warmup", "3", "--no-cpu", "--config", config]
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=1200, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]  # rank 0 alone prints
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["steps"] == 3 and line["value"] > 0
    assert line["config"]["parallelism"].startswith("dp2")
    assert line["e2e"]["value"] > 0 and line["gpu_launches"] > 0
