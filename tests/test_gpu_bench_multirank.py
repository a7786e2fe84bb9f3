"""The bench's multi-rank path (one process per GPU under torch.distributed.run, weak scaling by
heads, barrier + max-over-ranks timing, rank 0 prints one JSON line) exercised on a one-GPU box:
ENTMAX_BENCH_SHARE_GPU=1 puts both ranks on cuda:0 and ENTMAX_BENCH_BACKEND=gloo carries the
collectives (NCCL refuses two ranks on one device).  The GPU-side work is the real kernels."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_one_json_line():
    env = dict(os.environ, ENTMAX_BENCH_SHARE_GPU="1", ENTMAX_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--no-sweep", "--no-rowwise", "--no-cpu-baseline",
           "--B", "1", "--N", "2048"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["config"]["global_batch"] == 2
