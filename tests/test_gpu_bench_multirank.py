"""The bench's multi-rank path: `bench.py --gpus 2` without an outer launcher re-executes
itself under torch.distributed.run; the B·H heads are split over the ranks (strong scaling), each
rank regenerates its own heads, times are the max over ranks with per-rank times and the max/mean
imbalance, rank 0 checks the shards bitwise against recomputing them, and prints one JSON line.
Exercised on a one-GPU box: ENTMAX_BENCH_SHARE_GPU=1 puts both ranks on cuda:0 and
ENTMAX_BENCH_BACKEND=gloo carries the collectives (NCCL refuses two ranks on one device).  The
GPU-side work is the real kernels."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(extra):
    env = dict(os.environ, ENTMAX_BENCH_SHARE_GPU="1", ENTMAX_BENCH_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "3",
           "--no-extras", "--no-cpu-baseline", "--B", "1", "--N", "2048"] + extra
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_two_ranks_strong_split():
    d = _run([])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["config"]["global_batch"] == 1 and "6 heads on rank 0" in d["config"]["parallelism"]
    assert len(d["per_rank_ms"]) == 2 and d["imbalance_max_over_mean"] >= 1.0
    assert d["ms_per_step"] == max(d["per_rank_ms"])
    assert d["shard_check"]["heads_checked"] == [0, 6]
    assert d["weak"]["global_batch"] == 2 and d["weak"]["value"] > 0


def test_bench_two_ranks_weak_split():
    d = _run(["--scaling", "weak"])
    assert d["scaling"] == "weak" and d["config"]["global_batch"] == 2
    assert d["shard_check"]["heads_checked"] == [0, 12]
