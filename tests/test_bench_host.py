"""Host-side accounting of bench.py (CPU): the visible-pair count behind the effective-TFLOP/s value,
checked by brute force on small masks."""
import numpy as np
import torch

import bench


def _brute(mask, N, causal, Br, Bc):
    tot = 0
    for bh in range(mask.shape[0]):
        for i in range(N):
            for j in range(N):
                if causal and j > i:
                    continue
                tot += int(mask[bh, i // Br, j // Bc])
    return tot


def test_visible_pairs_matches_brute_force():
    rng = np.random.default_rng(0)
    for N, causal in ((5, False), (5, True), (37, True), (40, False), (64, True)):
        Br = Bc = 16
        Tr = Tc = -(-N // Br)
        m = (rng.random((3, Tr, Tc)) < 0.6).astype(np.uint8)
        got = bench.visible_pairs_in_active_blocks(torch.from_numpy(m), N, causal, Br, Bc)
        assert got == _brute(m, N, causal, Br, Bc)
        full = np.ones_like(m)
        assert bench.visible_pairs_in_active_blocks(torch.from_numpy(full), N, causal, Br, Bc) == \
            3 * bench.total_visible_pairs(N, causal)


def test_oracle_pool_timing_mode_and_cpu_model():
    """BASELINE.md §3 mode (ii): the process-pool oracle leg runs one worker per host core and counts the
    same effective flops as the single-process leg for the same rows."""
    import os
    cfg = dict(B=1, H=1, N=256, d=64, alpha=1.5, causal=True, n_iter=3, gen="gaussian")
    dt, fl, workers = bench.oracle_sample_pool(cfg, rows_per_worker=4)
    assert workers == len(os.sched_getaffinity(0)) and dt > 0
    rows = min(4 * workers, 256)
    assert fl == 14.0 * 64 * sum(min(r + 1, 256) for r in range(rows))
    assert isinstance(bench.cpu_model(), str) and bench.cpu_model()
