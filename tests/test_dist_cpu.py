"""Host-side multi-GPU logic on CPU: world-size-2 gloo processes shard the heads, regenerate their
own inputs from per-head seeds, reduce timings with max-over-ranks and gather results — the same
code paths bench.py uses under torchrun with NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from paper_2502_12082_b200.dist import gather_heads, max_over_ranks, shard_heads


def test_shard_heads_partitions_exactly():
    for n in (1, 7, 16, 48, 96):
        for w in (1, 2, 3, 4, 8):
            got = [list(shard_heads(n, w, r)) for r in range(w)]
            flat = [x for g in got for x in g]
            assert flat == list(range(n))
            assert max(map(len, got)) - min(map(len, got)) <= 1
    with pytest.raises(ValueError):
        shard_heads(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        B, H, N, d = 2, 3, 64, 16
        heads = shard_heads(B * H, world, rank)
        q, k, v, do = synth.make_inputs(B, H, N, d, seed=5, heads=heads)
        # a per-rank "result": row sums of q (stands in for the rank's kernel output)
        local = torch.from_numpy(q.sum(-1))
        full = gather_heads(local, B * H)
        t = max_over_ranks(10.0 + rank)
        if rank == 0:
            out.put((full.numpy(), t))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_shard_gather_and_max():
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    full, t = out.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    q_ref, _, _, _ = synth.make_inputs(2, 3, 64, 16, seed=5)
    np.testing.assert_array_equal(full, q_ref.reshape(6, 64, 16).sum(-1))   # bit-identical regeneration
    assert t == 11.0                                                          # max over ranks
