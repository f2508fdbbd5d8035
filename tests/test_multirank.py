"""World-size-2 gloo test of the multi-GPU host path (CPU only): partition the
sorted edge stream at segment boundaries, let each rank reduce its shard with a
segment base, time max over ranks, all-gather the rows, and check the assembly
against the unsharded result.  The per-shard reduction here is the oracle (the
CPU stand-in for the CUDA call bench.py makes on GPUs)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, kind, E, S, F):
    from paper_2404_03019_b200 import shard
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        L = synth.stress_lengths(kind, E, S, seed=3)
        idx = synth.lengths_to_index(L, "i64")
        X = synth.values(9, 0, E, F, "f32", "int")
        sb, eb = oracle.partition(idx, S, world)
        e0, e1, s0, s1 = shard.shard_of(sb, eb, rank)
        # every edge of the shard belongs to the shard's rows: no straddling segment
        assert np.all((idx[e0:e1] >= s0) & (idx[e0:e1] < s1))
        local = oracle.segment_reduce(X[e0:e1], idx[e0:e1] - s0, s1 - s0, "sum")
        t = shard.max_over_ranks([0.5 + rank, 2.0 - rank])
        assert t == [0.5 + world - 1, 2.0]
        tot = shard.sum_over_ranks([e1 - e0, s1 - s0])
        assert tot == [float(E), float(S)]
        full = shard.allgather_rows(torch.from_numpy(local.rounded), sb)
        ref = oracle.segment_reduce(X, idx, S, "sum")
        assert full.shape == (S, F)
        assert np.array_equal(full.numpy(), ref.rounded)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["powerlaw", "single", "gaps", "singletons"])
def test_two_rank_shards_gloo(kind):
    mp.spawn(_worker, args=(2, _free_port(), kind, 5_000, 700, 6), nprocs=2, join=True)


def test_shard_of_validation():
    from paper_2404_03019_b200 import shard
    assert shard.shard_of([0, 3, 9], [0, 10, 20], 1) == (10, 20, 3, 9)
    with pytest.raises(ValueError):
        shard.shard_of([0, 3, 9], [0, 10, 20], 2)
    with pytest.raises(ValueError):
        shard.shard_of([0, 5, 3], [0, 1, 2], 1)
