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


def _split_worker(rank, world, port, kind, E, S, F, op):
    """Exact edge split (R21): the real host plan and exchange
    (shard.split_plan / shard.exchange_partials over gloo); the per-part GPU
    calls are stood in for by the oracle (fp64) and a numpy fold."""
    from paper_2404_03019_b200 import shard
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        L = synth.stress_lengths(kind, E, S, seed=4)
        idx = synth.lengths_to_index(L, "i64")
        X = synth.values(10, 0, E, F, "f32", "int" if op != "max" else "signed")
        sb, eb, keys = oracle.partition_exact(idx, S, world)
        assert list(eb) == [(p * E) // world for p in range(world + 1)]
        plan = shard.split_plan(sb, eb, keys)[rank]
        e0, e1, s0, s1 = plan["e0"], plan["e1"], plan["s0"], plan["s1"]
        loc_i, loc_x = idx[e0:e1], X[e0:e1]
        h = int(np.searchsorted(loc_i, loc_i[0], side="right")) if plan["head_open"] else 0
        t = int(np.searchsorted(loc_i, loc_i[-1], side="left")) if plan["tail_open"] else e1 - e0
        # stand-in for geot_segment_reduce_split: the part's rows (head piece excluded) ...
        own = oracle.segment_reduce(loc_x[h:], loc_i[h:] - s0, s1 - s0, op).y64
        # ... and the fp64 partials of its two pieces (sum / max; mean divides at the end)
        fold = (lambda a: a.max(axis=0)) if op == "max" else (lambda a: a.sum(axis=0, dtype=np.float64))
        part = torch.zeros((2, F), dtype=torch.float64)
        cnt = torch.zeros(2, dtype=torch.int64)
        if plan["head_open"]:
            part[0], cnt[0] = torch.from_numpy(fold(loc_x[:h].astype(np.float64))), h
        if plan["tail_open"]:
            part[1], cnt[1] = torch.from_numpy(fold(loc_x[t:].astype(np.float64))), (e1 - e0) - t
        all_p, all_c = shard.exchange_partials(part, cnt)
        assert all_p.shape == (2 * world, F) and all_c.shape == (2 * world,)
        if plan["chain"]:
            tot = all_p[plan["chain"]].numpy()
            v = tot.max(axis=0) if op == "max" else tot.sum(axis=0)
            n = int(all_c[plan["chain"]].sum())
            own[plan["row"]] = v / n if op == "mean" else v
        full = shard.allgather_rows(torch.from_numpy(own), sb)
        ref = oracle.segment_reduce(X, idx, S, op)
        np.testing.assert_array_equal(full.numpy(), ref.y64)  # integer inputs: exact in fp64
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,op", [("single", "sum"), ("powerlaw15", "sum"), ("alternating", "mean"),
                                     ("gaps", "max"), ("uniform", "sum")])
@pytest.mark.parametrize("world", [2, 3])
def test_exact_split_gloo(kind, op, world):
    mp.spawn(_split_worker, args=(world, _free_port(), kind, 3_001, 40, 3, op), nprocs=world, join=True)


def test_split_plan_hub_across_parts():
    """A hub covering parts 1..2 entirely: part 0 owns it and folds its own
    tail piece and the head pieces of parts 1, 2 and 3, in rank order."""
    from paper_2404_03019_b200 import shard
    idx = np.array([0, 1, 1] + [1] * 6 + [1, 1, 2])  # E = 12, P = 4: parts of 3 edges
    sb, eb, keys = oracle.partition_exact(idx, 3, 4)
    plans = shard.split_plan(sb, eb, keys)
    assert [p["head_open"] for p in plans] == [False, True, True, True]
    assert [p["tail_open"] for p in plans] == [True, True, True, False]
    assert plans[0]["chain"] == [1, 2, 4, 6] and plans[0]["row"] == 1
    assert all(p["chain"] is None for p in plans[1:])
    assert [(p["s0"], p["s1"]) for p in plans] == [(0, 2), (2, 2), (2, 2), (2, 3)]
