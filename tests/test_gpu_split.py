"""f4 "Alternative partition": the exact edge split with a
one-step exchange of the straddling partials (reading R21), on the
GPU through the C ABI, against the CPU oracle.

  * geot_partition_exact: bounds and boundary keys bit-exact vs oracle.partition_exact;
  * every part reduced by geot_segment_reduce_split on its own slice, the
    partials of all parts concatenated (the exchange, here in one process), the
    owners' straddling rows folded by geot_combine_partials, the parts' rows
    assembled — equal to oracle.segment_reduce of the whole graph (integer
    mode: bit-exact; real mode: the Σ|x| rule);
  * two processes on the GPU running shard.exact_split_reduce with the real
    exchange (gloo all-gather).
"""
import os
import socket

import numpy as np
import pytest

import oracle
import synth
from parity_helpers import check, from_torch_vals, to_torch_vals

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def geot():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2404_03019_b200 as g
    return g


def split_reduce_all_parts(geot, X, idx, S, P, op):
    """Run every part of the exact split in this process; return the assembled
    output rows and the partition."""
    from paper_2404_03019_b200 import shard
    xt = to_torch_vals(X)
    it = torch.from_numpy(idx).to(torch.int32).cuda()
    sb, eb, keys = [t.cpu().numpy() for t in geot.geot_partition_exact(it, S, P)]
    osb, oeb, okeys = oracle.partition_exact(idx, S, P)
    np.testing.assert_array_equal(sb, osb)
    np.testing.assert_array_equal(eb, oeb)
    np.testing.assert_array_equal(keys, okeys)
    plans = shard.split_plan(sb, eb, keys)
    outs, parts, cnts = [], [], []
    for pl in plans:
        o, pa, c = geot.geot_segment_reduce_split(xt[pl["e0"]:pl["e1"]], it[pl["e0"]:pl["e1"]], pl["s0"],
                                                  pl["s1"] - pl["s0"], op, pl["head_open"], pl["tail_open"])
        outs.append(o)
        parts.append(pa)
        cnts.append(c)
    all_p, all_c = torch.cat(parts, 0), torch.cat(cnts, 0)  # the exchange (all-gather) in one process
    for pl, o in zip(plans, outs):
        if pl["chain"]:
            geot.geot_combine_partials(all_p, all_c, pl["chain"], o[pl["row"]], op)
    torch.cuda.synchronize()
    return torch.cat(outs, 0), plans


@pytest.mark.parametrize("kind", ["single", "powerlaw15", "alternating", "gaps", "uniform", "singletons"])
@pytest.mark.parametrize("P", [2, 3, 8])
@pytest.mark.parametrize("op", ["sum", "mean", "max"])
def test_exact_split_int(geot, kind, P, op):
    E, S, F = 90_000, 300, 16
    L = synth.stress_lengths(kind, E, S, seed=P)
    idx = synth.lengths_to_index(L, "i64")
    X = synth.values(P + 30, 0, E, F, "f32", "int")
    y, plans = split_reduce_all_parts(geot, X, idx, S, P, op)
    ref = oracle.segment_reduce(X, idx, S, op, nthreads=oracle.default_threads())
    check(from_torch_vals(y), ref, op, "f32", "int", counts=L, what=f"exact split {kind} P={P} {op}")
    assert sum(pl["e1"] - pl["e0"] for pl in plans) == E
    assert max(pl["e1"] - pl["e0"] for pl in plans) - min(pl["e1"] - pl["e0"] for pl in plans) <= 1


@pytest.mark.parametrize("F,dtype", [(1, "f32"), (4, "f32"), (128, "f32"), (128, "bf16"), (64, "bf16"), (3, "f32")])
@pytest.mark.parametrize("mode", ["real", "int"])
def test_exact_split_widths(geot, F, dtype, mode):
    E, S = 200_000, 2_000
    L = synth.stress_lengths("powerlaw15", E, S, seed=F)
    idx = synth.lengths_to_index(L, "i64")
    X = synth.values(F + 40, 0, E, F, dtype, mode)
    for P in (2, 5):
        y, _ = split_reduce_all_parts(geot, X, idx, S, P, "sum")
        ref = oracle.segment_reduce(X, idx, S, "sum", nthreads=oracle.default_threads())
        check(from_torch_vals(y), ref, "sum", dtype, mode, counts=L, what=f"exact split F={F} {dtype} {mode} P={P}")


def test_exact_split_hub_spanning_parts(geot):
    """One hub covering several whole parts: the owner folds the pieces of all of them."""
    E, S, F, P = 120_000, 50, 8, 8
    L = np.zeros(S, dtype=np.int64)
    L[3], L[10], L[40] = 5_000, 100_000, 15_000  # segment 10 spans parts 0..7's middles
    idx = synth.lengths_to_index(L, "i64")
    X = synth.values(77, 0, E, F, "f32", "int")
    y, plans = split_reduce_all_parts(geot, X, idx, S, P, "mean")
    owners = [pl for pl in plans if pl["chain"]]
    assert any(len(pl["chain"]) >= 6 for pl in owners)
    check(from_torch_vals(y), oracle.segment_reduce(X, idx, S, "mean"), "mean", "f32", "int", counts=L,
          what="hub spanning parts")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist
    import paper_2404_03019_b200 as geot
    from paper_2404_03019_b200 import shard
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        E, S, F = 150_000, 700, 32
        L = synth.stress_lengths("powerlaw15", E, S, seed=9)
        idx = synth.lengths_to_index(L, "i64")
        X = synth.values(91, 0, E, F, "f32", "int")
        it = torch.from_numpy(idx).to(torch.int32).cuda()
        sb, eb, keys = [t.cpu().numpy() for t in geot.geot_partition_exact(it, S, world)]
        plan = shard.split_plan(sb, eb, keys)[rank]
        xt = torch.from_numpy(X[plan["e0"]:plan["e1"]]).cuda()
        y = shard.exact_split_reduce(xt, it[plan["e0"]:plan["e1"]], plan, "sum")
        full = shard.allgather_rows(y.cpu(), sb)
        if rank == 0:
            np.save(os.path.join(out_dir, "y.npy"), full.numpy())
    finally:
        dist.destroy_process_group()


def test_exact_split_two_processes(geot, tmp_path):
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    E, S, F = 150_000, 700, 32
    L = synth.stress_lengths("powerlaw15", E, S, seed=9)
    idx = synth.lengths_to_index(L, "i64")
    X = synth.values(91, 0, E, F, "f32", "int")
    ref = oracle.segment_reduce(X, idx, S, "sum", nthreads=oracle.default_threads())
    check(np.load(os.path.join(tmp_path, "y.npy")), ref, "sum", "f32", "int", counts=L, what="two-process split")


def test_split_part_without_segments_keeps_workspace_healthy(geot):
    """A part lying inside one segment (num_segments = 0, no reduction workspace)
    must not write its piece partials over the control words of the cached
    workspace: the next ticketed (stream / narrow) call would see it poisoned."""
    E, S, F, P = 90_000, 300, 16, 3
    L = synth.stress_lengths("single", E, S, seed=P)
    idx = synth.lengths_to_index(L, "i64")
    X = synth.values(33, 0, E, F, "f32", "int")
    y, plans = split_reduce_all_parts(geot, X, idx, S, P, "sum")
    assert any(pl["s1"] == pl["s0"] for pl in plans)  # the case: a part with no segment of its own
    assert all(v == 0 for v in geot.geot_workspace_check(repair=False).values())
    # and a ticketed kernel on the same workspace still writes its output
    L2 = synth.segment_lengths(200_000, 20_000, "powerlaw", 1)
    idx2 = synth.lengths_to_index(L2, "i32")
    X2 = synth.values(5, 0, 200_000, 1, "f32", "int")
    y2 = geot.geot_segment_reduce(to_torch_vals(X2), torch.from_numpy(idx2).cuda(), 20_000, "sum", cfg={"variant": 2})
    check(from_torch_vals(y2), oracle.segment_reduce(X2, idx2, 20_000, "sum"), "sum", "f32", "int", counts=L2,
          what="narrow after a segment-less split part")
