"""f4: the all-gather fused into the reduction epilogue.

geot_segment_reduce_allgather writes every finished row of a shard into every
replica of the full output.  Checked two ways against the CPU oracle:
  * one process, several replicas on one GPU (the kernels' multi-destination
    epilogue, every kernel variant, empty segments, shard boundaries);
  * two processes on one GPU (gloo rendezvous on 127.0.0.1), each mapping the
    other's replica through CUDA IPC (shard.open_peer_replicas) — the same
    plumbing that reaches peer GPUs over NVLink on a multi-GPU node.
Integer-mode inputs: every partial sum is exact, so the result is bit-exact."""
import os
import socket

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def geot():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2404_03019_b200 as g
    return g


def _case(E, S, F, kind, seed, dtype="f32"):
    L = synth.stress_lengths(kind, E, S, seed)
    idx = synth.lengths_to_index(L, "i64")
    X = synth.values(seed + 5, 0, E, F, dtype, "int")
    return idx, X


def _vals(X):
    if X.dtype == np.uint16:
        return torch.from_numpy(X.view(np.int16)).view(torch.bfloat16).cuda()
    return torch.from_numpy(X).cuda()


# (E, S, F, dtype): narrow (F=1, 4), edge tile (F=3, 16), stream (F=128 fp32, F=128 bf16)
CASES = [(300_000, 20_000, 1, "f32"), (300_000, 20_000, 4, "f32"), (200_000, 15_000, 3, "f32"),
         (200_000, 15_000, 16, "f32"), (200_000, 15_000, 128, "f32"), (200_000, 15_000, 128, "bf16")]


@pytest.mark.parametrize("E,S,F,dtype", CASES)
@pytest.mark.parametrize("op", ["sum", "mean", "max"])
def test_allgather_epilogue_replicas(geot, E, S, F, dtype, op):
    idx, X = _case(E, S, F, "gaps", 11, dtype)
    ref = oracle.segment_reduce(X, idx, S, op, nthreads=oracle.default_threads())
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    P = 3  # ranks; every rank writes its rows into all P replicas
    reps = [torch.full((S, F), 7.0, dtype=tdt, device="cuda") for _ in range(P)]
    it = torch.from_numpy(idx).to(torch.int32).cuda()
    sb, eb = geot.geot_partition(it, S, P)
    sb, eb = sb.cpu().tolist(), eb.cpu().tolist()
    xt = _vals(X)
    for r in range(P):
        geot.geot_segment_reduce_allgather(xt[eb[r]:eb[r + 1]], it[eb[r]:eb[r + 1]], sb[r], sb[r + 1] - sb[r],
                                           reps, op)
    torch.cuda.synchronize()
    want = ref.rounded
    for q, rep in enumerate(reps):
        got = rep.cpu()
        got = got.view(torch.int16).numpy().view(np.uint16) if tdt == torch.bfloat16 else got.numpy()
        assert np.array_equal(got.view(np.uint8), want.view(np.uint8)), f"replica {q} differs ({op}, F={F})"


def test_allgather_rejects_bad_outs(geot):
    x = torch.ones((10, 4), device="cuda")
    i = torch.zeros(10, dtype=torch.int32, device="cuda")
    with pytest.raises(ValueError):
        geot.geot_segment_reduce_allgather(x, i, 0, 1, [], "sum")
    with pytest.raises(ValueError):
        geot.geot_segment_reduce_allgather(x, i, 0, 1, [torch.empty((1, 3), device="cuda")], "sum")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _ipc_worker(rank, world, port, E, S, F):
    import torch.distributed as dist

    import paper_2404_03019_b200 as g
    from paper_2404_03019_b200 import shard
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        idx, X = _case(E, S, F, "powerlaw15", 21)
        mine = torch.full((S, F), -3.0, device="cuda")
        reps = shard.open_peer_replicas(mine)
        it = torch.from_numpy(idx).to(torch.int32).cuda()
        sb, eb = g.geot_partition(it, S, world)
        sb, eb = sb.cpu().tolist(), eb.cpu().tolist()
        xt = torch.from_numpy(X).cuda()
        g.geot_segment_reduce_allgather(xt[eb[rank]:eb[rank + 1]], it[eb[rank]:eb[rank + 1]], sb[rank],
                                        sb[rank + 1] - sb[rank], reps, "sum")
        torch.cuda.synchronize()
        dist.barrier()  # every rank's rows have landed in every replica
        ref = oracle.segment_reduce(X, idx, S, "sum")
        assert np.array_equal(mine.cpu().numpy(), ref.rounded), f"rank {rank}: replica differs"
        dist.barrier()  # keep the mappings alive until every rank has checked
    finally:
        dist.destroy_process_group()


def test_allgather_two_ranks_cuda_ipc(geot):
    import torch.multiprocessing as mp
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    mp.spawn(_ipc_worker, args=(2, _free_port(), 250_000, 18_000, 64), nprocs=2, join=True)


# ---------------------------------------------------------------------------
# f4, NVLS form (geot_segment_reduce_multicast): rows stored through one
# multicast address with multimem.st.  Needs NVSwitch multicast (a multi-GPU
# NVLink node with the fabric manager): on a box without it, torch symmetric
# memory hands out multicast_ptr = 0 and the bit-exact check is skipped with
# that reason; the argument contract is checked everywhere.
def test_multicast_rejects_bad_args(geot):
    x = torch.ones((10, 4), device="cuda")
    i = torch.zeros(10, dtype=torch.int32, device="cuda")
    full = torch.zeros((1, 4), device="cuda")
    with pytest.raises(ValueError):  # no multicast address
        geot.geot_segment_reduce_multicast(x, i, 0, 1, full, 0, "sum")
    with pytest.raises(ValueError):  # replica shape
        geot.geot_segment_reduce_multicast(x, i, 0, 1, torch.zeros((1, 3), device="cuda"), 1 << 40, "sum")
    xb = torch.ones((10, 1), device="cuda", dtype=torch.bfloat16)  # 2-byte rows: no multimem form
    with pytest.raises(RuntimeError, match="UNSUPPORTED"):
        geot.geot_segment_reduce_multicast(xb, i, 0, 1, torch.zeros((1, 1), device="cuda", dtype=torch.bfloat16),
                                           1 << 40, "sum")


def _mc_worker(rank, world, port, E, S, F, op, q):
    import torch.distributed as dist

    import paper_2404_03019_b200 as g
    from paper_2404_03019_b200 import shard
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        torch.cuda.set_device(rank)
        try:
            rep, mc = shard.open_multicast_replica((S, F), torch.float32)
        except Exception as ex:  # noqa: BLE001  (no symmetric-memory backend here)
            q.put(("skip", f"symmetric memory unavailable: {str(ex)[:120]}"))
            return
        if not mc:
            q.put(("skip", "NVLS multicast unavailable on this system (multicast_ptr = 0)"))
            return
        idx, X = _case(E, S, F, "gaps", 31)
        it = torch.from_numpy(idx).to(torch.int32).cuda()
        sb, eb = g.geot_partition(it, S, world)
        sb, eb = sb.cpu().tolist(), eb.cpu().tolist()
        xt = torch.from_numpy(X).cuda()
        rep.fill_(-5.0)
        torch.cuda.synchronize()
        dist.barrier()
        g.geot_segment_reduce_multicast(xt[eb[rank]:eb[rank + 1]], it[eb[rank]:eb[rank + 1]], sb[rank],
                                        sb[rank + 1] - sb[rank], rep, mc, op)
        torch.cuda.synchronize()
        dist.barrier()
        ref = oracle.segment_reduce(X, idx, S, op)
        ok = np.array_equal(rep.cpu().numpy().view(np.uint8), ref.rounded.view(np.uint8))
        q.put(("ok" if ok else "fail", f"rank {rank}"))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("F,op", [(128, "sum"), (4, "max"), (3, "mean")])
def test_multicast_replicas_bit_exact(geot, F, op):
    import torch.multiprocessing as mp
    world = torch.cuda.device_count()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_mc_worker, args=(world, _free_port(), 220_000, 16_000, F, op, q), nprocs=world, join=True,
                       start_method="spawn")
    res = [q.get() for _ in range(world)]
    if any(r[0] == "skip" for r in res):
        pytest.skip(next(r[1] for r in res if r[0] == "skip"))
    assert all(r[0] == "ok" for r in res), res
