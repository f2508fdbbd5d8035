"""Multi-GPU host logic (H9): segment-boundary shards, the
max-over-ranks step time, the optional output all-gather (NCCL), and the
peer-replica mapping of the fused all-gather epilogue (f4).

The reduction itself needs no collective: rank p owns output rows
[s_p, s_{p+1}) and edges [e_p, e_{p+1}) of the partition computed by
`geot_partition` (include/geot.h), and reduces them with `seg_base = s_p`.
torch.distributed (NCCL on GPUs, gloo in the CPU tests) carries only the
barrier, the max-over-ranks time and — optionally, timed separately — the
all-gather of the output rows.  Pure host code: imports no kernel library.
"""
from __future__ import annotations

from typing import Sequence


def shard_of(seg_bounds: Sequence[int], edge_bounds: Sequence[int], rank: int):
    """(e0, e1, s0, s1): the edge range and output-row range rank `rank` owns."""
    P = len(seg_bounds) - 1
    if not 0 <= rank < P or len(edge_bounds) != P + 1:
        raise ValueError("rank out of range or bounds of different length")
    e0, e1 = int(edge_bounds[rank]), int(edge_bounds[rank + 1])
    s0, s1 = int(seg_bounds[rank]), int(seg_bounds[rank + 1])
    if e1 < e0 or s1 < s0:
        raise ValueError("bounds must be non-decreasing")
    return e0, e1, s0, s1


def max_over_ranks(values, group=None):
    """Element-wise max of a list of floats over all ranks (timing rule)."""
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return [float(v) for v in t.tolist()]


def sum_over_ranks(values, group=None):
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=dev)
    dist.all_reduce(t, group=group)
    return [float(v) for v in t.tolist()]


def allgather_rows(local_out, seg_bounds: Sequence[int], group=None):
    """Assemble the full [S, F] output on every rank from the ranks' row blocks
    (rank p holds rows [s_p, s_{p+1})).  Row counts differ per rank, so blocks
    are padded to the largest and trimmed after one all_gather (COLL-0, the
    optional collective of the north_star; NCCL over NVLink on GPUs)."""
    import torch
    import torch.distributed as dist
    P = len(seg_bounds) - 1
    counts = [int(seg_bounds[p + 1]) - int(seg_bounds[p]) for p in range(P)]
    m = max(counts) if counts else 0
    F = local_out.shape[1]
    pad = torch.zeros((m, F), dtype=local_out.dtype, device=local_out.device)
    pad[: local_out.shape[0]] = local_out
    parts = [torch.empty_like(pad) for _ in range(P)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([parts[p][: counts[p]] for p in range(P)], dim=0)


def open_peer_replicas(local_full, group=None):
    """f4 plumbing: map every rank's full-output replica into this process.

    Each rank allocates its replica ([total_segments, F], contiguous) and calls
    this collectively; the CUDA IPC handles travel with all_gather_object and
    are opened here (peer access over NVLink is enabled lazily by the IPC
    open).  Returns the replicas in rank order (this rank's own tensor at its
    index) — the `outs` of geot_segment_reduce_allgather, which then writes
    this rank's rows into all of them.  Keep the returned tensors alive while
    peers may write; order reads after a stream sync + barrier on every rank."""
    import torch.distributed as dist
    from torch.multiprocessing.reductions import reduce_tensor
    if not local_full.is_cuda or not local_full.is_contiguous():
        raise ValueError("the replica must be a contiguous CUDA tensor")
    handle = reduce_tensor(local_full)
    objs = [None] * dist.get_world_size(group)
    dist.all_gather_object(objs, handle, group=group)
    me = dist.get_rank(group)
    return [local_full if r == me else fn(*args) for r, (fn, args) in enumerate(objs)]


def open_multicast_replica(shape, dtype, group=None):
    """f4 NVLS plumbing: a full-output replica in torch symmetric memory, rendezvoused
    across the group.  Returns (replica, multicast_ptr); multicast_ptr is 0 when the
    system has no NVLS multicast (e.g. one GPU, or no fabric manager) — then use
    open_peer_replicas + geot_segment_reduce_allgather (P unicast stores) instead."""
    import torch
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm_mem
    t = symm_mem.empty(tuple(shape), dtype=dtype, device=torch.device("cuda", torch.cuda.current_device()))
    g = group if group is not None else dist.group.WORLD
    h = symm_mem.rendezvous(t, g.group_name)
    return t, int(getattr(h, "multicast_ptr", 0) or 0)


# ---------------------------------------------------------------------------
# f4 "Alternative partition": the exact edge split with a one-step exchange
# (include/geot.h geot_partition_exact / geot_segment_reduce_split /
# geot_combine_partials; reading R21).  Pure host logic here: the
# plan is derived once per graph from the partition's bounds and boundary keys.
def split_plan(seg_bounds: Sequence[int], edge_bounds: Sequence[int], boundary_keys):
    """Per part p: its edges/rows, whether its head / tail piece straddles a
    split, and — for the part that holds a straddling segment's FIRST edge (the
    owner) — the slot chain to fold (own tail = slot 2p + 1, then the head
    piece 2q of every later part q the segment reaches, in rank order) and the
    local output row of that segment.  boundary_keys[p] = (idx[t_p - 1],
    idx[t_p]) with -1 outside the edge range."""
    P = len(edge_bounds) - 1
    keys = [(int(boundary_keys[p][0]), int(boundary_keys[p][1])) for p in range(P + 1)]
    eb = [int(e) for e in edge_bounds]
    sb = [int(s) for s in seg_bounds]
    # split p cuts a segment: the edges on both sides of t_p share their key
    cut = [0 < p < P and keys[p][0] >= 0 and keys[p][0] == keys[p][1] for p in range(P + 1)]
    plans = []
    for p in range(P):
        n = eb[p + 1] - eb[p]
        head = cut[p] and n > 0
        tail = cut[p + 1] and n > 0
        middle = n > 0 and keys[p][1] == keys[p + 1][0]  # first key == last key: one segment
        plan = {"e0": eb[p], "e1": eb[p + 1], "s0": sb[p], "s1": sb[p + 1], "head_open": head,
                "tail_open": tail, "chain": None, "row": None}
        if tail and not (head and middle):  # the straddling tail segment begins here: owner
            chain, q = [2 * p + 1], p + 1
            while q < P:
                nq = eb[q + 1] - eb[q]
                if nq > 0:
                    chain.append(2 * q)
                if cut[q + 1] and (nq == 0 or keys[q][1] == keys[q + 1][0]):
                    q += 1  # the segment covers part q entirely and continues
                    continue
                break
            plan["chain"] = chain
            plan["row"] = keys[p + 1][0] - sb[p]
        plans.append(plan)
    return plans


def exchange_partials(part, cnt, group=None):
    """All-gather every part's [2, F] fp32 partials and [2] counts (the one
    exchange step; NCCL on GPUs, CPU tensors under gloo).  Returns
    ([P * 2, F], [P * 2]) on part's device."""
    import torch
    import torch.distributed as dist
    P = dist.get_world_size(group)
    on_dev = dist.get_backend(group) == "nccl"
    p_, c_ = (part, cnt) if on_dev else (part.cpu(), cnt.cpu())
    parts = [torch.empty_like(p_) for _ in range(P)]
    cnts = [torch.empty_like(c_) for _ in range(P)]
    dist.all_gather(parts, p_.contiguous(), group=group)
    dist.all_gather(cnts, c_.contiguous(), group=group)
    return torch.cat(parts, 0).to(part.device), torch.cat(cnts, 0).to(cnt.device)


def exact_split_reduce(src, idx, plan, op="sum", out=None, group=None, cfg=None):
    """One rank of the exact-split reduction: reduce the part (rows
    [s0, s1)), exchange the straddling partials, fold the owned straddling row.
    src / idx are this part's edges [e0, e1) of the global arrays."""
    import paper_2404_03019_b200 as geot
    out, part, cnt = geot.geot_segment_reduce_split(src, idx, plan["s0"], plan["s1"] - plan["s0"], op,
                                                    plan["head_open"], plan["tail_open"], out=out, cfg=cfg)
    all_p, all_c = exchange_partials(part, cnt, group)
    if plan["chain"]:
        geot.geot_combine_partials(all_p, all_c, plan["chain"], out[plan["row"]], op)
    return out
