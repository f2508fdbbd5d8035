"""B200-native (sm_100a) GeoT segment reduction — thin Python binding of libgeot.

Every computation runs in the library's CUDA kernels (include/geot.h); this
module only marshals torch tensors (device memory, streams) into the C ABI.
There is no CPU or PyTorch fallback: a missing library raises on import.

Low-level functions carry the C names (`geot_segment_reduce`, ...).  The
paper-style API (Listings 2-3) is

    segment_reduce(idx, msg, reduce="sum")
    index_segment_reduce(src_idx, dst_idx, x, reduce="sum")
    index_weight_segment_reduce(src_idx, dst_idx, weight, x)

with an optional `num_segments`; when omitted it is idx[-1] + 1, which reads
one element back to the host (a synchronisation — pass it to avoid that).
"""
from __future__ import annotations

import ctypes
import threading

import torch

from . import _lib
from ._lib import GeotConfig, GeotError  # noqa: F401

_L = _lib.load()  # raises if libgeot.so is absent: no fallback

__all__ = [
    "geot_segment_reduce", "geot_gather_segment_reduce", "geot_gather_weight_segment_reduce",
    "geot_segment_offsets", "geot_validate_index", "geot_partition", "geot_select_config",
    "geot_workspace_size", "geot_launch_count", "geot_partition_exact", "geot_segment_reduce_split",
    "geot_combine_partials", "geot_workspace_check", "geot_plan", "segment_reduce", "index_segment_reduce",
    "index_weight_segment_reduce", "GeotConfig", "GeotError",
]

_OPS = {"sum": _lib.SUM, "mean": _lib.MEAN, "max": _lib.MAX}
_DT = {torch.float32: _lib.F32, torch.bfloat16: _lib.BF16}
_IT = {torch.int32: _lib.I32, torch.int64: _lib.I64}


def _op(reduce):
    try:
        return _OPS[reduce]
    except KeyError:
        raise ValueError(f"reduce must be one of {sorted(_OPS)}, got {reduce!r}") from None


def _dt(t):
    try:
        return _DT[t.dtype]
    except KeyError:
        raise TypeError(f"values must be float32 or bfloat16, got {t.dtype}") from None


def _it(t):
    try:
        return _IT[t.dtype]
    except KeyError:
        raise TypeError(f"indices must be int32 or int64, got {t.dtype}") from None


def _dev(*ts):
    for t in ts:
        if t is not None:
            if not t.is_cuda:
                raise ValueError("libgeot operates on CUDA tensors only (no CPU path)")
            if not t.is_contiguous():
                raise ValueError("tensors must be contiguous (row-major, row stride F)")
    return next(t for t in ts if t is not None).device


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(dev):
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _cfgp(cfg):
    if cfg is None:
        return None
    if isinstance(cfg, dict):
        c = GeotConfig()
        for k, v in cfg.items():
            setattr(c, k, int(v))
        cfg = c
    return ctypes.byref(cfg)


# per-(device, stream) growing workspace; the library needs no initialisation
_ws_lock = threading.Lock()
_ws_cache: dict = {}


def _workspace(dev, nbytes):
    if nbytes == 0:
        return None, 0
    key = (dev, torch.cuda.current_stream(dev).cuda_stream)
    with _ws_lock:
        buf = _ws_cache.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=dev)
            with torch.cuda.device(dev):  # zero-filled once (geot_workspace_init)
                _lib.check(_L.geot_workspace_init(_ptr(buf), buf.numel(), _stream(dev)), "geot_workspace_init")
            _ws_cache[key] = buf
    return buf, buf.numel()


def _ws_status(dev, buf):
    h = ctypes.c_int32(0)
    with torch.cuda.device(dev):
        _lib.check(_L.geot_workspace_status(_ptr(buf), buf.numel(), _stream(dev), ctypes.byref(h)),
                   "geot_workspace_status")
    return int(h.value)


def geot_workspace_check(repair=True):
    """Synchronising health check of every cached workspace (include/geot.h
    geot_workspace_status): {(device, stream): status}; a poisoned one (bit 1)
    is re-initialised when repair is set."""
    res = {}
    with _ws_lock:
        items = list(_ws_cache.items())
    for (dev, sid), buf in items:
        st = _ws_status(dev, buf)
        if st & 1 and repair:
            with torch.cuda.device(dev):
                _lib.check(_L.geot_workspace_init(_ptr(buf), buf.numel(), _stream(dev)), "geot_workspace_init")
        res[(dev, sid)] = st
    return res


def _checked(dev, run):
    """Run a reduction, then verify its workspace; on poison re-initialise it and
    run once more (the output of a poisoned call is not written)."""
    run()
    key = (dev, torch.cuda.current_stream(dev).cuda_stream)
    buf = _ws_cache.get(key)
    if buf is None or not _ws_status(dev, buf) & 1:
        return
    with torch.cuda.device(dev):
        _lib.check(_L.geot_workspace_init(_ptr(buf), buf.numel(), _stream(dev)), "geot_workspace_init")
    run()
    if _ws_status(dev, buf) & 1:
        raise GeotError(1, "workspace poisoned again after re-initialisation (concurrent use of one stream's workspace?)")


def geot_launch_count() -> int:
    return int(_L.geot_launch_count())


def geot_select_config(nnz, num_segments, F, op="sum", dtype=torch.float32, itype=torch.int32, fused=False,
                       skew=None):
    """H2 selection (pure host).  skew = longest segment / (nnz / num_segments), when
    known (geot_plan computes it once per graph); None = unknown."""
    c = GeotConfig()
    _lib.check(_L.geot_select_config_ex(nnz, num_segments, F, _op(op), _DT[dtype], _IT[itype], int(fused),
                                        float(skew) if skew else 0.0, ctypes.byref(c)), "geot_select_config")
    return c


def geot_plan(idx, num_segments, F, op="sum", dtype=torch.float32, fused=False):
    """A cached plan for one graph: the segment-length skew measured once (one
    offsets pass, one device->host read) and the configuration the selector
    picks with it.  Pass the returned config as cfg= to the reductions."""
    off = geot_segment_offsets(idx, num_segments)
    E = idx.numel()
    maxlen = int((off[1:] - off[:-1]).max().item()) if num_segments else 0
    skew = maxlen / (E / max(num_segments, 1)) if E else 0.0
    return geot_select_config(E, num_segments, F, op, dtype, idx.dtype, fused, skew=skew)


def geot_workspace_size(nnz, num_segments, F, op="sum", dtype=torch.float32, itype=torch.int32, fused=False,
                        cfg=None) -> int:
    return int(_L.geot_workspace_size(nnz, num_segments, F, _op(op), _DT[dtype], _IT[itype], int(fused),
                                      _cfgp(cfg)))


def geot_segment_reduce_allgather(src, idx, seg_base, num_segments, outs, op="sum", cfg=None):
    """f4: reduce this shard (segments [seg_base, seg_base + num_segments)) and store every
    finished row into each replica in `outs` (full [total_segments, F] buffers; peer replicas
    must be mapped into this process, e.g. by shard.open_peer_replicas).  Fused all-gather
    epilogue: no collective follows; order peer reads after this call (stream sync + barrier)."""
    dev = _dev(src, idx)
    if src.dim() != 2 or idx.dim() != 1 or src.shape[0] != idx.shape[0]:
        raise ValueError("src must be [nnz, F] and idx [nnz]")
    E, F = src.shape
    if not 1 <= len(outs) <= 8:
        raise ValueError("1..8 output replicas")
    for o in outs:
        if o.dim() != 2 or o.shape[1] != F or o.dtype != src.dtype or o.shape[0] < seg_base + num_segments:
            raise ValueError("every replica must be [total_segments, F] with src's dtype")
        if not o.is_contiguous():
            raise ValueError("replicas must be contiguous")
    ptrs = (ctypes.c_void_p * len(outs))(*[o.data_ptr() for o in outs])
    ws_n = _L.geot_workspace_size(E, num_segments, F, _op(op), _dt(src), _it(idx), 0, _cfgp(cfg))
    ws, ws_bytes = _workspace(dev, ws_n)
    with torch.cuda.device(dev):
        st = _L.geot_segment_reduce_allgather(_ptr(src), _ptr(idx), E, seg_base, num_segments, F, _op(op), _dt(src),
                                              _it(idx), ptrs, len(outs), _ptr(ws), ws_bytes, _cfgp(cfg),
                                              _stream(dev))
    _lib.check(st, "geot_segment_reduce_allgather")
    return outs


def geot_segment_reduce_multicast(src, idx, seg_base, num_segments, local_out, mc_ptr, op="sum", cfg=None):
    """f4, NVLS form: as geot_segment_reduce_allgather, but the peers' replicas are reached
    through one multicast address `mc_ptr` (an int: e.g. torch symmetric memory's
    `multicast_ptr`, see shard.open_multicast_replica) written with multimem.st; local_out is
    this rank's [total_segments, F] replica.  Raises if mc_ptr is 0 (no multicast here)."""
    dev = _dev(src, idx, local_out)
    if src.dim() != 2 or idx.dim() != 1 or src.shape[0] != idx.shape[0]:
        raise ValueError("src must be [nnz, F] and idx [nnz]")
    E, F = src.shape
    if (local_out.dim() != 2 or local_out.shape[1] != F or local_out.dtype != src.dtype
            or local_out.shape[0] < seg_base + num_segments or not local_out.is_contiguous()):
        raise ValueError("local_out must be a contiguous [total_segments, F] replica with src's dtype")
    if not mc_ptr:
        raise ValueError("no multicast address (NVLS unavailable on this system)")
    ws_n = _L.geot_workspace_size(E, num_segments, F, _op(op), _dt(src), _it(idx), 0, _cfgp(cfg))
    ws, ws_bytes = _workspace(dev, ws_n)
    with torch.cuda.device(dev):
        st = _L.geot_segment_reduce_multicast(_ptr(src), _ptr(idx), E, seg_base, num_segments, F, _op(op), _dt(src),
                                              _it(idx), _ptr(local_out), ctypes.c_void_p(int(mc_ptr)), _ptr(ws),
                                              ws_bytes, _cfgp(cfg), _stream(dev))
    _lib.check(st, "geot_segment_reduce_multicast")
    return local_out


def _num_segments(idx, num_segments):
    if num_segments is not None:
        return int(num_segments)
    return int(idx[-1].item()) + 1 if idx.numel() else 0  # device->host read (documented)


def geot_segment_reduce(src, idx, num_segments=None, op="sum", out=None, seg_base=0, cfg=None, checked=False):
    """out[r,:] = op over {src[e,:] : idx[e] == seg_base + r}.
    checked=True synchronises after the call and repairs a poisoned workspace
    (geot_workspace_check), re-running the call once."""
    dev = _dev(src, idx, out)
    if src.dim() != 2 or idx.dim() != 1 or src.shape[0] != idx.shape[0]:
        raise ValueError("src must be [nnz, F] and idx [nnz]")
    S = _num_segments(idx, num_segments) - (seg_base if num_segments is None else 0)
    E, F = src.shape
    if out is None:
        out = torch.empty((S, F), dtype=src.dtype, device=dev)
    elif out.shape != (S, F) or out.dtype != src.dtype:
        raise ValueError("out must be [num_segments, F] with src's dtype")
    ws_n = _L.geot_workspace_size(E, S, F, _op(op), _dt(src), _it(idx), 0, _cfgp(cfg))

    def run():
        ws, ws_bytes = _workspace(dev, ws_n)
        with torch.cuda.device(dev):
            st = _L.geot_segment_reduce_ex(_ptr(src), _ptr(idx), E, seg_base, S, F, _op(op), _dt(src), _it(idx),
                                           _ptr(out), _ptr(ws), ws_bytes, _cfgp(cfg), _stream(dev))
        _lib.check(st, "geot_segment_reduce")

    if checked:
        _checked(dev, run)
    else:
        run()
    return out


def geot_gather_segment_reduce(x, src_idx, dst_idx, num_segments=None, op="sum", weight=None, out=None,
                               seg_base=0, cfg=None):
    """out[r,:] = op over {w[e] * x[src_idx[e],:] : dst_idx[e] == seg_base + r}."""
    dev = _dev(x, src_idx, dst_idx, weight, out)
    if x.dim() != 2 or src_idx.shape != dst_idx.shape or src_idx.dim() != 1:
        raise ValueError("x must be [V, F]; src_idx and dst_idx [nnz]")
    if src_idx.dtype != dst_idx.dtype:
        raise TypeError("src_idx and dst_idx must share one index dtype")
    if weight is not None and (weight.dtype != torch.float32 or weight.shape != dst_idx.shape):
        raise ValueError("weight must be float32 [nnz]")
    S = _num_segments(dst_idx, num_segments) - (seg_base if num_segments is None else 0)
    V, F = x.shape
    E = dst_idx.shape[0]
    if out is None:
        out = torch.empty((S, F), dtype=x.dtype, device=dev)
    elif out.shape != (S, F) or out.dtype != x.dtype:
        raise ValueError("out must be [num_segments, F] with x's dtype")
    ws_n = _L.geot_workspace_size(E, S, F, _op(op), _dt(x), _it(dst_idx), 1, _cfgp(cfg))
    ws, ws_bytes = _workspace(dev, ws_n)
    with torch.cuda.device(dev):
        st = _L.geot_gather_segment_reduce_ex(_ptr(x), V, _ptr(src_idx), _ptr(dst_idx), _ptr(weight), E, seg_base,
                                              S, F, _op(op), _dt(x), _it(dst_idx), _ptr(out), _ptr(ws), ws_bytes,
                                              _cfgp(cfg), _stream(dev))
    _lib.check(st, "geot_gather_segment_reduce")
    return out


def geot_gather_weight_segment_reduce(x, src_idx, dst_idx, weight, num_segments=None, out=None):
    return geot_gather_segment_reduce(x, src_idx, dst_idx, num_segments, "sum", weight=weight, out=out)


def geot_segment_offsets(idx, num_segments):
    """offsets[s] = #{e : idx[e] < s}, s = 0..num_segments (int64, device)."""
    dev = _dev(idx)
    off = torch.empty(num_segments + 1, dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        _lib.check(_L.geot_segment_offsets(_ptr(idx), _it(idx), idx.numel(), num_segments, _ptr(off),
                                           _stream(dev)), "geot_segment_offsets")
    return off


def geot_validate_index(idx, num_segments, src_idx=None, num_x_rows=0) -> int:
    """Bit mask (1 unsorted, 2 idx out of range, 4 src out of range); synchronises."""
    dev = _dev(idx, src_idx)
    status = torch.empty(1, dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        _lib.check(_L.geot_validate_index(_ptr(idx), _it(idx), idx.numel(), num_segments, _ptr(src_idx),
                                          num_x_rows, _ptr(status), _stream(dev)), "geot_validate_index")
    return int(status.item())


def geot_partition(idx, num_segments, nparts):
    """(seg_bounds, edge_bounds): int64 [nparts+1] device tensors (H9)."""
    dev = _dev(idx)
    sb = torch.empty(nparts + 1, dtype=torch.int64, device=dev)
    eb = torch.empty(nparts + 1, dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        _lib.check(_L.geot_partition(_ptr(idx), _it(idx), idx.numel(), num_segments, nparts, _ptr(sb), _ptr(eb),
                                     _stream(dev)), "geot_partition")
    return sb, eb


def geot_partition_exact(idx, num_segments, nparts):
    """Exact edge split (include/geot.h, R21): (seg_bounds, edge_bounds,
    boundary_keys [nparts+1, 2] = {idx[t_p - 1], idx[t_p]} or -1), int64 device tensors."""
    dev = _dev(idx)
    sb = torch.empty(nparts + 1, dtype=torch.int64, device=dev)
    eb = torch.empty(nparts + 1, dtype=torch.int64, device=dev)
    keys = torch.empty((nparts + 1, 2), dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        _lib.check(_L.geot_partition_exact(_ptr(idx), _it(idx), idx.numel(), num_segments, nparts, _ptr(sb), _ptr(eb),
                                           _ptr(keys), _stream(dev)), "geot_partition_exact")
    return sb, eb, keys


def geot_segment_reduce_split(src, idx, seg_base, num_segments, op="sum", head_open=False, tail_open=False,
                              out=None, cfg=None):
    """One part of the exact split: (out, partials [2, F] fp32, counts [2] int64); see include/geot.h."""
    dev = _dev(src, idx, out)
    if src.dim() != 2 or idx.dim() != 1 or src.shape[0] != idx.shape[0]:
        raise ValueError("src must be [nnz, F] and idx [nnz]")
    E, F = src.shape
    S = int(num_segments)
    if out is None:
        out = torch.empty((S, F), dtype=src.dtype, device=dev)
    elif out.shape != (S, F) or out.dtype != src.dtype:
        raise ValueError("out must be [num_segments, F] with src's dtype")
    part = torch.empty((2, F), dtype=torch.float32, device=dev)
    cnt = torch.empty(2, dtype=torch.int64, device=dev)
    ws_n = _L.geot_split_workspace_size(E, S, F, _op(op), _dt(src), _it(idx), _cfgp(cfg))
    ws, ws_bytes = _workspace(dev, ws_n)
    with torch.cuda.device(dev):
        st = _L.geot_segment_reduce_split(_ptr(src), _ptr(idx), E, seg_base, S, F, _op(op), _dt(src), _it(idx),
                                          int(bool(head_open)), int(bool(tail_open)), _ptr(out), _ptr(part),
                                          _ptr(cnt), _ptr(ws), ws_bytes, _cfgp(cfg), _stream(dev))
    _lib.check(st, "geot_segment_reduce_split")
    return out, part, cnt


def geot_combine_partials(partials, counts, slots, out_row, op="sum"):
    """out_row = finalize(fold of partials[slots] in order) (include/geot.h)."""
    dev = _dev(partials, counts, out_row)
    if partials.dtype != torch.float32 or counts.dtype != torch.int64:
        raise TypeError("partials must be float32 and counts int64")
    F = partials.shape[-1]
    if out_row.numel() != F:
        raise ValueError("out_row must hold F elements")
    n = partials.numel() // F
    if any(not 0 <= int(s_) < n for s_ in slots) or not 1 <= len(slots) <= 64:
        raise ValueError("1..64 slot ids within the partials")
    arr = (ctypes.c_int32 * len(slots))(*[int(s_) for s_ in slots])
    with torch.cuda.device(dev):
        _lib.check(_L.geot_combine_partials(_ptr(partials), _ptr(counts), arr, len(slots), F, _op(op), _dt(out_row),
                                            _ptr(out_row), _stream(dev)), "geot_combine_partials")
    return out_row


def geot_segment_reduce_backward(grad_out, idx, op="sum", offsets=None, src=None, out=None, grad_src=None):
    """Gradient w.r.t. src of geot_segment_reduce (seg_base 0); see include/geot.h."""
    dev = _dev(grad_out, idx, offsets, src, out, grad_src)
    S, F = grad_out.shape
    E = idx.numel()
    if grad_src is None:
        grad_src = torch.empty((E, F), dtype=grad_out.dtype, device=dev)
    if op == "mean" and offsets is None:
        offsets = geot_segment_offsets(idx, S)
    ties = torch.empty((S, F), dtype=torch.float32, device=dev) if op == "max" else None
    with torch.cuda.device(dev):
        _lib.check(_L.geot_segment_reduce_backward(_ptr(grad_out), _ptr(idx), E, S, F, _op(op), _dt(grad_out),
                                                   _it(idx), _ptr(offsets), _ptr(src), _ptr(out), _ptr(ties),
                                                   _ptr(grad_src), _stream(dev)), "geot_segment_reduce_backward")
    return grad_src


def geot_gather_segment_reduce_backward(grad_out, x, src_idx, dst_idx, op="sum", weight=None, offsets=None,
                                        need_x=True, need_w=False):
    """(grad_x, grad_weight) of the fused form (fp32); grad_x by fp32 atomics."""
    dev = _dev(grad_out, x, src_idx, dst_idx, weight, offsets)
    _check_gather_backward_args(x, op, grad_out)
    S, F = grad_out.shape
    V = x.shape[0]
    E = dst_idx.numel()
    if op == "mean" and offsets is None:
        offsets = geot_segment_offsets(dst_idx, S)
    gx = torch.empty((V, F), dtype=torch.float32, device=dev) if need_x else None
    gw = torch.empty(E, dtype=torch.float32, device=dev) if need_w else None
    with torch.cuda.device(dev):
        _lib.check(_L.geot_gather_segment_reduce_backward(_ptr(grad_out), _ptr(src_idx), _ptr(dst_idx),
                                                          _ptr(weight), E, S, V, F, _op(op), _it(dst_idx),
                                                          _ptr(offsets), _ptr(x), _ptr(gx), _ptr(gw), _stream(dev)),
                   "geot_gather_segment_reduce_backward")
    return gx, gw


def _check_gather_backward_args(x, reduce, grad_out=None):
    """The fused-form backward kernels take fp32 x / grad_out and sum/mean only."""
    if x.dtype != torch.float32 or (grad_out is not None and grad_out.dtype != torch.float32):
        raise TypeError("the fused-form backward supports float32 x and grad_out only")
    if reduce not in ("sum", "mean"):
        raise ValueError(f"the fused-form backward supports reduce='sum' or 'mean', got {reduce!r}")


class _SegmentReduceFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, src, idx, num_segments, reduce):
        out = geot_segment_reduce(src, idx, num_segments, reduce)
        ctx.reduce = reduce
        ctx.save_for_backward(idx, src if reduce == "max" else None, out if reduce == "max" else None)
        return out

    @staticmethod
    def backward(ctx, grad_out):
        idx, src, out = ctx.saved_tensors
        g = geot_segment_reduce_backward(grad_out.contiguous(), idx, ctx.reduce, src=src, out=out)
        return g, None, None, None


class _GatherSegmentReduceFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, src_idx, dst_idx, weight, num_segments, reduce):
        out = geot_gather_segment_reduce(x, src_idx, dst_idx, num_segments, reduce, weight=weight)
        ctx.reduce = reduce
        ctx.save_for_backward(x, src_idx, dst_idx, weight)
        return out

    @staticmethod
    def backward(ctx, grad_out):
        x, src_idx, dst_idx, weight = ctx.saved_tensors
        need_w = weight is not None and ctx.needs_input_grad[3]
        gx, gw = geot_gather_segment_reduce_backward(grad_out.contiguous(), x, src_idx, dst_idx, ctx.reduce,
                                                     weight=weight, need_x=ctx.needs_input_grad[0], need_w=need_w)
        return gx, None, None, gw, None, None


def segment_reduce_autograd(idx, msg, reduce="sum", num_segments=None):
    """segment_reduce with gradients w.r.t. msg (sum/mean/max)."""
    return _SegmentReduceFn.apply(msg, idx, _num_segments(idx, num_segments), reduce)


def index_segment_reduce_autograd(src_idx, dst_idx, x, reduce="sum", weight=None, num_segments=None):
    """Fused form with gradients w.r.t. x (and weight): fp32, sum/mean."""
    _check_gather_backward_args(x, reduce)  # refuse before the forward runs
    return _GatherSegmentReduceFn.apply(x, src_idx, dst_idx, weight, _num_segments(dst_idx, num_segments), reduce)


# ------------------------------------------------------------ paper-style API
def segment_reduce(idx, msg, reduce="sum", num_segments=None):
    """geot.segment_reduce(edge_index[1], msg, reduce=...)  — PAPER.md:289."""
    return geot_segment_reduce(msg, idx, num_segments, reduce)


def index_segment_reduce(src_idx, dst_idx, x, reduce="sum", num_segments=None):
    """geot.index_segment_reduce(edge_index[0], edge_index[1], x, reduce=...) — PAPER.md:293."""
    return geot_gather_segment_reduce(x, src_idx, dst_idx, num_segments, reduce)


def index_weight_segment_reduce(src_idx, dst_idx, weight, x, num_segments=None):
    """Weighted fused form (SpMM on sorted COO) — PAPER.md:330."""
    return geot_gather_segment_reduce(x, src_idx, dst_idx, num_segments, "sum", weight=weight)
