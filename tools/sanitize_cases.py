"""Small invocations of every kernel of the family, for compute-sanitizer
(memcheck / racecheck / synccheck; SURVEY §5 "Race detection / sanitizers"):

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py

Each case runs once on small synthetic inputs (power-law lengths with empty
segments) and is checked bit-exactly against a plain torch reference in integer
mode, so a sanitizer run is also a correctness run.  Forced configurations
exercise every variant: edge-tile (+ fix-up), narrow (2-D TMA ring + output
window), stream (1-D TMA ring / LDG pipeline), the fused gather forms, the
offsets / validate / partition kernels and the backward kernels.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2404_03019_b200 as geot  # noqa: E402
import synth  # noqa: E402
import synth.device as sd  # noqa: E402


def ref_reduce(X, idx, S, op):
    """torch segment reduction (test-side reference; integer-valued inputs)."""
    out = torch.zeros(S, X.shape[1], dtype=torch.float64, device=X.device)
    ii = idx.long()
    if op == "max":
        out = torch.full((S, X.shape[1]), float("-inf"), dtype=torch.float64, device=X.device)
        out.scatter_reduce_(0, ii[:, None].expand_as(X), X.double(), "amax")
        out[torch.isinf(out)] = 0
        return out
    out.index_add_(0, ii, X.double())
    if op == "mean":
        cnt = torch.bincount(ii, minlength=S).double().clamp(min=1)
        out = out / cnt[:, None]
    return out


def case(E, S, F, dt, op, cfg, fused=False):
    L = synth.segment_lengths(E, S, "powerlaw", 11)
    idx = sd.index_from_lengths(L)
    tdt = torch.float32 if dt == "f32" else torch.bfloat16
    if fused:
        x = sd.values(S, F, 5, dtype=tdt, mode="int")
        src = sd.src_index(E, S, 1005)
        y = geot.geot_gather_segment_reduce(x, src, idx, S, op, cfg=cfg)
        ref = ref_reduce(x[src.long()], idx, S, op)
    else:
        X = sd.values(E, F, 5, dtype=tdt, mode="int")
        y = geot.geot_segment_reduce(X, idx, S, op, cfg=cfg)
        ref = ref_reduce(X, idx, S, op)
    torch.cuda.synchronize()
    ok = torch.equal(y.double(), ref.to(tdt).double())
    print(f"{'fused ' if fused else ''}E={E} S={S} F={F} {dt} {op} cfg={cfg}: {'ok' if ok else 'MISMATCH'}", flush=True)
    return ok


def main():
    allok = True
    E, S = 70_000, 9_000
    for op in ("sum", "mean", "max"):
        allok &= case(E, S, 1, "f32", op, {"variant": 2})          # narrow
        allok &= case(E, S, 4, "bf16", op, {"variant": 2})
        allok &= case(E, S, 128, "f32", op, {"variant": 3})        # stream, selector's pipeline
        allok &= case(E, S, 16, "f32", op, {"variant": 3})         # stream, 8 agents per warp (3-D TMA)
        allok &= case(E, S, 16, "f32", op, {"variant": 2})         # narrow, lane groups of 4
        allok &= case(E, S, 64, "bf16", op, {"variant": 1})        # edge tile + fix-up
        allok &= case(E, S, 12, "f32", op, {"variant": 1})         # scalar-vector edge tile
        allok &= case(E, S, 64, "f32", op, {"variant": 3}, fused=True)
    allok &= case(E, S, 32, "f32", "sum", {"variant": 3, "warps_per_cta": 8, "rows_per_group": 4, "stages": 1})
    allok &= case(E, S, 48, "f32", "sum", {"variant": 1}, fused=True)
    # integer kernels
    L = synth.segment_lengths(E, S, "powerlaw", 11)
    idx = sd.index_from_lengths(L)
    off = geot.geot_segment_offsets(idx, S)
    allok &= bool(torch.equal(off[1:] - off[:-1], torch.as_tensor(L, device=off.device, dtype=off.dtype)))
    allok &= geot.geot_validate_index(idx, S) == 0
    geot.geot_partition(idx, S, 4)
    # backward kernels
    X = sd.values(E, 32, 5, dtype=torch.float32, mode="int").requires_grad_(True)
    y = geot.segment_reduce_autograd(idx, X, "mean", num_segments=S)
    y.sum().backward()
    x = sd.values(S, 32, 5, dtype=torch.float32, mode="int").requires_grad_(True)
    src = sd.src_index(E, S, 1005)
    y = geot.index_segment_reduce_autograd(src, idx, x, "sum", num_segments=S)
    y.sum().backward()
    torch.cuda.synchronize()
    print("ALL OK" if allok else "FAILURES", flush=True)
    sys.exit(0 if allok else 1)


if __name__ == "__main__":
    main()
