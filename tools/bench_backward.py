"""Time the gradient kernels (f3, backward.cu) and the weighted fused form
(f1, index_weight_segment_reduce = SpMM on sorted COO) on
BASELINE-shaped inputs; one JSON line per case.

    python tools/bench_backward.py [--reps 20]

Bytes (algorithmic, per call):
  segment backward (sum/mean):  E*F*s (dX written) + S*F*s (dY read once) + E*4 (idx) [+ (S+1)*8 offsets]
  gather backward w.r.t. x:     E*F*4 logical (dY rows gathered by dst, reduced into dx by src) + 2E*4 + V*F*4
  SDDMM (edge-weight grad):      2*E*F*4 logical (x rows by src, dY rows by dst) + 2E*4 + E*4
  weighted fused forward:        E*F*4 logical gathered rows + 2E*4 + E*4 (w) + S*F*4
The gather-shaped kernels are L2-bound (Reddit's x / dY = 59.6 MB stay in the
126 MB L2): reported as logical GB/s beside the measured L2 row-gather ceiling
(profiles/l2_gather_peak.json); the segment backward is HBM-bound.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2404_03019_b200 as geot  # noqa: E402
from tools.sweep import make_inputs, time_call  # noqa: E402

ARXIV = (1_166_243, 169_343)
REDDIT = (114_615_892, 232_965)


def line(**kw):
    print(json.dumps(kw), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")

    # segment_reduce backward, arxiv-shaped F=128 fp32 and products-shaped bf16
    for (E, S, F, dt) in ((ARXIV[0], ARXIV[1], 128, "f32"), (61_859_140, 2_449_029, 128, "bf16")):
        L, idx, X, _ = make_inputs(E, S, F, dt, "powerlaw", 5)
        off = geot.geot_segment_offsets(idx, S)
        dY = torch.randn(S, F, device="cuda").to(X.dtype)
        dX = torch.empty_like(X)
        esz = X.element_size()
        for op in ("sum", "mean"):
            fn = lambda: geot.geot_segment_reduce_backward(dY, idx, op, offsets=off, grad_src=dX)  # noqa: E731
            med, _ = time_call(fn, args.reps, flush if E * F * esz < 4 * (126 << 20) else None)
            B = E * F * esz + S * F * esz + E * 4 + (S + 1) * 8
            line(kernel="segment_reduce_backward", op=op, E=E, S=S, F=F, dtype=dt, us=round(med * 1e3, 1),
                 GBps=round(B / (med * 1e-3) / 1e9, 1), bytes=B)
        del X, dX, dY, idx, off
        torch.cuda.empty_cache()

    # fused (Reddit-shaped): weighted forward at F in {16, 32, 64, 128}; x-gradient and SDDMM at F = 64
    E, S = REDDIT
    for F in (16, 32, 64, 128):
        L, idx, x, src = make_inputs(E, S, F, "f32", "powerlaw", 5, fused=True, V=S)
        w = torch.rand(E, device="cuda", dtype=torch.float32)
        out = torch.empty(S, F, device="cuda", dtype=torch.float32)
        fn = lambda: geot.geot_gather_weight_segment_reduce(x, src, idx, w, S, out=out)  # noqa: E731
        med, _ = time_call(fn, args.reps)
        B = E * F * 4 + 3 * E * 4 + S * F * 4
        line(kernel="index_weight_segment_reduce", E=E, S=S, F=F, dtype="f32", us=round(med * 1e3, 1),
             GBps_logical=round(B / (med * 1e-3) / 1e9, 1), bytes_logical=B)
        if F == 64:
            off = geot.geot_segment_offsets(idx, S)
            dY = torch.randn(S, F, device="cuda")
            for op in ("sum", "mean"):
                fn = lambda: geot.geot_gather_segment_reduce_backward(dY, x, src, idx, op, weight=w,  # noqa: E731
                                                                        offsets=off, need_x=True, need_w=False)
                try:
                    med, _ = time_call(fn, args.reps)
                    B = E * F * 4 + 2 * E * 4 + E * 4 + S * F * 4
                    line(kernel="gather_backward_x", op=op, E=E, S=S, F=F, us=round(med * 1e3, 1),
                         GBps_logical=round(B / (med * 1e-3) / 1e9, 1), bytes_logical=B)
                except TypeError as e:
                    line(kernel="gather_backward_x", error=str(e))
            fn = lambda: geot.geot_gather_segment_reduce_backward(dY, x, src, idx, "sum", weight=w,  # noqa: E731
                                                                    offsets=off, need_x=False, need_w=True)
            try:
                med, _ = time_call(fn, args.reps)
                B = 2 * E * F * 4 + 3 * E * 4
                line(kernel="sddmm", E=E, S=S, F=F, us=round(med * 1e3, 1),
                     GBps_logical=round(B / (med * 1e-3) / 1e9, 1), bytes_logical=B)
            except TypeError as e:
                line(kernel="sddmm", error=str(e))
        del x, src, idx, w, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
