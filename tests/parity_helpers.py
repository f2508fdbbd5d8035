"""Shared helpers of the parity tests: build seeded inputs with `synth`, run the
CUDA path through the C ABI (paper_2404_03019_b200), run the oracle, compare.

Comparison rule (SURVEY.md §8(c) "Parity rule"):
  * max, offsets, counts, partition bounds, and everything in integer mode:
    bit-exact against the oracle's rounded result;
  * sum / mean with real inputs: |y - y64| <= tol * A, A = sum |x| over the
    segment (mean: A / count), tol = 1e-5 (fp32 inputs) or 1e-2 (bf16 inputs).
"""
from __future__ import annotations

import numpy as np

import oracle
import synth

TOL = {"f32": 1e-5, "bf16": 1e-2}


def make_case(E, S, F, dtype="f32", mode="real", kind="powerlaw", seed=0, lengths=None):
    L = synth.stress_lengths(kind, E, S, seed) if lengths is None else np.asarray(lengths)
    idx = synth.lengths_to_index(L, "i64")
    X = synth.values(seed + 17, 0, E, F, dtype, mode)
    return L, idx, X


def to_torch_vals(X, device="cuda"):
    import torch
    if X.dtype == np.uint16:
        return torch.from_numpy(X.view(np.int16)).view(torch.bfloat16).to(device)
    return torch.from_numpy(X).to(device)


def from_torch_vals(t):
    import torch
    t = t.detach().cpu()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view(np.uint16)
    return t.numpy()


def as_f64(a):
    if a.dtype == np.uint16:
        return synth.bf16_bits_to_f32(a).astype(np.float64)
    return a.astype(np.float64)


def check(y, ref: "oracle.Result", op, dtype, mode, counts=None, what=""):
    """Assert y (numpy, dtype storage) matches the oracle result."""
    assert y.shape == ref.rounded.shape, (what, y.shape, ref.rounded.shape)
    if op == "max" or mode == "int":
        bad = np.nonzero(y.view(np.uint32 if y.dtype == np.float32 else np.uint16)
                         != ref.rounded.view(np.uint32 if y.dtype == np.float32 else np.uint16))
        if bad[0].size:
            i = (bad[0][0], bad[1][0])
            raise AssertionError(f"{what}: {bad[0].size} elements differ bitwise; first at {i}: "
                                 f"gpu={as_f64(y)[i]!r} oracle={ref.y64[i]!r}")
        return
    yy = as_f64(y)
    A = ref.absum
    if op == "mean":
        c = np.maximum(counts, 1)[:, None].astype(np.float64)
        A = A / c
    err = np.abs(yy - ref.y64)
    lim = TOL[dtype] * A
    bad = np.nonzero(err > lim)
    if bad[0].size:
        i = (bad[0][0], bad[1][0])
        raise AssertionError(f"{what}: {bad[0].size} elements out of tolerance; first at {i}: gpu={yy[i]!r} "
                             f"oracle={ref.y64[i]!r} A={A[i]!r} rel={err[i] / max(A[i], 1e-300):.3e}")
