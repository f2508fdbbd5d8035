"""Pins for the oracle's gradients against finite differences
of the forward oracle (an independent computation: the derivative of P:85's
definition taken numerically), plus the tie-splitting convention (reading R19)
on a hand case.  No GPU needed."""
import numpy as np

import oracle


def numeric_vjp_X(X, idx, S, op, dY, h):
    """d<dY, f(X)>/dX by central differences of the forward oracle (fp64 y64)."""
    g = np.zeros(X.shape, dtype=np.float64)
    for e in range(X.shape[0]):
        for f in range(X.shape[1]):
            Xp, Xm = X.copy(), X.copy()
            Xp[e, f] += h
            Xm[e, f] -= h
            fp = oracle.segment_reduce(Xp, idx, S, op).y64
            fm = oracle.segment_reduce(Xm, idx, S, op).y64
            g[e, f] = np.sum(dY * (fp - fm)) / (2 * h)
    return g


def test_sum_mean_vjp_equals_finite_differences():
    rng = np.random.default_rng(0)
    for op in ("sum", "mean"):
        for _ in range(6):
            E, S, F = int(rng.integers(1, 14)), int(rng.integers(1, 6)), int(rng.integers(1, 4))
            idx = np.sort(rng.integers(0, S, size=E))
            X = rng.integers(-8, 9, size=(E, F)).astype(np.float32)  # exact: linear ops, h = 1
            dY = rng.integers(-5, 6, size=(S, F)).astype(np.float64)
            np.testing.assert_allclose(oracle.segment_reduce_backward(dY, X, idx, op),
                                       numeric_vjp_X(X, idx, S, op, dY, 1.0), rtol=1e-12, atol=1e-12)


def test_max_vjp_equals_finite_differences_without_ties():
    rng = np.random.default_rng(1)
    for _ in range(6):
        E, S, F = int(rng.integers(1, 14)), int(rng.integers(1, 6)), int(rng.integers(1, 4))
        idx = np.sort(rng.integers(0, S, size=E))
        X = (rng.permutation(E * F).reshape(E, F) * 0.125 - 3).astype(np.float32)  # distinct, gaps 0.125
        dY = rng.normal(size=(S, F))
        np.testing.assert_allclose(oracle.segment_reduce_backward(dY, X, idx, "max"),
                                   numeric_vjp_X(X, idx, S, "max", dY, 2.0 ** -6), rtol=1e-9, atol=1e-12)


def test_max_ties_split_evenly():
    X = np.array([[2.0], [5.0], [5.0], [1.0], [5.0]], dtype=np.float32)
    idx = np.array([0, 0, 0, 0, 1])
    dY = np.array([[6.0], [4.0]])
    np.testing.assert_array_equal(oracle.segment_reduce_backward(dY, X, idx, "max")[:, 0], [0, 3, 3, 0, 4])


def test_gather_vjp_equals_finite_differences():
    rng = np.random.default_rng(2)
    for op in ("sum", "mean"):
        for weighted in (False, True):
            V, E, S, F = 5, 12, 4, 3
            dst = np.sort(rng.integers(0, S, size=E))
            src = rng.integers(0, V, size=E)
            x = rng.integers(-4, 5, size=(V, F)).astype(np.float32)
            w = rng.integers(1, 4, size=E).astype(np.float32) if weighted else None
            dY = rng.integers(-3, 4, size=(S, F)).astype(np.float64)
            dx, dw = oracle.gather_segment_reduce_backward(dY, x, src, dst, op, weight=w)

            def fwd(xx, ww):
                return oracle.gather_segment_reduce(xx, src, dst, S, op, weight=ww).y64

            num = np.zeros_like(dx)
            for v in range(V):
                for f in range(F):
                    xp, xm = x.copy(), x.copy()
                    xp[v, f] += 1
                    xm[v, f] -= 1
                    num[v, f] = np.sum(dY * (fwd(xp, w) - fwd(xm, w))) / 2
            np.testing.assert_allclose(dx, num, rtol=1e-12, atol=1e-12)
            # weight gradient: f is linear in w -> exact with h = 1
            w0 = np.ones(E, np.float32) if w is None else w
            numw = np.zeros(E)
            for e in range(E):
                wp, wm = w0.copy(), w0.copy()
                wp[e] += 1
                wm[e] -= 1
                numw[e] = np.sum(dY * (fwd(x, wp) - fwd(x, wm))) / 2
            np.testing.assert_allclose(dw, numw, rtol=1e-12, atol=1e-12)
