"""CPU oracle of the weighted GMRES (TEST INFRASTRUCTURE ONLY).

Restates pkg/src/helmdd/wgmres.py:74-203 step by step: r0 = rhs - op(x0),
beta = ||r0||_W; per iteration w = op(V_j), modified Gram-Schmidt against
the cached W V, ||w||_W, the always-taken measurement corr = (W V)^T w with a
second pass when max|corr| > 1e-12 ||w||_W, breakdown test at 1e-14 of the
column scale, Givens update, stop when |g_{j+1}| <= rtol * beta;
x = x0 + V H^{-1} g.
"""

import numpy as np
import scipy.linalg


def weighted_gmres(op, rhs, weight=None, rtol=1e-6, maxit=200, x0=None, basis_state=None):
    """``basis_state`` (timing slices of the CPU baseline only): (V, WV), a
    list of j+1 basis vectors and their W images to resume from, so that
    iterations j, j+1, ... run with the cost they have deep into a solve (the
    per-iteration work grows with j); the returned x is then meaningless."""
    apply = op if callable(op) else (lambda v: op @ v)
    rhs = np.asarray(rhs, dtype=float)
    n = rhs.size
    W = (lambda v: v.copy()) if weight is None else (lambda v: weight @ v)
    x0 = np.zeros(n) if x0 is None else np.asarray(x0, dtype=float)
    r0 = rhs - apply(x0) if x0.any() else rhs.copy()
    wr0 = W(r0)
    beta = float(np.sqrt(r0 @ wr0))
    if beta == 0.0:
        return x0.copy(), dict(iterations=0, history=np.array([0.0]), converged=True, breakdown=False, reorth=0)
    j_start = 0
    if basis_state is not None:
        basis, wbasis = list(basis_state[0]), list(basis_state[1])
        j_start = len(basis) - 1
        maxit = int(min(maxit + j_start, n))
    else:
        maxit = int(min(maxit, n))
        basis, wbasis = [r0 / beta], [wr0 / beta]
    H = np.zeros((maxit + 1, maxit))
    cs, sn = np.ones(maxit), np.zeros(maxit)
    g = np.zeros(maxit + 1)
    g[j_start] = beta
    hist = [beta]
    converged = breakdown = False
    reorth = 0
    for j in range(j_start, maxit):
        w = np.array(apply(basis[j]), dtype=float, copy=True)
        col = np.zeros(j + 2)
        for i in range(j + 1):
            col[i] = float(wbasis[i] @ w)
            w -= col[i] * basis[i]
        ww = W(w)
        hn = float(np.sqrt(max(w @ ww, 0.0)))
        corr = np.array([wbasis[i] @ w for i in range(j + 1)])
        if np.abs(corr).max() > 1e-12 * max(hn, 1e-300):
            reorth += 1
            for i in range(j + 1):
                w -= corr[i] * basis[i]
            col[: j + 1] += corr
            ww = W(w)
            hn = float(np.sqrt(max(w @ ww, 0.0)))
        col[j + 1] = hn
        if hn <= 1e-14 * max(np.abs(col).max(), 1e-300):
            breakdown = True
        else:
            basis.append(w / hn)
            wbasis.append(ww / hn)
        for i in range(j):
            a, b = col[i], col[i + 1]
            col[i], col[i + 1] = cs[i] * a - sn[i] * b, sn[i] * a + cs[i] * b
        d = np.hypot(col[j], col[j + 1])
        cs[j], sn[j] = (1.0, 0.0) if d == 0.0 else (col[j] / d, -col[j + 1] / d)
        col[j] = cs[j] * col[j] - sn[j] * col[j + 1]
        col[j + 1] = 0.0
        H[: j + 2, j] = col
        g[j + 1] = sn[j] * g[j]
        g[j] = cs[j] * g[j]
        hist.append(abs(g[j + 1]))
        if hist[-1] <= rtol * beta or breakdown:
            converged = True
            break
    m = len(hist) - 1
    if j_start:
        return None, dict(iterations=m, history=np.asarray(hist), converged=converged, breakdown=breakdown,
                          reorth=reorth)
    y = scipy.linalg.solve_triangular(H[:m, :m], g[:m], lower=False) if m else np.zeros(0)
    x = x0 + (np.column_stack(basis[:m]) @ y if m else 0.0)
    return x, dict(iterations=m, history=np.asarray(hist), converged=converged, breakdown=breakdown, reorth=reorth)
