"""Independent dense oracles (TEST INFRASTRUCTURE ONLY).

Restates the reference test oracles pkg/tests/oracles.py:100-124 and
146-180: the explicit dense one-/two-level Schwarz matrices and a textbook
(Euclidean, unrestarted) GMRES with per-step least squares.
"""

import numpy as np


def dense_one_level(forms, dec):
    n = forms.helmholtz.shape[0]
    B = forms.helmholtz.toarray()
    M = np.zeros((n, n))
    for _i, _j, sub in dec.fine_flat():
        idof = np.asarray(sub.idof)
        if idof.size:
            M[np.ix_(idof, idof)] += np.linalg.inv(B[np.ix_(idof, idof)])
    return M


def dense_two_level(forms, dec, Z):
    M = dense_one_level(forms, dec)
    Zd = np.asarray(Z.todense()) if hasattr(Z, "todense") else np.asarray(Z)
    if Zd.shape[1]:
        B0 = Zd.T @ forms.helmholtz.toarray() @ Zd
        M = M + Zd @ np.linalg.solve(B0, Zd.T)
    return M


def textbook_gmres(A, b, maxit, rtol=0.0):
    n = b.size
    beta = np.linalg.norm(b)
    V = np.zeros((n, maxit + 1))
    H = np.zeros((maxit + 1, maxit))
    V[:, 0] = b / beta
    hist = [beta]
    m = maxit
    for j in range(maxit):
        w = A @ V[:, j]
        for i in range(j + 1):
            H[i, j] = V[:, i] @ w
            w = w - H[i, j] * V[:, i]
        H[j + 1, j] = np.linalg.norm(w)
        e1 = np.zeros(j + 2)
        e1[0] = beta
        if H[j + 1, j] <= 1e-14 * max(np.abs(H[: j + 2, j]).max(), 1.0):
            m = j + 1
            y = np.linalg.lstsq(H[: m + 1, :m], e1, rcond=None)[0]
            hist.append(np.linalg.norm(e1 - H[: m + 1, :m] @ y))
            return V[:, :m] @ y, np.array(hist)
        V[:, j + 1] = w / H[j + 1, j]
        y = np.linalg.lstsq(H[: j + 2, : j + 1], e1, rcond=None)[0]
        hist.append(np.linalg.norm(e1 - H[: j + 2, : j + 1] @ y))
        if hist[-1] <= rtol * beta:
            m = j + 1
            break
    e1 = np.zeros(m + 1)
    e1[0] = beta
    y = np.linalg.lstsq(H[: m + 1, :m], e1, rcond=None)[0]
    return V[:, :m] @ y, np.array(hist)
