"""Analysis consumers of the solve phase.

``fov_bounds`` restates helmdd.analysis.fov_bounds (analysis.py:342-375):
the measured field-of-values constants of T = M^{-1} B in the D_k metric.
The reference applies T one vector at a time (n applies in dense mode, 500
in sampled mode); here the applies run as batched device applies of up to
16 columns (``as_operator("T").apply_multi``), and so do the D_k products.
The random vectors are drawn in the reference's order from the same
generator, so the sampled bounds agree with the reference to rounding.
"""

import numpy as np
import scipy.linalg

from . import _lib


def _batched(op, U):
    return op.apply_multi(U)


def fov_bounds(forms, precond, mode="dense", samples=500, rng=None, batch=None):
    """(c1, c2): the smallest eigenvalue of the D_k-symmetric part of T and
    the largest of T^T D_k T in the D_k pencil (dense), or their inner bounds
    from random Rayleigh quotients (sampled).  analysis.py:342-375."""
    Dk = forms.dk
    n = forms.n_dofs if hasattr(forms, "n_dofs") else Dk.shape[0]
    batch = int(batch or _lib.MAX_RHS)
    T_op = precond.as_operator("T")
    D_op = precond.as_operator("Dk")
    if mode == "dense":
        T = np.empty((n, n))
        for j0 in range(0, n, batch):
            j1 = min(n, j0 + batch)
            E = np.zeros((n, j1 - j0))
            E[np.arange(j0, j1), np.arange(j1 - j0)] = 1.0
            T[:, j0:j1] = _batched(T_op, E)
        Dk_d = Dk.toarray()
        M1 = Dk_d @ T
        sym = 0.5 * (M1 + M1.T)
        c1 = float(scipy.linalg.eigh(sym, Dk_d, eigvals_only=True)[0])
        c2 = float(scipy.linalg.eigh(T.T @ M1, Dk_d, eigvals_only=True)[-1])
        return c1, c2
    if mode == "sampled":
        rng = rng or np.random.default_rng(0)
        c1 = np.inf
        c2 = 0.0
        done = 0
        while done < samples:
            b = min(batch, samples - done)
            U = np.stack([rng.standard_normal(n) for _ in range(b)], axis=1)  # the reference's draw order
            TU = _batched(T_op, U)
            DU = _batched(D_op, U)
            DTU = _batched(D_op, TU)
            for c in range(b):  # the reference's per-sample reductions, in order
                denom = float(U[:, c] @ DU[:, c])
                c1 = min(c1, float(TU[:, c] @ DU[:, c]) / denom)
                c2 = max(c2, float(TU[:, c] @ DTU[:, c]) / denom)
            done += b
        return float(c1), float(c2)
    raise ValueError("mode must be 'dense' or 'sampled'")
