"""Analysis consumers of the solve phase.

Consumers of the device applies in helmdd.analysis, restated with batched
device work: ``fov_bounds`` (analysis.py:342-375), ``check_tf_stability``
(:427-454), ``check_t0_stability`` (:457-480) and ``check_prop26_identity``
(:497-515), returning the reference's CheckReport.

``fov_bounds`` restates helmdd.analysis.fov_bounds (analysis.py:342-375):
the measured field-of-values constants of T = M^{-1} B in the D_k metric.
The reference applies T one vector at a time (n applies in dense mode, 500
in sampled mode); here the applies run as batched device applies of up to
16 columns (``as_operator("T").apply_multi``), and so do the D_k products.
The random vectors are drawn in the reference's order from the same
generator, so the sampled bounds agree with the reference to rounding.
"""

from dataclasses import dataclass, field

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


# ---------------------------------------------------------------- lemma checks
SLACK_RTOL = 1e-9


@dataclass
class CheckReport:
    """Outcome of one inequality sweep (analysis.py:16-36)."""

    name: str
    trials: int
    violations: int
    worst_margin: float     # min over trials of rhs - lhs + slack (>= 0 passes)
    witness: int            # trial index attaining the worst margin
    slack_rtol: float = SLACK_RTOL
    extra: dict = field(default_factory=dict)

    @property
    def passed(self):
        return self.violations == 0


def _slack(lhs, rhs):
    """analysis.py:186-187."""
    return SLACK_RTOL * (abs(lhs) + abs(rhs))


def _sweep(name, margins, extra=None):
    """analysis.py:190-200."""
    margins = np.asarray(margins)
    worst = int(margins.argmin()) if margins.size else 0
    return CheckReport(name=name, trials=int(margins.size), violations=int(np.sum(margins < 0.0)),
                       worst_margin=float(margins[worst]) if margins.size else np.inf, witness=worst,
                       extra=extra or {})


def _chunks(total, batch):
    for c0 in range(0, total, batch):
        yield c0, min(total, c0 + batch)


def check_tf_stability(forms, dec, precond, trials=20, rng=None):
    """Local stability of the fine projectors (analysis.py:427-454): for
    blocks with H^f_{i,j} k <= sqrt(2)/2, ||T_{i,j} u||_{1,k,loc} <=
    2 ||u||_{1,k,loc}.  B u runs as batched device SpMMs, the local solves
    as device band solves (``ls.lu.solve``); draws in the reference's order."""
    from .factor import submatrix
    from .fem import local_forms_sparse

    rng = rng or np.random.default_rng(0)
    k = forms.k
    n = forms.n_dofs
    margins = []
    by_pair = {(ls.coarse_index, ls.fine_index): ls for ls in precond.local_solvers}
    B_op = precond.as_operator("B")
    for i, j, sub in dec.fine_flat():
        if sub.diameter * k > np.sqrt(2.0) / 2.0 or sub.idof.size == 0:
            continue
        A_loc, S_loc = local_forms_sparse(forms, sub.elements, sub.ovdof)
        dk_ov = (A_loc + k**2 * S_loc).tocsr()
        dk_ii = submatrix(forms.dk, sub.idof, sub.idof)
        ls = by_pair[(i, j)]
        U = np.stack([rng.standard_normal(n) for _ in range(trials)], axis=1) if trials else np.zeros((n, 0))
        for c0, c1 in _chunks(trials, _lib.MAX_RHS):
            BU = B_op.apply_multi(U[:, c0:c1])
            for c in range(c1 - c0):
                tfu = ls.lu.solve(np.ascontiguousarray(BU[sub.idof, c]))
                lhs = float(np.sqrt(tfu @ (dk_ii @ tfu)))
                u_ov = U[sub.ovdof, c0 + c]
                rhs = 2.0 * float(np.sqrt(u_ov @ (dk_ov @ u_ov)))
                margins.append(rhs - lhs + _slack(lhs, rhs))
    return _sweep("tf_stability", margins)


def check_t0_stability(forms, coarse, precond, theory, trials=20, rng=None):
    """Coarse-projector stability ||u - T_0 u||_{1,k} <= 2 ||u||_{1,k}
    (analysis.py:457-480), asserted only under 2 k Lambda^2 sqrt(Theta)
    (1 + Cstab) <= 1/2.  T_0 u = apply_coarse(B u) on the device; the D_k
    norms as batched device SpMMs."""
    rng = rng or np.random.default_rng(0)
    cond = 2.0 * theory.k * theory.lambda_overlap**2 * np.sqrt(theory.theta) * (1.0 + theory.cstab_estimate)
    margins = []
    if cond <= 0.5 and precond.has_coarse:
        n = forms.n_dofs
        U = np.stack([rng.standard_normal(n) for _ in range(trials)], axis=1) if trials else np.zeros((n, 0))
        B_op, D_op = precond.as_operator("B"), precond.as_operator("Dk")
        for c0, c1 in _chunks(trials, _lib.MAX_RHS):
            Uc = U[:, c0:c1]
            BU = B_op.apply_multi(Uc)
            T0U = np.stack([precond.apply_coarse(np.ascontiguousarray(BU[:, c])) for c in range(c1 - c0)], axis=1)
            Dm = Uc - T0U
            DD = D_op.apply_multi(Dm)
            DU = D_op.apply_multi(Uc)
            for c in range(c1 - c0):
                lhs = float(np.sqrt(Dm[:, c] @ DD[:, c]))
                rhs = 2.0 * float(np.sqrt(Uc[:, c] @ DU[:, c]))
                margins.append(rhs - lhs + _slack(lhs, rhs))
    return _sweep("t0_stability", margins, extra={"hypothesis_value": float(cond)})


def check_prop26_identity(forms, precond, trials=50, rng=None):
    """<M^{-1} B u, v>_{D_k} through D_k equals (T u, v)_{1,k} through the
    split A + k^2 S to 1e-12 relative (analysis.py:497-515).  M^{-1} B U and
    T U run as batched device applies, the D_k / A / S products as batched
    device SpMMs; u, v drawn in the reference's order."""
    from .schwarz import CsrOperator

    rng = rng or np.random.default_rng(0)
    n = forms.n_dofs
    k2 = forms.k**2
    draws = [(rng.standard_normal(n), rng.standard_normal(n)) for _ in range(trials)]
    B_op, M_op, T_op, D_op = (precond.as_operator(x) for x in ("B", "M", "T", "Dk"))
    A_op, S_op = CsrOperator(forms.stiffness), CsrOperator(forms.mass)
    margins = []
    for c0, c1 in _chunks(trials, _lib.MAX_RHS):
        U = np.stack([draws[c][0] for c in range(c0, c1)], axis=1)
        V = np.stack([draws[c][1] for c in range(c0, c1)], axis=1)
        MBU = M_op.apply_multi(B_op.apply_multi(U))
        DMBU = D_op.apply_multi(MBU)
        TU = T_op.apply_multi(U)
        ATU, STU = A_op.apply_multi(TU), S_op.apply_multi(TU)
        for c in range(c1 - c0):
            lhs = float(V[:, c] @ DMBU[:, c])
            rhs = float(V[:, c] @ ATU[:, c]) + k2 * float(V[:, c] @ STU[:, c])
            tol = 1e-12 * (abs(lhs) + abs(rhs))
            margins.append(tol - abs(lhs - rhs))
    return _sweep("prop26_identity", margins)
