"""Drop-in GPU ``weighted_gmres`` (pkg/src/helmdd/wgmres.py:74-203).

Same signature, same report, same semantics: full (unrestarted) GMRES on the
already preconditioned operator, Arnoldi orthonormalisation in the
<u, v>_W = v^T W u inner product with cached W V, the reference's measured
conditional reorthogonalisation, Givens rotations and the stopping test
``|g_{j+1}| <= rtol * beta`` on the host, lucky breakdown handled as
convergence, ``maxit = min(maxit, n)``.

Orthogonalisation (``orth``), numerics not semantics:
  "measured" — the reference's scheme decision for decision: a classical
      first pass (one fused device reduction, where the reference runs MGS),
      the always-taken measurement pass, and a second pass exactly when
      wgmres.py:142-148 takes one;
  "dcgs2" (default) — delayed classical Gram-Schmidt twice: every vector is
      reorthogonalised once, one iteration late, with the reorthogonalisation
      and projection dots sharing one read of the basis and the correction
      sharing one read with the projection update (two basis reads per
      iteration instead of three to four; include/helmgpu.h).  At config 5
      the reference's rule fires on ~80% of iterations, so both schemes
      orthogonalise twice almost always; parity bars are tested for both.

The operator must live on the device: a ``DeviceOperator`` from
``TwoLevelPreconditioner.as_operator()``, or a matrix (scipy sparse / dense
ndarray), which is uploaded as a device CSR operator.  Host callables raise
TypeError — there is no CPU fallback.  ``weight`` may be None (Euclidean),
the ``forms.dk`` the preconditioner was built from (its device copy is
used), or any SPD matrix (uploaded).
"""

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .schwarz import CsrOperator, DeviceOperator, _as_device, _as_device_batch, _from_device_batch, _stream, _torch, _vp


@dataclass
class GmresReport:
    """Convergence record (wgmres.py:20-36)."""

    iterations: int
    residual_history: np.ndarray
    converged: bool
    elman_envelope: np.ndarray = None
    gamma_used: float = None
    envelope_clamped: bool = False
    breakdown: bool = False
    reorth_passes: int = field(default=0, compare=False)


def elman_gamma(c1, c2, c2_bounds="norm_squared"):
    """Field-of-values decay rate (wgmres.py:39-54)."""
    if c1 <= 0.0 or c2 <= 0.0:
        raise ValueError("both constants must be positive, got %g, %g" % (c1, c2))
    if c2_bounds == "norm_squared":
        return float(c1 / np.sqrt(c2))
    if c2_bounds == "norm":
        return float(c1 / c2)
    raise ValueError("c2_bounds must be 'norm_squared' or 'norm'")


def _envelope(gamma, r0, iterations):
    """wgmres.py:63-71."""
    if gamma is None:
        return None, False
    m = np.arange(iterations + 1)
    if gamma >= 1.0:
        env = np.zeros(iterations + 1)
        env[0] = r0
        return env, True
    return r0 * (1.0 - gamma**2) ** (m / 2.0), False


def _device_op(op):
    if isinstance(op, (DeviceOperator, CsrOperator)):
        return op, op
    if callable(op) and not hasattr(op, "shape"):
        raise TypeError(
            "weighted_gmres on the GPU needs a device operator (precond.as_operator()) or a matrix; "
            "a host callable would run the operator on the CPU"
        )
    o = CsrOperator(op)
    return o, o


def _device_weight(weight, op):
    if weight is None:
        return None, None
    pre = getattr(op, "precond", None)
    if pre is not None and getattr(pre.forms, "dk", None) is weight:
        w = DeviceOperator(pre, 3)
        return w, w
    if isinstance(weight, (DeviceOperator, CsrOperator)):
        return weight, weight
    w = CsrOperator(weight)
    return w, w


class _orth_mode:
    """Select the library's orthogonalisation for one call."""

    def __init__(self, orth):
        self.mode = None if orth is None else _lib.ORTH[orth]

    def __enter__(self):
        if self.mode is not None:
            lib = _lib.load()
            self.prev = lib.hg_get_orthogonalization()
            _lib.check(lib.hg_set_orthogonalization(self.mode), "hg_set_orthogonalization")

    def __exit__(self, *exc):
        if self.mode is not None:
            _lib.load().hg_set_orthogonalization(self.prev)


def weighted_gmres(op, rhs, weight=None, rtol=1e-6, maxit=200, x0=None, gamma=None, orth=None):
    """Solve op(x) = rhs by full GMRES in the ``weight`` inner product.

    Returns (x, GmresReport); x has the type of ``rhs`` (numpy in, numpy
    out; CUDA tensor in, CUDA tensor out).  ``orth``: "dcgs2" (default) or
    "measured" (see the module docstring)."""
    with _orth_mode(orth):
        return _weighted_gmres(op, rhs, weight, rtol, maxit, x0, gamma)


def _weighted_gmres(op, rhs, weight, rtol, maxit, x0, gamma):
    dop, keep_op = _device_op(op)
    dw, keep_w = _device_weight(weight, dop)
    torch = _torch()
    n = dop.n
    r, was_np = _as_device(rhs, n)
    x0t = None
    if x0 is not None:
        x0t, _ = _as_device(x0, n)
    x = torch.empty_like(r)
    maxit_eff = int(max(0, min(maxit, n)))
    hist = np.zeros(maxit_eff + 1)
    info = np.zeros(4, dtype=np.int32)
    _lib.check(
        _lib.load().hg_gmres(
            dop._handle,
            dw._handle if dw is not None else None,
            _vp(r),
            _vp(x0t) if x0t is not None else None,
            _vp(x),
            float(rtol),
            maxit_eff,
            _lib.ptr(hist, ctypes.c_double),
            _lib.ptr(info, ctypes.c_int32),
            _stream(),
        ),
        "hg_gmres",
    )
    it = int(info[0])
    history = hist[: it + 1].copy()
    env, clamped = _envelope(gamma, history[0], it)
    rep = GmresReport(
        iterations=it,
        residual_history=history,
        converged=bool(info[1]),
        elman_envelope=env,
        gamma_used=gamma,
        envelope_clamped=clamped,
        breakdown=bool(info[2]),
        reorth_passes=int(info[3]),
    )
    del keep_op, keep_w
    return (x.cpu().numpy() if was_np else x), rep


def _reports(hist, info, gamma):
    reps = []
    for c in range(info.shape[0]):
        it = int(info[c, 0])
        history = hist[c, : it + 1].copy()
        env, clamped = _envelope(gamma, history[0], it)
        reps.append(GmresReport(
            iterations=it,
            residual_history=history,
            converged=bool(info[c, 1]),
            elman_envelope=env,
            gamma_used=gamma,
            envelope_clamped=clamped,
            breakdown=bool(info[c, 2]),
            reorth_passes=int(info[c, 3]),
        ))
    return reps


def weighted_gmres_batch(op, rhs, weight=None, rtol=1e-6, maxit=200, gamma=None, orth=None):
    """nrhs independent ``weighted_gmres`` solves (x0 = 0) in lock step
    (no reference function — column c is checked against
    ``weighted_gmres(op, rhs[:, c], ...)``).  Every iteration applies ``op``
    once to the whole batch of Krylov vectors; each column keeps its own
    basis, reorthogonalisation decisions, Givens rotations and stopping test.

    rhs: numpy (n, nrhs) or CUDA tensor (nrhs, n).  Returns (X, [GmresReport])
    with X in the layout of rhs."""
    with _orth_mode(orth):
        return _weighted_gmres_batch(op, rhs, weight, rtol, maxit, gamma)


def _weighted_gmres_batch(op, rhs, weight, rtol, maxit, gamma):
    dop, keep_op = _device_op(op)
    dw, keep_w = _device_weight(weight, dop)
    torch = _torch()
    n = dop.n
    R, was_np = _as_device_batch(rhs, n)
    nrhs = R.shape[0]
    X = torch.empty_like(R)
    maxit_eff = int(max(0, min(maxit, n)))
    hist = np.zeros((nrhs, maxit_eff + 1))
    info = np.zeros((nrhs, 4), dtype=np.int32)
    _lib.check(
        _lib.load().hg_gmres_batch(
            dop._handle,
            dw._handle if dw is not None else None,
            _vp(R),
            n,
            _vp(X),
            n,
            nrhs,
            float(rtol),
            maxit_eff,
            _lib.ptr(hist, ctypes.c_double),
            _lib.ptr(info, ctypes.c_int32),
            _stream(),
        ),
        "hg_gmres_batch",
    )
    reps = _reports(hist, info, gamma)
    del keep_op, keep_w
    return _from_device_batch(X, was_np), reps
