"""Setup phase, part 3: local H_k-GenEO eigenproblems and the coarse space.

Restates pkg/src/helmdd/eigencoarse.py (pencil 83-101, shifted dense solve
152-217, mode selection 220-245, Z / B0 / rank filter 248-339) plus the
scalable variants SURVEY §8c asks for on the ~1M-dof configs:

* ``solve_indefinite_gevp``  — the reference's dense algorithm (eigh of C,
  gamma doubling under an LDL^T pivot test, LU of B + gamma C, eigh of the
  congruent K = F^T (B + gamma C)^{-1} F), for small subdomains.
* ``solve_gevp_lanczos``     — the same finite spectrum from ARPACK: the
  C-kernel rows Gamma = ovdof \\ idof are eliminated exactly through a sparse
  LU of B + g C, and K = F_I^T [(B + g C)^{-1}]_II F_I is applied
  matrix-free with C_II = F_I F_I^T a banded Cholesky factor.  The shift g
  is chosen near the bottom of the spectrum (not the reference's 2k^2, which
  squeezes the whole finite spectrum into a relative width of ~1e-3 and
  stalls Lanczos); eigenvalues map back as lambda = 1/mu - g exactly as
  eigencoarse.py:195-199 does.
* ``select_modes``           — with ``truncate=True`` implements the capped
  selection of SURVEY D5 (m_i = min(#{lambda < tau}, cap)); without it the
  reference's ModeCapError semantics are kept.
* ``build_coarse_space``     — Z kept as dense per-subdomain blocks on the
  coarse idof (the support of pou * p), B0 = Z^T B Z assembled block by
  block over interacting subdomain pairs, symmetrised, then the reference's
  rank filter.  The rank filter's dense eigh is replaced by a certificate
  (inverse/forward power iteration on the LU of B0) when B0 is large; only
  if the certificate cannot rule out near-null columns is the dense eigh run.
"""

import os
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from .errors import EigensolveError, ModeCapError, SingularOperatorError
from .fem import local_forms_sparse
from .factor import submatrix

_GAMMA_ATTEMPTS = 40
_PIVOT_RTOL = 1e-12


@dataclass(frozen=True)
class LocalGevp:
    subdomain_index: int
    b_mat: object
    c_mat: object
    dk_mat: object
    weights: np.ndarray
    k: float
    idof_in_ov: np.ndarray = None


@dataclass(frozen=True)
class LocalGevpResult:
    """Finite spectrum (ascending) with C-normalised eigenvectors over ovdof.

    ``n_finite`` is the size of the whole finite spectrum; with the Lanczos
    solver only the lowest ``eigenvalues.size`` of them are known
    (``partial`` is then True).
    """

    subdomain_index: int
    eigenvalues: np.ndarray
    eigenvectors: np.ndarray
    n_nonpositive: int
    n_kernel: int
    shift_gamma: float
    partial: bool = False
    n_finite: int = -1


@dataclass(frozen=True)
class ModeSelection:
    m_per_subdomain: list
    tau: float
    theta: float
    overflow: list


@dataclass
class CoarseSpace:
    """Coarse basis and operator B0 = Z^T B Z.

    ``blocks[i]`` = (index array, dense block) with the columns of coarse
    subdomain i restricted to its interior dofs; ``Z`` (sparse CSC, as the
    reference stores it) is built lazily from them.
    """

    blocks: list
    n_dofs: int
    per_subdomain_counts: list
    tau: float
    theta: float
    B0: np.ndarray
    column_meta: list
    removed: list
    _Z: object = field(default=None, repr=False)
    _b0_lu: object = field(default=None, repr=False)

    @property
    def m_total(self):
        return len(self.column_meta)

    @property
    def Z(self):
        if self._Z is None:
            rows, cols, vals = [], [], []
            col0 = 0
            for idx, blk in self.blocks:
                if blk.shape[1] == 0:
                    continue
                r = np.repeat(idx, blk.shape[1])
                c = np.tile(np.arange(col0, col0 + blk.shape[1]), idx.size)
                rows.append(r)
                cols.append(c)
                vals.append(blk.ravel())
                col0 += blk.shape[1]
            if col0:
                Z = sp.csc_matrix(
                    (np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                    shape=(self.n_dofs, col0),
                )
                Z.eliminate_zeros()
            else:
                Z = sp.csc_matrix((self.n_dofs, 0))
            self._Z = Z
        return self._Z


# ---------------------------------------------------------------- pencils


def assemble_local_gevp(i, forms, dec, validate=True, dense=True):
    """Pencil (B_i, C_i = W D_i W) over the active dofs of coarse subdomain i
    (eigencoarse.py:83-101).  ``dense=False`` keeps the matrices sparse."""
    sub = dec.coarse[i]
    if dense:
        from .fem import assemble_local_forms

        A, S = (sp.csr_matrix(x) for x in assemble_local_forms(forms, sub.elements, sub.ovdof))
    else:
        A, S = local_forms_sparse(forms, sub.elements, sub.ovdof)
    k2 = forms.k**2
    b = (A - k2 * S).tocsr()
    dk = (A + k2 * S).tocsr()
    w = sub.pou
    Wd = sp.diags(w)
    c = (Wd @ dk @ Wd).tocsr()
    if dense:
        b, c, dk = b.toarray(), c.toarray(), dk.toarray()
        # the reference scales D elementwise: dk * w[:,None] * w[None,:]
        c = dk * w[:, None] * w[None, :]
        if validate:
            _validate_pencil(i, b, c)
    return LocalGevp(i, b, c, dk, w, forms.k, np.asarray(sub.idof_in_ov))


def _validate_pencil(i, b_mat, c_mat):
    """Reference checks of eigencoarse.py:104-126 (PSD weight, disjoint kernels)."""
    scale_c = np.linalg.norm(c_mat)
    if scale_c == 0.0:
        raise EigensolveError("coarse subdomain %d has an all-zero weight matrix" % i)
    cmin = scipy.linalg.eigvalsh(c_mat, subset_by_index=[0, 0])[0]
    if cmin < -1e-10 * scale_c:
        raise EigensolveError("weight matrix of subdomain %d is not PSD (%.3e)" % (i, cmin))
    smin = np.linalg.svd(np.vstack([b_mat, c_mat]), compute_uv=False)[-1]
    if smin <= 1e-10 * max(np.linalg.norm(b_mat), scale_c):
        raise EigensolveError("pencil of subdomain %d has intersecting kernels (%.3e)" % (i, smin))


def _ldl_min_pivot(mat):
    _, d, _ = scipy.linalg.ldl(mat)
    vals = []
    j, m = 0, d.shape[0]
    while j < m:
        if j + 1 < m and d[j + 1, j] != 0.0:
            vals.extend(np.linalg.eigvalsh(d[j : j + 2, j : j + 2]))
            j += 2
        else:
            vals.append(d[j, j])
            j += 1
    return float(np.abs(vals).min())


def solve_indefinite_gevp(gevp, gamma0=None, max_attempts=_GAMMA_ATTEMPTS, pivot_rtol=_PIVOT_RTOL,
                          c_rank_rtol=1e-12, mu_rtol=1e-12):
    """Dense shifted solve of B p = lambda C p (eigencoarse.py:152-217)."""
    B = np.asarray(gevp.b_mat)
    C = np.asarray(gevp.c_mat)
    n = B.shape[0]
    c_evals, c_vecs = scipy.linalg.eigh(C)
    if c_evals[-1] <= 0.0:
        raise EigensolveError("subdomain %d weight matrix has empty range" % gevp.subdomain_index)
    keep = c_evals > c_rank_rtol * max(c_evals[-1], 0.0)
    F = c_vecs[:, keep] * np.sqrt(c_evals[keep])

    gamma = gamma0 if gamma0 is not None else 2.0 * gevp.k**2
    if gamma <= 0.0:
        gamma = 1.0
    shifted = None
    for _ in range(max_attempts):
        cand = B + gamma * C
        if _ldl_min_pivot(cand) > pivot_rtol * np.linalg.norm(cand):
            shifted = cand
            break
        gamma *= 2.0
    if shifted is None:
        raise EigensolveError("no invertible shift found for subdomain %d" % gevp.subdomain_index)

    X = scipy.linalg.lu_solve(scipy.linalg.lu_factor(shifted), F)
    K = F.T @ X
    mu, U = scipy.linalg.eigh(0.5 * (K + K.T))
    finite = np.abs(mu) > mu_rtol * max(np.abs(mu).max() if mu.size else 0.0, 1e-300)
    mu_f = mu[finite]
    lam = 1.0 / mu_f - gamma
    vecs = (X @ U[:, finite]) / mu_f[None, :]
    vecs = vecs / np.sqrt(np.einsum("ij,ij->j", vecs, C @ vecs))[None, :]
    order = np.argsort(lam, kind="stable")
    lam, vecs = lam[order], vecs[:, order]
    return LocalGevpResult(gevp.subdomain_index, lam, vecs, int(np.sum(lam <= 0.0)), int(n - lam.size),
                           float(gamma), False, int(lam.size))


def _band_cholesky_factor(D):
    """Sparse lower factor L with D = L L^T for a banded SPD sparse matrix."""
    D = sp.csr_matrix(D)
    n = D.shape[0]
    coo = D.tocoo()
    bw = int(np.abs(coo.row - coo.col).max()) if coo.nnz else 0
    ab = np.zeros((bw + 1, n))
    low = coo.row >= coo.col
    ab[(coo.row - coo.col)[low], coo.col[low]] = coo.data[low]
    cb = scipy.linalg.cholesky_banded(ab, lower=True)
    rows, cols, vals = [], [], []
    for d in range(bw + 1):
        j = np.arange(n - d)
        rows.append(j + d)
        cols.append(j)
        vals.append(cb[d, : n - d])
    return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n))


def solve_gevp_lanczos(gevp, n_wanted, shift=None, tol=0.0, ncv=None):
    """Lowest ``n_wanted`` finite eigenpairs of (B, C) by ARPACK.

    With g = -sigma: mu = 1/(lambda + g) are the eigenvalues of
    K = F_I^T [(B + g C)^{-1}]_II F_I, self-adjoint; the largest mu are the
    lowest lambda above -g.  Eigenvectors map back as
    p = (B + g C)^{-1} [F_I u; 0] / mu, then C-normalised (eigencoarse.py:201-204).
    Eigenvalues below -g (mu < 0) are found by asking for the largest
    magnitude; if any appear the shift is widened and the solve repeated.
    """
    B = sp.csr_matrix(gevp.b_mat)
    C = sp.csr_matrix(gevp.c_mat)
    n = B.shape[0]
    I = np.asarray(gevp.idof_in_ov)
    nI = I.size
    if nI == 0:
        raise EigensolveError("subdomain %d weight matrix has empty range" % gevp.subdomain_index)
    n_wanted = int(min(n_wanted, nI))
    CII = C[I][:, I]
    L = _band_cholesky_factor(CII)
    LT = L.T.tocsr()
    g = 2.0 if shift is None else float(shift)
    normB = spla.norm(B)
    for _attempt in range(_GAMMA_ATTEMPTS):
        M = (B + g * C).tocsc()
        try:
            lu = spla.splu(M)
            ok = np.abs(lu.U.diagonal()).min() > _PIVOT_RTOL * spla.norm(M)
        except RuntimeError:
            ok = False
        if not ok:
            g *= 2.0
            continue

        def kmat(u):
            rhs = np.zeros(n)
            rhs[I] = L @ u
            return LT @ lu.solve(rhs)[I]

        op = spla.LinearOperator((nI, nI), matvec=kmat, dtype=float)
        k_ask = min(n_wanted + 1, nI - 1)
        if k_ask < 1 or nI <= 3:
            K = np.column_stack([kmat(e) for e in np.eye(nI)])
            mu, U = np.linalg.eigh(0.5 * (K + K.T))
            order = np.argsort(-np.abs(mu))[:k_ask if k_ask >= 1 else nI]
            mu, U = mu[order], U[:, order]
        else:
            nc = ncv or min(nI, max(2 * k_ask + 1, k_ask + 40))
            # seeded start vector: ARPACK's own default draws from a per-process
            # stream, so results would depend on which pool worker ran which block
            v0 = np.random.default_rng(7919 + gevp.subdomain_index).standard_normal(nI)
            mu, U = spla.eigsh(op, k=k_ask, which="LM", tol=tol, ncv=nc, maxiter=100 * nI, v0=v0)
        if np.any(mu < 0.0):
            # an eigenvalue below -g: widen the shift so the lowest ones are positive
            lam_neg = 1.0 / mu[mu < 0.0] - g
            g = max(2.0 * g, 2.0 * (-lam_neg.min()) + 1.0)
            continue
        lam = 1.0 / mu - g
        order = np.argsort(lam, kind="stable")
        lam, U, mu = lam[order], U[:, order], mu[order]
        rhs = np.zeros((n, lam.size))
        rhs[I] = L @ U
        vecs = lu.solve(rhs) / mu[None, :]
        vecs = vecs / np.sqrt(np.einsum("ij,ij->j", vecs, C @ vecs))[None, :]
        return LocalGevpResult(gevp.subdomain_index, lam, vecs, int(np.sum(lam <= 0.0)), int(n - nI),
                               float(g), True, int(nI))
    raise EigensolveError("no invertible shift found for subdomain %d" % gevp.subdomain_index)


# ---------------------------------------------------------------- selection


def select_modes(results, tau_target, caps=None, truncate=False):
    """m_i = #{finite eigenvalues < tau_target} (eigencoarse.py:220-245).

    ``truncate=False`` raises ModeCapError above a cap, as the reference does;
    ``truncate=True`` keeps the lowest ``cap`` modes instead.  A
    partial (Lanczos) spectrum is exact for this purpose as long as it holds
    at least cap + 1 eigenvalues or all eigenvalues below tau.
    """
    if tau_target <= 0.0:
        raise ValueError("tau_target must be positive, got %g" % tau_target)
    m_per, overflow = [], []
    tau = np.inf
    for idx, res in enumerate(results):
        ev = res.eigenvalues
        m = int(np.searchsorted(ev, tau_target, side="left"))
        known_all = (not res.partial) or ev.size >= res.n_finite
        if m == ev.size and not known_all:
            # every known eigenvalue is below tau: the true count is >= ev.size
            if caps is None or not truncate or caps[idx] >= ev.size:
                raise EigensolveError(
                    "subdomain %d: partial spectrum (%d of %d) does not reach tau=%g"
                    % (idx, ev.size, res.n_finite, tau_target)
                )
        if caps is not None and m > caps[idx]:
            if not truncate:
                raise ModeCapError(idx, m, caps[idx])
            m = int(caps[idx])
        m_per.append(m)
        if m >= ev.size and known_all:
            overflow.append(idx)
        else:
            tau = min(tau, float(ev[m]))
    theta = 0.0 if np.isinf(tau) else 1.0 / tau
    return ModeSelection(m_per, float(tau), theta, overflow)


# ---------------------------------------------------------------- coarse space


def _interaction_pairs(forms, index_sets):
    n = forms.n_dofs
    rows = np.concatenate([idx for idx in index_sets]) if index_sets else np.zeros(0, int)
    cols = np.concatenate([np.full(idx.size, i) for i, idx in enumerate(index_sets)]) if index_sets else rows
    P = sp.csr_matrix((np.ones(rows.size), (rows, cols)), shape=(n, len(index_sets)))
    Bp = abs(forms.helmholtz)
    pat = (P.T @ Bp @ P).tocoo()
    return sorted(zip(pat.row.tolist(), pat.col.tolist()))


def _sym_extreme_certificate(B0, rtol):
    """True when |lambda|_min(B0) > rtol * |lambda|_max(B0) with a wide margin.

    Power iteration on B0 (largest |lambda|) and on B0^{-1} through its LU
    (smallest |lambda|); both converge from below/above so the estimate is
    only trusted with a 1e4 safety factor.
    """
    m = B0.shape[0]
    rng = np.random.default_rng(1)
    x = rng.standard_normal(m)
    lmax = 0.0
    for _ in range(60):
        y = B0 @ x
        lmax = np.linalg.norm(y) / np.linalg.norm(x)
        x = y / np.linalg.norm(y)
    lu = scipy.linalg.lu_factor(B0)
    x = rng.standard_normal(m)
    inv_max = 0.0
    for _ in range(60):
        y = scipy.linalg.lu_solve(lu, x)
        inv_max = np.linalg.norm(y) / np.linalg.norm(x)
        x = y / np.linalg.norm(y)
    return (1.0 / inv_max) > 1e6 * rtol * lmax, lu


def _near_null_columns(mat):
    """Reference rank filter step (eigencoarse.py:324-339)."""
    vals, vecs = scipy.linalg.eigh(mat)
    scale = np.abs(vals).max()
    small = np.flatnonzero(np.abs(vals) <= _PIVOT_RTOL * scale)
    drop = []
    for j in small:
        pos = int(np.abs(vecs[:, j]).argmax())
        if pos not in drop:
            drop.append(pos)
    return drop


def device_available():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def coarse_operator_device(forms, blocks, pairs, certificate_iters=60):
    """B0 = 0.5 (Z^T B Z + (Z^T B Z)^T), its getrf factors and the rank
    certificate's two estimates, computed on the device (hg_coarse_setup,
    csrc/hg_coarse_setup.cu; eigencoarse.py:286-287, schwarz.py:90).
    Returns (B0, (lu, piv), info, (lambda_max, ||B0^-1||))."""
    import ctypes

    from . import _lib

    B = sp.csr_matrix(forms.helmholtz)
    B.sort_indices()
    n = B.shape[0]
    nb = len(blocks)
    m = sum(b.shape[1] for _, b in blocks)
    keep = []

    def arr(a, dtype, ctype):
        a = np.ascontiguousarray(a, dtype=dtype)
        keep.append(a)
        return _lib.ptr(a, ctype)

    i32, i64, f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    d = _lib.HgPrecondDesc()
    d.n, d.nnz = n, B.nnz
    d.indptr = arr(B.indptr, np.int32, i32)
    d.indices = arr(B.indices, np.int32, i32)
    d.b_data = arr(B.data, np.float64, f64)
    d.m, d.n_cblk = m, nb
    d.cblk_n = arr([i.size for i, _ in blocks], np.int32, i32)
    d.cblk_m = arr([b.shape[1] for _, b in blocks], np.int32, i32)
    d.cblk_idx_off = arr(np.concatenate([[0], np.cumsum([i.size for i, _ in blocks])]), np.int64, i64)
    d.cblk_idx = arr(np.concatenate([i for i, _ in blocks]), np.int32, i32)
    d.cblk_z_off = arr(np.concatenate([[0], np.cumsum([b.size for _, b in blocks])[:-1]]), np.int64, i64)
    z = np.concatenate([b.ravel() for _, b in blocks])
    d.z_len = z.size
    d.z_data = arr(z, np.float64, f64)
    nbr = [[] for _ in range(nb)]
    for a, b in pairs:
        if blocks[a][1].shape[1] and blocks[b][1].shape[1]:
            nbr[b].append(a)
    pair_ptr = np.concatenate([[0], np.cumsum([len(x) for x in nbr])]).astype(np.int32)
    pair_blk = np.asarray([a for x in nbr for a in x] or [0], dtype=np.int32)
    B0 = np.empty((m, m))
    lu = np.empty((m, m))
    piv = np.empty(m, dtype=np.int32)
    info = np.zeros(1, dtype=np.int32)
    cert = np.zeros(2)
    _lib.check(_lib.load().hg_coarse_setup(ctypes.byref(d), _lib.ptr(pair_ptr, i32), _lib.ptr(pair_blk, i32),
                                           _lib.ptr(B0, f64), _lib.ptr(lu, f64), _lib.ptr(piv, i32),
                                           _lib.ptr(info, i32), _lib.ptr(cert, f64), int(certificate_iters)),
               "hg_coarse_setup")
    return B0, (lu, piv.astype(np.int64)), int(info[0]), (float(cert[0]), float(cert[1]))


def build_coarse_space(results, selection, dec, forms, dense_rank_filter_max=3000, device=None):
    """Z blocks and B0 = Z^T B Z, symmetrised and rank filtered (eigencoarse.py:248-321).

    ``device``: build B0, its LU and the rank certificate on the GPU
    (coarse_operator_device); None = when a CUDA device is present and the
    coarse space is large (m > dense_rank_filter_max), HG_HOST_SETUP=1 forces
    the host."""
    n = forms.n_dofs
    blocks, meta = [], []
    for res, m, sub in zip(results, selection.m_per_subdomain, dec.coarse):
        idof = np.asarray(sub.idof)
        pos = np.asarray(sub.idof_in_ov)
        blk = sub.pou[pos][:, None] * res.eigenvectors[pos, :m]
        blocks.append((idof, np.ascontiguousarray(blk)))
        meta.extend((res.subdomain_index, ell) for ell in range(m))
    m_total = len(meta)
    counts = [b.shape[1] for _, b in blocks]
    if m_total == 0:
        return CoarseSpace(blocks, n, counts, selection.tau, selection.theta, np.zeros((0, 0)), [], [])

    offs = np.concatenate([[0], np.cumsum(counts)])
    pairs = _interaction_pairs(forms, [idx for idx, _ in blocks])
    if device is None:
        device = (m_total > dense_rank_filter_max and device_available()
                  and os.environ.get("HG_HOST_SETUP", "0") != "1")
    keep = list(range(m_total))
    removed = []
    certified = False
    b0_lu = None
    import time

    t0 = time.perf_counter()
    if device:
        B0, lu_piv, info, (lmax, inv_max) = coarse_operator_device(forms, blocks, pairs)
        if info == 0:
            b0_lu = lu_piv
            if m_total > dense_rank_filter_max:  # coarse._sym_extreme_certificate's test
                certified = (1.0 / inv_max) > 1e6 * _PIVOT_RTOL * lmax
    else:
        B0 = np.zeros((m_total, m_total))
        B = forms.helmholtz
        for a, b in pairs:
            if counts[a] == 0 or counts[b] == 0:
                continue
            ia, za = blocks[a]
            ib, zb = blocks[b]
            Bab = submatrix(B, ia, ib)
            B0[offs[a]:offs[a + 1], offs[b]:offs[b + 1]] = za.T @ (Bab @ zb)
        B0 = 0.5 * (B0 + B0.T)
        if m_total > dense_rank_filter_max:
            certified, b0_lu = _sym_extreme_certificate(B0, _PIVOT_RTOL)
    if not certified:
        while keep:
            drop = _near_null_columns(B0[np.ix_(keep, keep)])
            if not drop:
                break
            for p in sorted(drop, reverse=True):
                removed.append(meta[keep[p]])
                del keep[p]
        if not keep:
            raise SingularOperatorError(
                "coarse operator is singular for every basis subset; the coarse problem is not well posed"
            )
    if removed:
        B0 = B0[np.ix_(keep, keep)]
        kept = set(keep)
        new_blocks = []
        for i, (idx, blk) in enumerate(blocks):
            cols = [c for c in range(counts[i]) if (offs[i] + c) in kept]
            new_blocks.append((idx, np.ascontiguousarray(blk[:, cols])))
        blocks = new_blocks
        meta = [meta[i] for i in keep]
        counts = [b.shape[1] for _, b in blocks]
    cs = CoarseSpace(blocks, n, counts, selection.tau, selection.theta, B0, meta, removed)
    cs.build_seconds = {"operator_lu_certificate" if device else "operator_certificate": time.perf_counter() - t0,
                        "device": bool(device)}
    if b0_lu is not None and not removed:
        cs._b0_lu = b0_lu  # getrf of B0 already computed by the certificate; factorize reuses it
    return cs


def spectrum_rows(results, selection):
    rows = []
    for res, m in zip(results, selection.m_per_subdomain):
        for ell, lam in enumerate(res.eigenvalues):
            rows.append((res.subdomain_index, ell, float(lam), int(ell < m)))
    return rows
