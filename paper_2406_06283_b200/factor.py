"""Setup phase, part 4: factorisations and their device layout.

* Local blocks: ``B[idof][:, idof]`` factored by LAPACK ``dgbtrf`` (band LU
  with partial pivoting) instead of the reference's SuperLU
  (schwarz.py:104-131).  Same operator, same pivoting rule; the singular-pivot
  test of schwarz.py:116-121 (smallest |u_jj| <= 1e-12 * ||block||_F) is kept
  and names the (i, j) pair in the error.
* Coarse operator: ``lu_factor(B0)`` (getrf, schwarz.py:88-99) with the same
  pivot check.  The dense factors of the block-sparse B0 are exactly zero
  outside a band; ``pack_b0`` measures that band and stores only it.

Record layout consumed by the band-solve kernel (include/helmgpu.h):
  forward  record j  = [l_{j+1,j}, ..., l_{j+kl,j}, ipiv_j]   (stride even)
  backward record r  = [u_{j-1,j}, ..., u_{j-kv,j}, 1/u_jj],  j = n-1-r
"""

from dataclasses import dataclass

import numpy as np
import scipy.linalg
import scipy.sparse as sp
from scipy.linalg import lapack

from .errors import SingularOperatorError

_SINGULAR_RTOL = 1e-12


@dataclass
class BandLU:
    n: int
    kl: int
    ku: int
    lub: np.ndarray   # LAPACK band storage (2kl+ku+1, n)
    piv: np.ndarray   # 0-based
    norm: float

    @property
    def kv(self):
        return self.kl + self.ku

    def solve(self, b):
        """Host dgbtrs (used for tests of the device kernel)."""
        x, info = lapack.dgbtrs(self.lub, self.kl, self.ku, np.asarray(b, dtype=float), self.piv)
        if info != 0:
            raise ValueError("dgbtrs info=%d" % info)
        return x

    @property
    def u_diagonal(self):
        return self.lub[self.kv]


def submatrix(A, rows, cols):
    """A[rows][:, cols] (CSR) for sorted unique ``cols`` via a column lookup
    table — O(nnz of the selected rows), unlike scipy's column fancy indexing."""
    A = sp.csr_matrix(A)
    rows = np.asarray(rows)
    cols = np.asarray(cols)
    sub = A[rows]
    lut = np.full(A.shape[1], -1, dtype=np.int64)
    lut[cols] = np.arange(cols.size)
    c = lut[sub.indices]
    keep = c >= 0
    counts = np.diff(sub.indptr)
    kc = np.zeros(rows.size, dtype=np.int64)
    nz = counts > 0
    if nz.any():
        kc[nz] = np.add.reduceat(keep.astype(np.int64), sub.indptr[:-1][nz])
    indptr = np.concatenate([[0], np.cumsum(kc)])
    return sp.csr_matrix((sub.data[keep], c[keep], indptr), shape=(rows.size, cols.size))


def block_bandwidth(block):
    coo = sp.coo_matrix(block)
    if coo.nnz == 0:
        return 0
    return int(np.abs(coo.row - coo.col).max())


def band_lu(block, label=None):
    """dgbtrf of a sparse banded block; raises SingularOperatorError on a
    (numerically) singular pivot, naming ``label`` like schwarz.py:111-121."""
    block = sp.csr_matrix(block)
    n = block.shape[0]
    kl = ku = block_bandwidth(block)
    coo = block.tocoo()
    ab = np.zeros((2 * kl + ku + 1, n))
    ab[kl + ku + coo.row - coo.col, coo.col] = coo.data
    lub, piv, info = lapack.dgbtrf(ab, kl, ku)
    norm = float(sp.linalg.norm(block)) if n else 0.0
    where = "fine subdomain (%d, %d)" % label if label is not None else "local block"
    if info > 0:
        raise SingularOperatorError(
            "local Helmholtz block on %s is singular (k^2 equals a local Dirichlet eigenvalue): "
            "zero pivot at %d" % (where, info)
        )
    if info < 0:
        raise ValueError("dgbtrf argument error %d" % info)
    piv_abs = np.abs(lub[kl + ku])
    if n and piv_abs.min() <= _SINGULAR_RTOL * norm:
        raise SingularOperatorError(
            "local Helmholtz block on %s is numerically singular (smallest pivot %.3e)" % (where, piv_abs.min())
        )
    return BandLU(n, kl, ku, lub, piv.astype(np.int64), norm)


def _even(x):
    return x + (x & 1)


MIN_RECORD_WIDTH = 3  # the kernel's replicated front reads the first 3 multipliers


def pack_band_records(f):
    """(fwd records, bwd records, fstride, bstride, kl_rec, kv_rec) for one
    BandLU; widths below MIN_RECORD_WIDTH are zero padded (kl_rec, kv_rec)."""
    n, kl, kv = f.n, f.kl, f.kv
    klp, kvp = max(kl, MIN_RECORD_WIDTH), max(kv, MIN_RECORD_WIDTH)
    fs, bs = _even(klp + 1), _even(kvp + 1)
    fwd = np.zeros((n, fs))
    bwd = np.zeros((n, bs))
    if n == 0:
        return fwd, bwd, fs, bs, klp, kvp
    fwd[:, klp] = f.piv
    if kl:
        L = f.lub[kv + 1 : kv + 1 + kl, :].T.copy()        # L[j, t-1] = l_{j+t, j}
        j = np.arange(n)[:, None]
        t = np.arange(1, kl + 1)[None, :]
        L[j + t >= n] = 0.0
        fwd[:, 0:kl] = L
    jj = n - 1 - np.arange(n)                                # backward order
    bwd[:, kvp] = 1.0 / f.lub[kv, jj]
    if kv:
        U = f.lub[kv - np.arange(1, kv + 1)[:, None], jj[None, :]].T.copy()  # U[r, t-1] = u_{j-t, j}
        U[(jj[:, None] - np.arange(1, kv + 1)[None, :]) < 0] = 0.0
        bwd[:, 0:kv] = U
    return fwd, bwd, fs, bs, klp, kvp


def lu_b0(B0, precomputed=None):
    """Dense LU of the coarse operator with the reference's pivot check
    (schwarz.py:88-99); ``precomputed`` = an existing (lu, piv) of B0."""
    if precomputed is not None:
        lu, piv = precomputed
    else:
        try:
            lu, piv = scipy.linalg.lu_factor(B0)
        except scipy.linalg.LinAlgError as exc:
            raise SingularOperatorError("coarse operator B0: %s" % exc)
    diag = np.abs(np.diag(lu))
    if diag.size and diag.min() <= _SINGULAR_RTOL * np.linalg.norm(B0):
        raise SingularOperatorError(
            "coarse operator B0 is numerically singular; the coarse problem is not well posed at this "
            "wavenumber (the condition sqrt(2) k Lambda^2 sqrt(Theta) (1 + Cstab) < 1 fails)"
        )
    return lu, piv


def perm_from_piv(piv):
    """Row permutation of getrs as a gather: (P c)[i] = c[perm[i]]."""
    m = piv.size
    p = np.arange(m)
    for i in range(m):
        k = piv[i]
        if k != i:
            p[i], p[k] = p[k], p[i]
    return p


def pack_b0(lu, piv, row_block=1024):
    """Band widths and row-major band storage of the getrf factors.

    Returns (perm, kl, ku, lband[m, kl], uband[m, ku+1]) where
    lband[i, t] = L[i, i-kl+t] and uband[i, t] = U[i, i+t].  Every entry of
    the dense factors outside the band is verified to be exactly zero."""
    m = lu.shape[0]
    kl = ku = 0
    for r0 in range(0, m, row_block):
        r1 = min(m, r0 + row_block)
        blk = lu[r0:r1]
        nz = blk != 0.0
        rows = np.arange(r0, r1)[:, None]
        cols = np.arange(m)[None, :]
        low = nz & (cols < rows)
        up = nz & (cols >= rows)
        if low.any():
            kl = max(kl, int((rows - cols)[low].max()))
        if up.any():
            ku = max(ku, int((cols - rows)[up].max()))
    lband = np.zeros((m, kl))
    uband = np.zeros((m, ku + 1))
    for t in range(kl):
        d = kl - t                       # L[i, i-d]
        i = np.arange(d, m)
        lband[i, t] = lu[i, i - d]
    for t in range(ku + 1):
        i = np.arange(0, m - t)
        uband[i, t] = lu[i, i + t]
    return perm_from_piv(np.asarray(piv)), kl, ku, lband, uband
