"""Drop-in GPU replacement of ``helmdd.schwarz.factorize`` and the
``TwoLevelPreconditioner`` it returns (pkg/src/helmdd/schwarz.py:37-101).

``factorize(forms, dec, coarse=None)`` accepts either this package's setup
objects or the reference's own (duck-typed: ``forms.helmholtz``,
``forms.dk``, ``dec.fine_flat()``, ``dec.coarse[i].idof``, ``coarse.Z``,
``coarse.B0``, ``coarse.column_meta``).  The factorisations happen on the
host (setup phase); everything the apply touches is uploaded once into a
device-resident handle of libhelmgpu.so, and every apply runs there.

Inputs to ``apply`` / ``apply_T`` / ``apply_coarse`` may be numpy arrays
(copied to the device and the result copied back, like the reference's
return type) or CUDA torch tensors (result stays on the device).  There is
no CPU path: without the library or a GPU the calls raise.
"""

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import scipy.linalg
import scipy.sparse as sp

from . import _lib
from .errors import SingularOperatorError
from .factor import (band_lu, lu_b0, pack_b0_tiles, pack_band_records, record_floor, submatrix, swizzle_tile_rows,
                     tile_span)

_DENSE_EIG_LIMIT = 1500


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2406_06283_b200: a CUDA device is required (no CPU fallback)")
    return torch


def _stream():
    return ctypes.c_void_p(_torch().cuda.current_stream().cuda_stream)


def _as_device(v, n):
    """(device tensor, was_numpy) for a numpy array or CUDA tensor of length n."""
    torch = _torch()
    if isinstance(v, torch.Tensor):
        t = v.detach()
        if t.device.type != "cuda":
            t = t.cuda()
        t = t.to(torch.float64).contiguous()
        if t.numel() != n:
            raise ValueError("vector has length %d, operator has %d" % (t.numel(), n))
        return t.reshape(n), False
    a = np.ascontiguousarray(np.asarray(v, dtype=np.float64)).reshape(-1)
    if a.size != n:
        raise ValueError("vector has length %d, operator has %d" % (a.size, n))
    return torch.from_numpy(a).cuda(), True


def _vp(t):
    return ctypes.c_void_p(t.data_ptr())


def _as_device_batch(V, n):
    """(device tensor of shape (nrhs, n), was_numpy) for a batch of vectors.

    numpy input is an (n, nrhs) matrix (scipy's column convention; 1-D =
    one column); a CUDA tensor is taken as (nrhs, n) — column c contiguous,
    i.e. a column-major (n, nrhs) matrix — which is the device layout."""
    torch = _torch()
    if isinstance(V, torch.Tensor):
        t = V.detach()
        if t.device.type != "cuda":
            t = t.cuda()
        t = t.to(torch.float64)
        if t.ndim == 1:
            t = t.reshape(1, -1)
        t = t.contiguous()
        if t.shape[1] != n:
            raise ValueError("batch has vectors of length %d, operator has %d" % (t.shape[1], n))
        was_np = False
    else:
        a = np.asarray(V, dtype=np.float64)
        if a.ndim == 1:
            a = a[:, None]
        if a.shape[0] != n:
            raise ValueError("batch has %d rows, operator has %d" % (a.shape[0], n))
        t = torch.from_numpy(np.ascontiguousarray(a.T)).cuda()
        was_np = True
    if not 1 <= t.shape[0] <= _lib.MAX_RHS:
        raise ValueError("batch of %d columns; 1..%d supported per call" % (t.shape[0], _lib.MAX_RHS))
    return t, was_np


def _from_device_batch(t, was_np):
    return t.cpu().numpy().T.copy() if was_np else t


class GpuBandLU:
    """``LocalSolver.lu`` stand-in: ``solve`` runs the device band solve of
    one block (hg_local_solve); the host factors stay available for tests."""

    def __init__(self, precond, index, host_factor):
        self._p = precond
        self._s = index
        self.host = host_factor
        self.shape = (host_factor.n, host_factor.n)

    def solve(self, rhs):
        torch = _torch()
        t, was_np = _as_device(rhs, self.host.n)
        out = torch.empty_like(t)
        _lib.check(
            _lib.load().hg_local_solve(self._p._handle, self._s, _vp(t), _vp(out), _stream()), "hg_local_solve"
        )
        return out.cpu().numpy() if was_np else out


class LocalSolver:
    """Mirror of schwarz.LocalSolver (schwarz.py:26-34); ``min_eig`` and
    ``spd_flag`` are computed lazily (they only feed reports)."""

    def __init__(self, coarse_index, fine_index, idof, lu, diameter, block):
        self.coarse_index = coarse_index
        self.fine_index = fine_index
        self.idof = idof
        self.lu = lu
        self.diameter = diameter
        self._block = block
        self._min_eig = None

    @property
    def min_eig(self):
        if self._min_eig is None:
            self._min_eig = _smallest_eigenvalue(self._block) if self.idof.size else np.inf
        return self._min_eig

    @property
    def spd_flag(self):
        return bool(self.min_eig > 0.0)


def _smallest_eigenvalue(block):
    """schwarz.py:134-145."""
    import scipy.sparse.linalg as spla

    m = block.shape[0]
    if m <= _DENSE_EIG_LIMIT:
        return float(scipy.linalg.eigvalsh(block.toarray(), subset_by_index=[0, 0])[0])
    try:
        return float(spla.eigsh(block.asfptype(), k=1, which="SA", maxiter=5000, return_eigenvectors=False)[0])
    except Exception:
        return float(scipy.linalg.eigvalsh(block.toarray())[0])


def _common_pattern(B, Dk):
    """B and D_k on the union of their patterns (explicit zeros kept), so the
    device holds one index structure for both (scipy's A - k^2 S may prune an
    exactly cancelling entry)."""
    out = []
    cb, cd = B.tocoo(), Dk.tocoo()
    rows = np.concatenate([cb.row, cd.row])
    cols = np.concatenate([cb.col, cd.col])
    for vals in (
        np.concatenate([cb.data, np.zeros(cd.nnz)]),
        np.concatenate([np.zeros(cb.nnz), cd.data]),
    ):
        M = sp.coo_matrix((vals, (rows, cols)), shape=B.shape).tocsr()
        M.sort_indices()
        out.append(M)
    if not np.array_equal(out[0].indices, out[1].indices):
        raise ValueError("B and D_k patterns could not be aligned")
    return out[0], out[1]


def coarse_blocks(coarse, dec):
    """Per-subdomain dense Z blocks [(index array, n_i x m_i block)] in column order."""
    if hasattr(coarse, "blocks"):
        return [(np.asarray(i), np.ascontiguousarray(b)) for i, b in coarse.blocks]
    Z = sp.csc_matrix(coarse.Z)
    meta = list(coarse.column_meta)
    out = []
    col = 0
    for i, sub in enumerate(dec.coarse):
        cols = []
        while col < len(meta) and meta[col][0] == i:
            cols.append(col)
            col += 1
        idof = np.asarray(sub.idof)
        if not cols:
            out.append((idof, np.zeros((idof.size, 0))))
            continue
        Zi = Z[:, cols]
        blk = Zi[idof].toarray()
        if Zi.nnz != np.count_nonzero(blk):
            raise ValueError("coarse columns of subdomain %d are not supported on its interior dofs" % i)
        out.append((idof, blk))
    if col != len(meta):
        raise ValueError("coarse.column_meta is not grouped by subdomain in ascending order")
    return out


class TwoLevelPreconditioner:
    """Device-resident M^{-1} r = Z B0^{-1} Z^T r + sum_s E_s B_s^{-1} R_s r."""

    def __init__(self, forms, dec, coarse=None, b0_lu=None):
        self.forms = forms
        self.n = forms.n_dofs if hasattr(forms, "n_dofs") else forms.helmholtz.shape[0]
        self._handle = None
        self._keep = []
        self.Z = None
        self.b0_piv = None
        B = sp.csr_matrix(forms.helmholtz)
        B.sort_indices()
        Dk = sp.csr_matrix(forms.dk) if getattr(forms, "dk", None) is not None else None
        if Dk is not None:
            Dk.sort_indices()
            if not (np.array_equal(Dk.indptr, B.indptr) and np.array_equal(Dk.indices, B.indices)):
                B, Dk = _common_pattern(B, Dk)
        self._B = B
        self._Dk = Dk

        # ---- local factorisations (schwarz.py:83-85, 104-131)
        self.local_solvers = []
        factors = []
        for i, j, sub in dec.fine_flat():
            idof = np.asarray(sub.idof)
            block = submatrix(B, idof, idof) if idof.size else sp.csr_matrix((0, 0))
            if idof.size:
                f = band_lu(block, label=(i, j))
            else:
                f = band_lu(sp.csr_matrix((0, 0)))
            factors.append((idof, f))
            self.local_solvers.append(LocalSolver(i, j, idof, None, getattr(sub, "diameter", np.nan), block))

        # ---- coarse operator (schwarz.py:87-100)
        cblocks = []
        lu = piv = None
        if coarse is not None and coarse.m_total > 0:
            if b0_lu is None:
                b0_lu = getattr(coarse, "_b0_lu", None)
            lu, piv = lu_b0(np.asarray(coarse.B0), b0_lu)
            self.b0_piv = (lu, piv)
            self.Z = coarse.Z if not hasattr(coarse, "blocks") else None
            self._coarse = coarse
            cblocks = coarse_blocks(coarse, dec)
        self._upload(B, Dk, factors, cblocks, lu, piv)
        for s, ls in enumerate(self.local_solvers):
            ls.lu = GpuBandLU(self, s, factors[s][1])

    # ------------------------------------------------------------------ upload
    def _upload(self, B, Dk, factors, cblocks, lu, piv):
        keep = self._keep
        lib = _lib.load()
        _torch()  # CUDA context present before the first allocation
        d = _lib.HgPrecondDesc()
        i32, i64, f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_double

        def arr(a, dtype, ctype):
            a = np.ascontiguousarray(a, dtype=dtype)
            keep.append(a)
            return _lib.ptr(a, ctype)

        d.n = self.n
        d.nnz = B.nnz
        d.indptr = arr(B.indptr, np.int32, i32)
        d.indices = arr(B.indices, np.int32, i32)
        d.b_data = arr(B.data, np.float64, f64)
        d.dk_data = arr(Dk.data, np.float64, f64) if Dk is not None else None

        ns, kls, kvs, fss, bss = [], [], [], [], []
        idx_off = [0]
        fwd_parts, bwd_parts, foff, boff = [], [], [], []
        fpos = bpos = 0
        kl_floor = record_floor(max([f.kl for _, f in factors], default=0))
        kv_floor = record_floor(max([f.kv for _, f in factors], default=0))
        for idof, f in factors:
            fw, bw, fs, bs, klp, kvp = pack_band_records(f, kl_floor, kv_floor)
            ns.append(f.n)
            kls.append(klp)
            kvs.append(kvp)
            fss.append(fs)
            bss.append(bs)
            idx_off.append(idx_off[-1] + idof.size)
            foff.append(fpos)
            boff.append(bpos)
            fwd_parts.append(fw.ravel())
            bwd_parts.append(bw.ravel())
            fpos += fw.size
            bpos += bw.size
        fwd = np.concatenate(fwd_parts) if fwd_parts else np.zeros(0)
        bwd = np.concatenate(bwd_parts) if bwd_parts else np.zeros(0)
        d.n_local = len(factors)
        d.local_n = arr(ns, np.int32, i32)
        d.local_kl = arr(kls, np.int32, i32)
        d.local_kv = arr(kvs, np.int32, i32)
        d.local_fstride = arr(fss, np.int32, i32)
        d.local_bstride = arr(bss, np.int32, i32)
        d.local_idx_off = arr(idx_off, np.int64, i64)
        d.local_idx = arr(np.concatenate([i for i, _ in factors]) if factors else np.zeros(0), np.int32, i32)
        d.local_fwd_off = arr(foff, np.int64, i64)
        d.local_fwd_len = fwd.size
        d.local_fwd = arr(fwd, np.float64, f64)
        d.local_bwd_off = arr(boff, np.int64, i64)
        d.local_bwd_len = bwd.size
        d.local_bwd = arr(bwd, np.float64, f64)

        m = sum(b.shape[1] for _, b in cblocks)
        d.m = m
        self.m = m
        self.local_sizes = ns
        self.cblock_shapes = [b.shape for _, b in cblocks]
        self.b0_bytes = 0
        if m:
            P = int(os.environ.get("HG_B0_PANEL", "64"))
            T = pack_b0_tiles(lu, piv, P)
            # coarse-solve kernel: one DSMEM cluster when the x ring fits in shared memory
            cs = min(16, T.K)
            ring = tile_span(T) + cs + 1
            mode = int(os.environ.get("HG_B0_MODE", "1"))
            if mode == 1 and (T.P != 64 or ring > 96):  # the tagged x ring must fit in shared memory
                mode = 0
            if mode == 1:
                T = T.premultiply()  # tiles D_t^{-1} T[t, j]: rows of a panel finish independently
            # guard: the tiled algorithm (inverted diagonal blocks) must agree with getrs
            c = np.random.default_rng(0).standard_normal(m)
            want = scipy.linalg.lu_solve((lu, piv), c)
            dev = float(np.abs(T.solve(c) - want).max() / max(np.abs(want).max(), 1e-300))
            if dev > 1e-11:
                raise SingularOperatorError(
                    "coarse tile factorisation deviates from getrs by %.2e (B0 too ill-conditioned for "
                    "inverted %dx%d diagonal blocks)" % (dev, P, P))
            self.b0_tiles = T
            self.b0_tile_dev = dev
            self.b0_bytes = T.nbytes + 4 * m + 4 * T.tile_col.size
            # dense mode: B0^{-1} applied as a streaming GEMV / DMMA GEMM beside the
            # local solves; kept only if it agrees with getrs (the reference's lu_solve)
            self.b0_dense = False
            self.b0_dense_dev = None
            dense = os.environ.get("HG_B0_DENSE", "0")  # measured slower by default: see DESIGN.md section 8
            if dense == "1" or (dense == "auto" and m <= 20000):  # "auto": whenever it fits
                torch = _torch()
                B0 = np.ascontiguousarray(np.asarray(self._coarse.B0), dtype=np.float64)
                Binv = torch.linalg.inv(torch.from_numpy(B0).cuda())
                Binv = np.ascontiguousarray(Binv.cpu().numpy())
                rng = np.random.default_rng(1)
                ddev = 0.0
                for _ in range(2):
                    c = rng.standard_normal(m)
                    want = scipy.linalg.lu_solve((lu, piv), c)
                    ddev = max(ddev, float(np.abs(Binv @ c - want).max() / max(np.abs(want).max(), 1e-300)))
                self.b0_dense_dev = ddev
                if ddev <= 1e-11:
                    self.b0_dense = True
                    d.b0_inv = arr(Binv, np.float64, f64)
                    self.b0_bytes = 8 * m * m + 16 * m
            d.n_cblk = len(cblocks)
            d.cblk_n = arr([i.size for i, _ in cblocks], np.int32, i32)
            d.cblk_m = arr([b.shape[1] for _, b in cblocks], np.int32, i32)
            d.cblk_idx_off = arr(np.concatenate([[0], np.cumsum([i.size for i, _ in cblocks])]), np.int64, i64)
            d.cblk_idx = arr(np.concatenate([i for i, _ in cblocks]), np.int32, i32)
            zsizes = [b.size for _, b in cblocks]
            d.cblk_z_off = arr(np.concatenate([[0], np.cumsum(zsizes)[:-1]]), np.int64, i64)
            z = np.concatenate([b.ravel() for _, b in cblocks])
            d.z_len = z.size
            d.z_data = arr(z, np.float64, f64)
            d.b0_perm = arr(T.perm, np.int32, i32)
            d.b0_panel = T.P
            d.b0_npanel = T.K
            d.b0_tile_ptr = arr(T.tile_ptr, np.int64, i64)
            d.b0_tile_col = arr(T.tile_col if T.tile_col.size else np.zeros(1), np.int32, i32)
            d.b0_ntile = int(T.tile_col.size)
            d.b0_ctas = int(os.environ.get("HG_B0_CTAS", "0"))
            self.b0_mode = mode
            if mode == 1:
                d.b0_mode, d.b0_cluster, d.b0_ring = 1, cs, ring
                dinv = swizzle_tile_rows(T.dinv)
                tiles = swizzle_tile_rows(T.tiles) if T.tiles.size else np.zeros(1)
            else:
                d.b0_mode, d.b0_cluster, d.b0_ring = 0, 0, 0
                dinv, tiles = T.dinv, (T.tiles if T.tiles.size else np.zeros(1))
            d.b0_dinv = arr(dinv, np.float64, f64)
            d.b0_tiles = arr(tiles, np.float64, f64)
        h = ctypes.c_void_p()
        _lib.check(lib.hg_precond_create(ctypes.byref(d), ctypes.byref(h)), "hg_precond_create")
        self._handle = h
        self._keep = []  # host copies no longer needed
        self.local_bands = [(f.kl, f.kv) for _, f in factors]

    # ------------------------------------------------------------------ API
    @property
    def has_coarse(self):
        return self.b0_piv is not None

    @property
    def device_bytes(self):
        return int(_lib.load().hg_precond_device_bytes(self._handle))

    def check(self):
        """Raise DeviceError if a device-side wait of this handle timed out or
        an apply failed part-way (hg_precond_status; the handle is then
        poisoned).  Numpy-returning calls check after their copy back; for
        device-tensor results call this after synchronising."""
        _lib.check(_lib.load().hg_precond_status(self._handle), "hg_precond_status")

    def _run(self, fn, v):
        torch = _torch()
        t, was_np = _as_device(v, self.n)
        out = torch.empty_like(t)
        _lib.check(getattr(_lib.load(), fn)(self._handle, _vp(t), _vp(out), _stream()), fn)
        if was_np:
            res = out.cpu().numpy()
            self.check()
            return res
        return out

    def apply(self, r):
        """M^{-1} r (schwarz.py:51-61); returns a new array."""
        return self._run("hg_precond_apply", r)

    def apply_multi(self, R):
        """M^{-1} applied to every column of R in ONE batched apply (SURVEY §8a
        row a15; column c equals ``apply(R[:, c])`` to rounding).  numpy R is
        (n, nrhs); a CUDA tensor is (nrhs, n) and the result stays on device."""
        torch = _torch()
        t, was_np = _as_device_batch(R, self.n)
        out = torch.empty_like(t)
        _lib.check(
            _lib.load().hg_precond_apply_multi(self._handle, _vp(t), self.n, _vp(out), self.n, t.shape[0], _stream()),
            "hg_precond_apply_multi",
        )
        res = _from_device_batch(out, was_np)
        if was_np:
            self.check()
        return res

    def profile_multi(self, R, iters=5):
        """Mean device ms per stage of the batched apply (stages serialised)."""
        torch = _torch()
        t, _ = _as_device_batch(R, self.n)
        out = torch.empty_like(t)
        ms = np.zeros(len(self.STAGES))
        _lib.check(
            _lib.load().hg_precond_profile_multi(self._handle, _vp(t), self.n, _vp(out), self.n, t.shape[0],
                                                 int(iters), _lib.ptr(ms, ctypes.c_double), _stream()),
            "hg_precond_profile_multi",
        )
        return dict(zip(self.STAGES, ms.tolist()))

    def apply_T(self, u):
        """T u = M^{-1} B u (schwarz.py:63-65)."""
        return self._run("hg_precond_apply_T", u)

    def apply_coarse(self, r):
        """Z B0^{-1} Z^T r (schwarz.py:67-71)."""
        return self._run("hg_precond_apply_coarse", r)

    def spmv(self, x, which="B"):
        torch = _torch()
        t, was_np = _as_device(x, self.n)
        out = torch.empty_like(t)
        _lib.check(
            _lib.load().hg_precond_spmv(self._handle, 0 if which == "B" else 1, _vp(t), _vp(out), _stream()),
            "hg_precond_spmv",
        )
        return out.cpu().numpy() if was_np else out

    STAGES = ("zt", "b0_solve", "zy", "local", "assemble")

    def profile(self, r, iters=10):
        """Mean device ms per apply stage, stages serialised (hg_precond_profile)."""
        torch = _torch()
        t, _ = _as_device(r, self.n)
        out = torch.empty_like(t)
        ms = np.zeros(len(self.STAGES))
        _lib.check(
            _lib.load().hg_precond_profile(self._handle, _vp(t), _vp(out), int(iters),
                                           _lib.ptr(ms, ctypes.c_double), _stream()),
            "hg_precond_profile",
        )
        return dict(zip(self.STAGES, ms.tolist()))

    def as_operator(self, kind="T"):
        """Device operator for weighted_gmres: "T" = M^{-1} B (cli.py:298),
        "M" = M^{-1}, "B" = B, "Dk" = D_k."""
        return DeviceOperator(self, {"M": 0, "T": 1, "B": 2, "Dk": 3}[kind])

    def solve_host(self, f, rtol=1e-6, maxit=200):
        """End-to-end solve through the C ABI with host buffers (hg_solve_host):
        rhs_p = M^{-1} f, x = GMRES(M^{-1} B, rhs_p, weight D_k)."""
        from .wgmres import GmresReport

        f = np.ascontiguousarray(np.asarray(f, dtype=np.float64))
        x = np.empty_like(f)
        maxit = int(min(maxit, self.n))
        hist = np.zeros(maxit + 1)
        info = np.zeros(4, dtype=np.int32)
        _lib.check(
            _lib.load().hg_solve_host(
                self._handle, _lib.ptr(f, ctypes.c_double), _lib.ptr(x, ctypes.c_double), float(rtol), maxit,
                _lib.ptr(hist, ctypes.c_double), _lib.ptr(info, ctypes.c_int32), _stream(),
            ),
            "hg_solve_host",
        )
        it = int(info[0])
        rep = GmresReport(iterations=it, residual_history=hist[: it + 1].copy(), converged=bool(info[1]),
                          breakdown=bool(info[2]))
        rep.reorth_passes = int(info[3])
        return x, rep

    def solve_host_batch(self, F, rtol=1e-6, maxit=200):
        """Batched end-to-end solve through the C ABI with host buffers
        (hg_solve_host_batch): F is (n, nrhs); returns (X, [GmresReport])."""
        from .wgmres import _reports

        F = np.asarray(F, dtype=np.float64)
        if F.ndim == 1:
            F = F[:, None]
        nrhs = F.shape[1]
        if not 1 <= nrhs <= _lib.MAX_RHS:
            raise ValueError("batch of %d columns; 1..%d supported per call" % (nrhs, _lib.MAX_RHS))
        Fc = np.ascontiguousarray(F.T)
        Xc = np.empty_like(Fc)
        maxit = int(min(maxit, self.n))
        hist = np.zeros((nrhs, maxit + 1))
        info = np.zeros((nrhs, 4), dtype=np.int32)
        _lib.check(
            _lib.load().hg_solve_host_batch(
                self._handle, _lib.ptr(Fc, ctypes.c_double), _lib.ptr(Xc, ctypes.c_double), nrhs, float(rtol),
                maxit, _lib.ptr(hist, ctypes.c_double), _lib.ptr(info, ctypes.c_int32), _stream(),
            ),
            "hg_solve_host_batch",
        )
        return Xc.T.copy(), _reports(hist, info, None)

    def close(self):
        if self._handle is not None:
            _lib.load().hg_precond_destroy(self._handle)
            self._handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DeviceOperator:
    """A linear operator that lives on the device (an HgOp)."""

    def __init__(self, precond, mode):
        self.precond = precond
        self.mode = mode
        self.n = precond.n
        h = ctypes.c_void_p()
        _lib.check(_lib.load().hg_op_create_precond(precond._handle, mode, ctypes.byref(h)), "hg_op_create_precond")
        self._handle = h

    def __call__(self, v):
        torch = _torch()
        t, was_np = _as_device(v, self.n)
        out = torch.empty_like(t)
        _lib.check(_lib.load().hg_op_apply(self._handle, _vp(t), _vp(out), _stream()), "hg_op_apply")
        if was_np:
            res = out.cpu().numpy()
            self.precond.check()
            return res
        return out

    def basis(self, nv, col=0):
        """The first nv Krylov basis vectors of column col of the last GMRES
        solve on this operator, as an (nv, n) CUDA tensor (inspection hook)."""
        return _basis(self._handle, self.n, col, nv)

    def release(self):
        """Free this operator's Krylov bases / GMRES workspaces (hg_op_release)."""
        _lib.check(_lib.load().hg_op_release(self._handle), "hg_op_release")

    def apply_multi(self, V):
        """op applied to every column of a batch (numpy (n, nrhs) or CUDA (nrhs, n))."""
        torch = _torch()
        t, was_np = _as_device_batch(V, self.n)
        out = torch.empty_like(t)
        _lib.check(
            _lib.load().hg_op_apply_multi(self._handle, _vp(t), self.n, _vp(out), self.n, t.shape[0], _stream()),
            "hg_op_apply_multi",
        )
        res = _from_device_batch(out, was_np)
        if was_np:
            self.precond.check()
        return res

    def __del__(self):
        try:
            if self._handle is not None:
                _lib.load().hg_op_destroy(self._handle)
                self._handle = None
        except Exception:
            pass


def _basis(handle, n, col, nv):
    torch = _torch()
    out = torch.empty((nv, n), dtype=torch.float64, device="cuda")
    _lib.check(_lib.load().hg_op_basis(handle, int(col), int(nv), _vp(out), _stream()), "hg_op_basis")
    return out


class CsrOperator:
    """A host sparse/dense matrix uploaded once as a device CSR operator."""

    def __init__(self, mat):
        A = sp.csr_matrix(mat, dtype=np.float64)
        A.sort_indices()
        self.n = A.shape[0]
        if A.shape[0] != A.shape[1]:
            raise ValueError("operator must be square")
        ip = np.ascontiguousarray(A.indptr, dtype=np.int32)
        ix = np.ascontiguousarray(A.indices, dtype=np.int32)
        dv = np.ascontiguousarray(A.data, dtype=np.float64)
        h = ctypes.c_void_p()
        _torch()
        _lib.check(
            _lib.load().hg_op_create_csr(
                self.n, A.nnz, _lib.ptr(ip, ctypes.c_int32), _lib.ptr(ix, ctypes.c_int32),
                _lib.ptr(dv, ctypes.c_double), ctypes.byref(h),
            ),
            "hg_op_create_csr",
        )
        self._handle = h
        self.matrix = A

    def __call__(self, v):
        torch = _torch()
        t, was_np = _as_device(v, self.n)
        out = torch.empty_like(t)
        _lib.check(_lib.load().hg_op_apply(self._handle, _vp(t), _vp(out), _stream()), "hg_op_apply")
        return out.cpu().numpy() if was_np else out

    def basis(self, nv, col=0):
        """The first nv Krylov basis vectors of column col of the last GMRES
        solve on this operator, as an (nv, n) CUDA tensor (inspection hook)."""
        return _basis(self._handle, self.n, col, nv)

    def release(self):
        """Free this operator's Krylov bases / GMRES workspaces (hg_op_release)."""
        _lib.check(_lib.load().hg_op_release(self._handle), "hg_op_release")

    def apply_multi(self, V):
        """op applied to every column of a batch (numpy (n, nrhs) or CUDA (nrhs, n))."""
        torch = _torch()
        t, was_np = _as_device_batch(V, self.n)
        out = torch.empty_like(t)
        _lib.check(
            _lib.load().hg_op_apply_multi(self._handle, _vp(t), self.n, _vp(out), self.n, t.shape[0], _stream()),
            "hg_op_apply_multi",
        )
        return _from_device_batch(out, was_np)

    def __del__(self):
        try:
            if self._handle is not None:
                _lib.load().hg_op_destroy(self._handle)
                self._handle = None
        except Exception:
            pass


def factorize(forms, dec, coarse=None):
    """GPU ``factorize`` (schwarz.py:74-101): host factorisations + upload."""
    return TwoLevelPreconditioner(forms, dec, coarse)
