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
import types
from dataclasses import dataclass

import numpy as np
import scipy.linalg
import scipy.sparse as sp

from . import _lib
from .errors import SingularOperatorError
from .factor import (BandLU, band_lu, block_bandwidth, lu_b0, pack_b0_tiles, pack_band_records, record_floor,
                     record_widths, submatrix, swizzle_tile_rows, tile_span, pack_spike, split_block)

_DENSE_EIG_LIMIT = 1500
_SINGULAR_RTOL = 1e-12
DEVICE_BAND_MAX = 79  # widest band half-width the device band LU compiles (hg_factor.cu windows)


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
    one block (hg_local_solve).  ``host`` = the host dgbtrf factors of the
    block (computed on first access when the device factorised it; tests)."""

    def __init__(self, precond, index, host_factor, solver_index=None):
        self._p = precond
        self._s = index  # device block
        self._ls = index if solver_index is None else solver_index
        self._host = host_factor if isinstance(host_factor, BandLU) else None
        self.shape = (host_factor.n, host_factor.n)

    @property
    def host(self):
        if self._host is None:
            ls = self._p.local_solvers[self._ls]
            self._host = band_lu(submatrix(self._p._B, ls.idof, ls.idof), label=(ls.coarse_index, ls.fine_index))
        return self._host

    def solve(self, rhs):
        torch = _torch()
        t, was_np = _as_device(rhs, self.host.n)
        out = torch.empty_like(t)
        _lib.check(
            _lib.load().hg_local_solve(self._p._handle, self._s, _vp(t), _vp(out), _stream()), "hg_local_solve"
        )
        return out.cpu().numpy() if was_np else out


_SPLIT_G = {}


def _split_one(block, nchunk, label):
    """factor.split_block with its guard: the split solve must be backward
    stable on the whole block (normwise backward error of two seeded solves
    <= 1e-13; a stable solver sits near 1e-16).  A chunk that is itself
    (numerically) singular — k^2 at a Dirichlet eigenvalue of the chunk, not
    of the block — or a failed guard leaves the subdomain unsplit."""
    try:
        sb = split_block(block, nchunk, label=label)
    except SingularOperatorError:
        return None
    if sb is None:
        return None
    rng = np.random.default_rng(2406)
    anorm = abs(block).sum(axis=1).max()
    for _ in range(2):
        r = rng.standard_normal(block.shape[0])
        x = sb.solve(r)
        eta = np.abs(r - block @ x).max() / (anorm * np.abs(x).max() + np.abs(r).max())
        if not eta <= 1e-13:
            return None
    return sb


def _split_worker(i):
    a = _SPLIT_G["todo"][i]
    if a is None:
        return None
    from threadpoolctl import threadpool_limits

    with threadpool_limits(1):
        return _split_one(*a)


def _split_all(todo):
    """factor.split_block of every entry, in a fork pool: the spikes are band
    solves with kl or 2 kl right-hand sides per chunk (seconds per 18k-row
    block).  Serial under a CUDA tool's injection (a fork crashes the tool)."""
    from .problems import _tool_injected

    workers = min(sum(a is not None for a in todo), os.cpu_count() or 1)
    if workers <= 1 or _tool_injected() or os.environ.get("HG_SPLIT_WORKERS") == "1":
        return [_split_one(*a) if a is not None else None for a in todo]
    import multiprocessing as mp
    from concurrent.futures import ProcessPoolExecutor

    _SPLIT_G["todo"] = todo
    try:
        with ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("fork")) as ex:
            return list(ex.map(_split_worker, range(len(todo))))
    finally:
        _SPLIT_G.clear()


class SplitLocalLU:
    """``LocalSolver.lu`` of a subdomain whose block is split into chunks and
    separators (factor.split_block).  Its solve is three device stages over
    ALL subdomains (chunk solves, separator systems, spike updates), so
    ``solve`` runs the whole one-level part on a residual supported on this
    subdomain's dofs (hg_precond_local_solutions) and reads this subdomain's
    pieces back: the same B_s^{-1} r as an unsplit block's hg_local_solve."""

    def __init__(self, precond, idof, pieces):
        self._p = precond
        self._idof = np.asarray(idof)
        self._pieces = pieces  # [(block-local rows, position in the local solution scratch)]
        self.shape = (self._idof.size, self._idof.size)

    def solve(self, rhs):
        torch = _torch()
        p = self._p
        t, was_np = _as_device(rhs, self._idof.size)
        r = torch.zeros(p.n, dtype=torch.float64, device=t.device)
        r[torch.from_numpy(self._idof).to(t.device)] = t
        xs = torch.empty(p.xs_len, dtype=torch.float64, device=t.device)
        _lib.check(_lib.load().hg_precond_local_solutions(p._handle, _vp(r), _vp(xs), _stream()),
                   "hg_precond_local_solutions")
        out = torch.empty_like(t)
        for rows, pos in self._pieces:
            out[torch.from_numpy(rows).to(t.device)] = xs[pos:pos + rows.size]
        return out.cpu().numpy() if was_np else out


class LocalSolver:
    """Mirror of schwarz.LocalSolver (schwarz.py:26-34); ``min_eig`` and
    ``spd_flag`` are computed lazily (they only feed reports)."""

    def __init__(self, coarse_index, fine_index, idof, lu, diameter, block, matrix=None):
        self.coarse_index = coarse_index
        self.fine_index = fine_index
        self.idof = idof
        self.lu = lu
        self.diameter = diameter
        self._block = block
        self._matrix = matrix  # global B, to cut the block on demand (cached handles)
        self._min_eig = None

    @property
    def min_eig(self):
        if self._min_eig is None:
            if self._block is None and self.idof.size:
                self._block = submatrix(self._matrix, self.idof, self.idof)
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

    def __init__(self, forms, dec, coarse=None, b0_lu=None, keep_image=False):
        import time

        self._t = time.perf_counter
        self.setup_times = {}
        self._keep_image = keep_image
        self._image_arrays = None
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

        # ---- local factorisations (schwarz.py:83-85, 104-131): on the device
        # (hg_factor.cu, dgbtrf semantics) unless a block's band is wider than
        # the compiled windows or HG_HOST_FACTOR=1 asks for LAPACK dgbtrf here
        t0 = self._t()
        self.local_solvers = []
        factors = []
        blocks = []
        for i, j, sub in dec.fine_flat():
            idof = np.asarray(sub.idof)
            block = submatrix(B, idof, idof) if idof.size else sp.csr_matrix((0, 0))
            blocks.append(block)
            self.local_solvers.append(LocalSolver(i, j, idof, None, getattr(sub, "diameter", np.nan), block,
                                                  matrix=B))
        bws = [block_bandwidth(b) if b.shape[0] else 0 for b in blocks]
        nsplit = self._split_chunks(blocks, bws)
        self.device_factor = (os.environ.get("HG_HOST_FACTOR", "0") != "1" and not self._host_only_factor()
                              and max(bws, default=0) <= DEVICE_BAND_MAX and nsplit < 2)
        # device blocks: one per subdomain, or (split subdomains) its chunks followed by a pseudo
        # block of the separator dofs (factor.split_block; include/helmgpu.h "Split local blocks")
        self.splits = []          # (subdomain index, SplitBlock, first device block)
        self._dev_block = []      # subdomain -> device block (None when split)
        self._dev_labels = []
        split_of = {}
        if nsplit >= 2:
            todo = [(b, nsplit, (ls.coarse_index, ls.fine_index)) if b.shape[0] else None
                    for ls, b in zip(self.local_solvers, blocks)]
            split_of = dict(enumerate(_split_all(todo)))
        for s, (ls, block, bw) in enumerate(zip(self.local_solvers, blocks, bws)):
            label = (ls.coarse_index, ls.fine_index)
            sb = split_of.get(s)
            if sb is not None:
                self.splits.append((s, sb, len(factors)))
                self._dev_block.append(None)
                for rows, f in sb.chunks:
                    factors.append((ls.idof[rows], f))
                    self._dev_labels.append(label)
                factors.append((ls.idof[sb.sep_rows], band_lu(sp.csr_matrix((0, 0)))))
                self._dev_labels.append(label)
                continue
            if self.device_factor:
                f = types.SimpleNamespace(n=block.shape[0], kl=bw, ku=bw, kv=2 * bw, block=block,
                                          norm=float(np.sqrt(np.sum(block.data ** 2))) if block.nnz else 0.0)
            elif block.shape[0]:
                f = band_lu(block, label=label)
            else:
                f = band_lu(sp.csr_matrix((0, 0)))
            self._dev_block.append(len(factors))
            factors.append((ls.idof, f))
            self._dev_labels.append(label)
        self.setup_times["local_blocks"] = self._t() - t0

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
            b = self._dev_block[s]
            ls.lu = GpuBandLU(self, b, factors[b][1], s) if b is not None else None
        off = np.concatenate([[0], np.cumsum([i.size for i, _ in factors])])
        self.xs_len = int(off[-1])
        for s, sb, b0 in self.splits:
            pieces = [(rows, int(off[b0 + p])) for p, (rows, _) in enumerate(sb.chunks)]
            pieces.append((sb.sep_rows, int(off[b0 + len(sb.chunks)])))
            self.local_solvers[s].lu = SplitLocalLU(self, self.local_solvers[s].idof, pieces)

    @staticmethod
    def _split_chunks(blocks, bws):
        """Chunks per subdomain for the split local solve (1 = none).  HG_LOCAL_SPLIT = P forces it;
        the default splits only decompositions with fewer blocks than half the SMs and wide bands
        (config 5 at 8 x 8: 64 blocks of 18k rows, kl = 136) in two."""
        env = os.environ.get("HG_LOCAL_SPLIT", "auto")
        if env != "auto":
            return max(1, int(env))
        nb = sum(1 for b in blocks if b.shape[0])
        if nb == 0 or nb > 74 or max(bws, default=0) < 96:
            return 1
        return 2  # measured at 5-8: 2 chunks (128 chains, one wave) beat 4 and 8 (more spike bytes, same wave count)

    def _host_only_factor(self):
        return getattr(self, "_host_only", False)  # host_image(): no device to factor on

    # ------------------------------------------------------------------ upload
    def _upload(self, B, Dk, factors, cblocks, lu, piv):
        arrays, meta = self._image(B, Dk, factors, cblocks, lu, piv)
        meta["labels"] = [[int(a), int(b)] for a, b in self._dev_labels]
        if getattr(self, "_host_only", False):
            self._image_arrays, self._meta = arrays, meta
            return
        t0 = self._t()
        self._create(arrays, meta)  # upload + device band LU + panel records
        self.setup_times["create"] = self._t() - t0
        if self.m:
            t0 = self._t()
            if meta.get("b0_split"):
                # the bisected coarse solve against getrs first; beyond the bar it is switched off
                # (and leaves the image), and the full chain is checked as before
                meta["b0_split_dev"] = self._check_coarse_solve(strict=False)
                if not meta["b0_split_dev"] <= 1e-11:
                    _lib.check(_lib.load().hg_debug_set(self._handle, _lib.DEBUG_B0_SPLIT, 0), "hg_debug_set")
                    meta["b0_split"] = 0
                    arrays = {k: v for k, v in arrays.items() if k not in self.B0_SPLIT_KEYS}
            self.b0_split = bool(meta.get("b0_split"))
            if self.b0_split:
                # the full chain too (the bisected one can be switched off: the tuning below, tests)
                self._set_tune(b0_split_on=False)
            meta["b0_tile_dev"] = self.b0_tile_dev = self._check_coarse_solve()
            self.setup_times["b0_guard"] = self._t() - t0
            if self.b0_split:
                t0 = self._t()
                if os.environ.get("HG_B0_SPLIT", "auto") == "1":  # forced: no timing
                    meta["tune"] = {"b0_split_on": True, "local_stages": int(os.environ.get("HG_LOCAL_STAGES", "0")),
                                    "b0_tile_stages": int(os.environ.get("HG_B0_TILE_STAGES", "0"))}
                    self._set_tune(b0_split_on=True, local_stages=meta["tune"]["local_stages"],
                                   tile_stages=meta["tune"]["b0_tile_stages"])
                else:
                    meta["tune"] = self._tune_single_apply()
                if meta["tune"]["b0_split_on"] and (not meta.get("b0_dense") or meta.get("b0_inv_batched_only")):
                    meta["b0_bytes"] = self.b0_bytes = int(meta["b0_bytes_split"])
                self.setup_times["apply_tuning"] = self._t() - t0
        if "b0_inv" in arrays and not isinstance(arrays["b0_inv"], np.ndarray):  # device copy: host only if cached
            arrays = dict(arrays)
            binv = arrays.pop("b0_inv")
            if self._keep_image:
                arrays["b0_inv"] = binv.cpu().numpy()
        if "factor_info" in arrays:
            self._check_device_factor(arrays, meta)
            if self._keep_image:  # the cache stores the device-built records, not the factor inputs
                arrays = dict(arrays)
                for field, name, length in ((_lib.FIELD_LOCAL_FWD, "local_fwd", meta["local_fwd_len"]),
                                            (_lib.FIELD_LOCAL_BWD, "local_bwd", meta["local_bwd_len"])):
                    buf = np.empty(int(length))
                    _lib.check(_lib.load().hg_precond_read(self._handle, field, _lib.ptr(buf, ctypes.c_double),
                                                           int(length)), "hg_precond_read")
                    arrays[name] = buf
                for name in ("local_bw", "lcsr_indptr", "lcsr_cols", "lcsr_vals", "factor_info", "factor_min_pivot"):
                    arrays.pop(name, None)
                meta = dict(meta)
                meta.pop("lcsr_nnz", None)
        if self._keep_image:
            self._image_arrays = arrays
            self._meta = meta

    def _check_device_factor(self, arrays, meta):
        """The singular-block test of schwarz.py:111-121 on the device factors:
        an exactly-zero pivot (dgbtrf INFO) or min |u_jj| <= 1e-12 ||block||_F."""
        info, minp = arrays["factor_info"], arrays["factor_min_pivot"]
        for s, ls in enumerate(self.local_solvers):
            if ls.idof.size == 0:
                continue
            where = "fine subdomain (%d, %d)" % (ls.coarse_index, ls.fine_index)
            if info[s] > 0:
                raise SingularOperatorError(
                    "local Helmholtz block on %s is singular (k^2 equals a local Dirichlet eigenvalue): "
                    "zero pivot at %d" % (where, info[s]))
            if minp[s] <= _SINGULAR_RTOL * meta["local_norms"][s]:
                raise SingularOperatorError(
                    "local Helmholtz block on %s is numerically singular (smallest pivot %.3e)" % (where, minp[s]))

    @classmethod
    def from_image(cls, arrays, meta, forms=None):
        """A preconditioner straight from an image (the on-disk setup cache,
        cache.py): hg_precond_create on the stored arrays, no host setup."""
        from .cache import forms_from_image

        self = cls.__new__(cls)
        self._keep_image = True
        self._image_arrays = arrays
        self.forms = forms if forms is not None else forms_from_image(arrays, meta)
        self.n = int(meta["n"])
        self._handle = None
        self._keep = []
        self.Z = None
        self.b0_piv = None
        self._B = self.forms.helmholtz
        self._Dk = self.forms.dk
        self._create(arrays, meta)
        off = np.asarray(arrays["local_idx_off"])
        idx = arrays["local_idx"]
        self.local_solvers = []
        for s, (ci, fi) in enumerate(meta["labels"]):
            idof = np.asarray(idx[off[s]:off[s + 1]], dtype=np.int64)
            kl, kv = meta["local_bands"][s]
            ls = LocalSolver(ci, fi, idof, None, np.nan, None, matrix=self._B)
            if idof.size and int(arrays["local_n"][s]) == 0:
                # separator pseudo block of a split subdomain (a cached image lists device blocks,
                # not subdomains): no solve of its own
                ls.lu = None
            else:
                ls.lu = GpuBandLU(self, s, types.SimpleNamespace(n=int(idof.size), kl=kl, kv=kv))
            self.local_solvers.append(ls)
        return self

    def _image(self, B, Dk, factors, cblocks, lu, piv):
        """Everything hg_precond_create consumes, as host arrays (named after
        the HgPrecondDesc fields) plus scalars: the unit the on-disk setup
        cache (cache.py) stores."""
        A, M = {}, {}
        i32, i64, f64 = np.int32, np.int64, np.float64

        def put(name, a, dtype):
            A[name] = np.ascontiguousarray(a, dtype=dtype)

        M["n"] = int(self.n)
        M["nnz"] = int(B.nnz)
        k = getattr(self.forms, "k", None)
        M["k"] = None if k is None else float(k)
        put("indptr", B.indptr, i32)
        put("indices", B.indices, i32)
        put("b_data", B.data, f64)
        if Dk is not None:
            put("dk_data", Dk.data, f64)

        ns, kls, kvs, fss, bss = [], [], [], [], []
        idx_off = [0]
        fwd_parts, bwd_parts, foff, boff = [], [], [], []
        fpos = bpos = 0
        kl_floor = record_floor(max([f.kl for _, f in factors], default=0))
        kv_floor = record_floor(max([f.kv for _, f in factors], default=0))
        device = getattr(self, "device_factor", False)
        lptr, lcols, lvals = [], [], []
        nnz_pos = 0
        for idof, f in factors:
            if device:
                fs, bs, klp, kvp = record_widths(f.kl, f.kv, kl_floor, kv_floor)
                blk = f.block
                lptr.append(blk.indptr.astype(np.int64) + nnz_pos)
                lcols.append(blk.indices)
                lvals.append(blk.data)
                nnz_pos += blk.nnz
                fsize, bsize = f.n * fs, f.n * bs
            else:
                fw, bw, fs, bs, klp, kvp = pack_band_records(f, kl_floor, kv_floor)
                fwd_parts.append(fw.ravel())
                bwd_parts.append(bw.ravel())
                fsize, bsize = fw.size, bw.size
            ns.append(f.n)
            kls.append(klp)
            kvs.append(kvp)
            fss.append(fs)
            bss.append(bs)
            idx_off.append(idx_off[-1] + idof.size)
            foff.append(fpos)
            boff.append(bpos)
            fpos += fsize
            bpos += bsize
        M["n_local"] = len(factors)
        put("local_n", ns, i32)
        put("local_kl", kls, i32)
        put("local_kv", kvs, i32)
        put("local_fstride", fss, i32)
        put("local_bstride", bss, i32)
        put("local_idx_off", idx_off, i64)
        put("local_idx", np.concatenate([i for i, _ in factors]) if factors else np.zeros(0), i32)
        put("local_fwd_off", foff, i64)
        put("local_bwd_off", boff, i64)
        M["local_fwd_len"] = int(fpos)
        M["local_bwd_len"] = int(bpos)
        if device:
            put("local_bw", [f.kl for _, f in factors], i32)
            put("lcsr_indptr", np.concatenate(lptr) if lptr else np.zeros(0), i64)
            put("lcsr_cols", np.concatenate(lcols) if lcols else np.zeros(0), i32)
            put("lcsr_vals", np.concatenate(lvals) if lvals else np.zeros(0), f64)
            M["lcsr_nnz"] = int(nnz_pos)
            put("factor_info", np.zeros(len(factors)), i32)
            put("factor_min_pivot", np.zeros(len(factors)), f64)
            M["local_norms"] = [float(f.norm) for _, f in factors]
        else:
            put("local_fwd", np.concatenate(fwd_parts) if fwd_parts else np.zeros(0), f64)
            put("local_bwd", np.concatenate(bwd_parts) if bwd_parts else np.zeros(0), f64)
        M["local_bands"] = [[int(f.kl), int(f.kv)] for _, f in factors]
        self._image_splits(A, M, idx_off)

        m = sum(b.shape[1] for _, b in cblocks)
        M["m"] = int(m)
        M["cblock_shapes"] = [[int(b.shape[0]), int(b.shape[1])] for _, b in cblocks]
        M["b0_bytes"] = 0
        M["b0_mode"] = -1
        M["b0_dense"] = False
        if m:
            P = int(os.environ.get("HG_B0_PANEL", "64"))
            t0 = self._t()
            T = pack_b0_tiles(lu, piv, P)
            # coarse-solve kernel: one DSMEM cluster when the x ring fits in shared memory
            cs = min(16, T.K)
            ring = tile_span(T) + cs + 1
            mode = int(os.environ.get("HG_B0_MODE", "1"))
            if mode == 1 and (T.P != 64 or ring > 96):  # the tagged x ring must fit in shared memory
                mode = 0
            if mode == 1:
                T = T.premultiply()  # tiles D_t^{-1} T[t, j]: rows of a panel finish independently
            self.setup_times["b0_tiles"] = self._t() - t0
            # the tiled algorithm (inverted 64x64 diagonal blocks) is checked against getrs on
            # the device kernel itself once the handle exists (_check_coarse_solve); the host-only image
            # (no device) checks the host emulation of the same algorithm
            self.b0_tiles = T
            self._b0_lu = (lu, piv)
            if getattr(self, "_host_only", False):
                M["b0_tile_dev"] = self._tile_guard(lambda c: T.solve(c), m, P)
            t0 = self._t()
            M["b0_bytes"] = int(T.nbytes + 4 * m + 4 * T.tile_col.size)
            # dense mode: B0^{-1} applied as a streaming GEMV / DMMA GEMM beside the
            # local solves; kept only if it agrees with getrs (the reference's lu_solve)
            M["b0_dense_dev"] = None
            # "1": every apply; "multi" (default while B0^{-1} fits: m <= 20000, 3.2 GB): batched applies
            # only — there the chain is the critical path, while the single apply keeps the chain
            # (the 1.9 GB stream would contend with its local solves); "0": never
            host_only = getattr(self, "_host_only", False)  # host_image(): no device to invert on
            dense = os.environ.get("HG_B0_DENSE", "multi" if m <= 20000 and not host_only else "0")
            if dense in ("1", "multi") or (dense == "auto" and m <= 20000):  # "auto": whenever it fits
                # B0^{-1} on the device (setup; stays there: hg_precond_create copies device to device),
                # checked against getrs (the reference's lu_solve) on two seeded vectors
                torch = _torch()
                B0 = np.ascontiguousarray(np.asarray(self._coarse.B0), dtype=np.float64)
                Binv = torch.linalg.inv(torch.from_numpy(B0).cuda())
                rng = np.random.default_rng(1)
                ddev = 0.0
                getrs = self._getrs()
                for _ in range(2):
                    c = rng.standard_normal(m)
                    want = getrs(c)
                    got = (Binv @ torch.from_numpy(c).cuda()).cpu().numpy()
                    ddev = max(ddev, float(np.abs(got - want).max() / max(np.abs(want).max(), 1e-300)))
                M["b0_dense_dev"] = ddev
                if ddev <= 1e-11:
                    M["b0_dense"] = True
                    M["b0_inv_batched_only"] = 1 if dense == "multi" else 0
                    A["b0_inv"] = Binv.contiguous()
                    M["b0_bytes_multi"] = int(8 * m * m + 16 * m)
                    if dense != "multi":
                        M["b0_bytes"] = int(8 * m * m + 16 * m)
            self.setup_times["b0_inverse"] = self._t() - t0
            M["b0_split"] = 0
            if mode == 1 and not host_only and os.environ.get("HG_B0_SPLIT", "auto") != "0":
                t0 = self._t()
                self._b0_bisection(A, M, cs)
                self.setup_times["b0_bisection"] = self._t() - t0
            M["n_cblk"] = len(cblocks)
            put("cblk_n", [i.size for i, _ in cblocks], i32)
            put("cblk_m", [b.shape[1] for _, b in cblocks], i32)
            put("cblk_idx_off", np.concatenate([[0], np.cumsum([i.size for i, _ in cblocks])]), i64)
            put("cblk_idx", np.concatenate([i for i, _ in cblocks]), i32)
            zsizes = [b.size for _, b in cblocks]
            put("cblk_z_off", np.concatenate([[0], np.cumsum(zsizes)[:-1]]), i64)
            put("z_data", np.concatenate([b.ravel() for _, b in cblocks]), f64)
            M["z_len"] = int(A["z_data"].size)
            put("b0_perm", T.perm, i32)
            M["b0_panel"] = int(T.P)
            M["b0_npanel"] = int(T.K)
            put("b0_tile_ptr", T.tile_ptr, i64)
            put("b0_tile_col", T.tile_col if T.tile_col.size else np.zeros(1), i32)
            M["b0_ntile"] = int(T.tile_col.size)
            M["b0_ctas"] = int(os.environ.get("HG_B0_CTAS", "0"))
            M["b0_mode"] = mode
            if mode == 1:
                M["b0_cluster"], M["b0_ring"] = int(cs), int(ring)
                dinv = swizzle_tile_rows(T.dinv)
                tiles = swizzle_tile_rows(T.tiles) if T.tiles.size else np.zeros(1)
            else:
                M["b0_cluster"], M["b0_ring"] = 0, 0
                dinv, tiles = T.dinv, (T.tiles if T.tiles.size else np.zeros(1))
            put("b0_dinv", dinv, f64)
            put("b0_tiles", tiles, f64)
        return A, M

    def _image_splits(self, A, M, idx_off):
        """Descriptor arrays of the split local blocks (helmgpu.h "Split local blocks")."""
        i32, i64, f64 = np.int32, np.int64, np.float64
        splits = getattr(self, "splits", [])
        M["n_split"] = len(splits)
        M["n_spike"] = 0
        M["split_sinv_len"] = M["spike_len"] = 0
        M["split_bytes"] = 0
        if not splits:
            return
        blk, row_off, fptr, fpos, fval, soff, sinv = [], [0], [0], [], [], [], []
        kblk, ksplit, kcol0, kw, koff, kdata = [], [], [], [], [], []
        spos = kpos = 0
        for si, (s, sb, b0) in enumerate(splits):
            nchunk = len(sb.chunks)
            blk.append(b0 + nchunk)
            row_off.append(row_off[-1] + sb.sep_rows.size)
            # block-local row -> position in the local solution scratch
            pos = np.full(sb.F.shape[1], -1, dtype=np.int64)
            for p, (rows, _) in enumerate(sb.chunks):
                pos[rows] = idx_off[b0 + p] + np.arange(rows.size)
            F = sp.csr_matrix(sb.F)
            F.sort_indices()
            if (pos[F.indices] < 0).any():
                raise ValueError("separator rows couple to a non-chunk column")
            fptr.extend((fptr[-1] + F.indptr[1:]).tolist())
            fpos.append(pos[F.indices])
            fval.append(F.data)
            soff.append(spos)
            sinv.append(sb.sinv.ravel())
            spos += sb.sinv.size
            for p, (c0, w, W) in enumerate(sb.spikes):
                if w == 0:
                    continue
                pk = pack_spike(W)
                kblk.append(b0 + p)
                ksplit.append(si)
                kcol0.append(c0)
                kw.append(w)
                koff.append(kpos)
                kdata.append(pk)
                kpos += pk.size
        A["split_blk"] = np.ascontiguousarray(blk, dtype=i32)
        A["split_row_off"] = np.ascontiguousarray(row_off, dtype=i64)
        A["split_f_indptr"] = np.ascontiguousarray(fptr, dtype=i64)
        A["split_f_pos"] = np.ascontiguousarray(np.concatenate(fpos), dtype=i64)
        A["split_f_val"] = np.ascontiguousarray(np.concatenate(fval), dtype=f64)
        A["split_sinv_off"] = np.ascontiguousarray(soff, dtype=i64)
        A["split_sinv"] = np.ascontiguousarray(np.concatenate(sinv), dtype=f64)
        M["split_sinv_len"] = int(spos)
        M["n_spike"] = len(kblk)
        A["spike_blk"] = np.ascontiguousarray(kblk, dtype=i32)
        A["spike_split"] = np.ascontiguousarray(ksplit, dtype=i32)
        A["spike_col0"] = np.ascontiguousarray(kcol0, dtype=i32)
        A["spike_w"] = np.ascontiguousarray(kw, dtype=i32)
        A["spike_off"] = np.ascontiguousarray(koff, dtype=i64)
        A["spike_data"] = np.ascontiguousarray(np.concatenate(kdata), dtype=f64)
        M["spike_len"] = int(kpos)
        # bytes one local solve reads beyond the chunk records: Sigma^{-1}, F, the spikes
        M["split_bytes"] = int(8 * spos + 16 * A["split_f_pos"].size + 8 * kpos)
        M["split_chunks"] = int(max(len(sb.chunks) for _, sb, _ in splits))
        M["split_cond"] = float(max(sb.cond for _, sb, _ in splits))

    def _b0_bisection(self, A, M, cs):
        """Descriptor arrays of the bisected single-RHS coarse solve (helmgpu.h
        "Bisected coarse solve"): B0 is banded, so two half chains + a dense
        separator system replace one chain of 2K hand-offs.  Built on the
        device (torch.linalg, setup only); declined when B0 is short
        (K < 96 panels unless HG_B0_SPLIT=1) or the halves' tile rings do not
        fit.  The caller checks the result against getrs (_check_coarse_solve)."""
        torch = _torch()
        B0 = np.ascontiguousarray(np.asarray(self._coarse.B0), dtype=np.float64)
        m = B0.shape[0]
        if os.environ.get("HG_B0_SPLIT", "auto") != "1" and (m + 63) // 64 < 96:
            return
        bw = 0
        for r0 in range(0, m, 1024):
            rr, cc = np.nonzero(B0[r0:r0 + 1024])
            if rr.size:
                bw = max(bw, int(np.abs(cc - (rr + r0)).max()))
        ns = max(bw, 1)
        forced = os.environ.get("HG_B0_SPLIT", "auto") == "1"
        if m - ns < (2 if forced else 8) * ns:  # halves shorter than the separator (than 4 of them): not worth it
            return
        a = (m - ns) // 2
        wl, wr = min(bw, a), min(bw, m - a - ns)
        Bd = torch.from_numpy(B0).cuda()
        S = slice(a, a + ns)
        sig = Bd[S, S].clone()
        halves, Ws = [], []
        for h in (slice(0, a), slice(a + ns, m)):
            Ah = Bd[h, h].contiguous()
            LU, piv = torch.linalg.lu_factor(Ah)
            E = Bd[h, S].contiguous()
            W = torch.linalg.lu_solve(LU, piv, E)
            W = W + torch.linalg.lu_solve(LU, piv, E - Ah @ W)  # one refinement step
            sig -= Bd[S, h] @ W
            Ws.append(W)
            T = pack_b0_tiles(LU.cpu().numpy(), piv.cpu().numpy().astype(np.int64) - 1, 64)
            # a full cluster per half chain (8 CTAs stream a half's tiles too slowly: 0.58 vs 0.37 ms)
            c = min(int(os.environ.get("HG_B0_SPLIT_CS", cs)), T.K)
            ring = tile_span(T) + c + 1
            if ring > 96:
                return
            halves.append((T.premultiply(), c, ring))
            del Ah, LU, E
        sinv = torch.linalg.inv(sig)
        F = torch.cat([Bd[S, a - wl:a], Bd[S, a + ns:a + ns + wr]], dim=1).contiguous()
        f64, i32, i64 = np.float64, np.int32, np.int64
        M["b0_split"] = 1
        M["b0s_a"], M["b0s_ns"], M["b0s_wl"], M["b0s_wr"] = int(a), int(ns), int(wl), int(wr)
        nbytes = 0
        for h, (T, c, ring) in enumerate(halves):
            pre = "b0h%d_" % h
            M[pre + "npanel"], M[pre + "ring"], M[pre + "cluster"] = int(T.K), int(ring), int(c)
            M[pre + "ntile"] = int(T.tile_col.size)
            A[pre + "perm"] = np.ascontiguousarray(T.perm, dtype=i32)
            A[pre + "dinv"] = np.ascontiguousarray(swizzle_tile_rows(T.dinv), dtype=f64)
            A[pre + "tile_ptr"] = np.ascontiguousarray(T.tile_ptr, dtype=i64)
            A[pre + "tile_col"] = np.ascontiguousarray(T.tile_col if T.tile_col.size else np.zeros(1), dtype=i32)
            A[pre + "tiles"] = np.ascontiguousarray(swizzle_tile_rows(T.tiles) if T.tiles.size else np.zeros(1),
                                                    dtype=f64)
            nbytes += T.nbytes + 4 * T.perm.size
        A["b0s_f"] = F.cpu().numpy()
        A["b0s_sinv"] = sinv.contiguous().cpu().numpy()
        A["b0s_w"] = torch.cat(Ws, dim=0).contiguous().cpu().numpy()
        nbytes += A["b0s_f"].nbytes + A["b0s_sinv"].nbytes + A["b0s_w"].nbytes
        M["b0_bytes_chain"] = int(M["b0_bytes"])
        M["b0_bytes_split"] = int(nbytes)

    B0_SPLIT_KEYS = ("b0h0_perm", "b0h0_dinv", "b0h0_tile_ptr", "b0h0_tile_col", "b0h0_tiles", "b0h1_perm",
                     "b0h1_dinv", "b0h1_tile_ptr", "b0h1_tile_col", "b0h1_tiles", "b0s_f", "b0s_sinv", "b0s_w")

    def _set_tune(self, b0_split_on=None, local_stages=None, tile_stages=None):
        lib = _lib.load()
        if tile_stages is not None:
            _lib.check(lib.hg_debug_set(self._handle, _lib.DEBUG_B0_TILE_STAGES, int(tile_stages)), "hg_debug_set")
        if b0_split_on is not None:
            _lib.check(lib.hg_debug_set(self._handle, _lib.DEBUG_B0_SPLIT, 1 if b0_split_on else 0), "hg_debug_set")
        if local_stages is not None:
            _lib.check(lib.hg_debug_set(self._handle, _lib.DEBUG_LOCAL_STAGES, int(local_stages)), "hg_debug_set")

    def _tune_single_apply(self):
        """Which single-RHS apply schedule this handle runs: the bisected coarse
        solve holds two clusters (32 SMs) instead of one, which only pays when
        the local solves' CTAs still fit beside them in one wave — with 4 ring
        stages instead of 6 where that takes a third CTA per SM.  Decided by
        timing the apply itself (device events, 3 + 12 applies per candidate);
        the default schedule (full chain, 6 stages) stays unless another one is
        at least 8% faster, so that near-ties never flip between runs.  The
        choice is part of the image (the setup cache reproduces it)."""
        torch = _torch()
        r = torch.from_numpy(np.random.default_rng(7).standard_normal(self.n)).cuda()

        def timed():
            for _ in range(3):
                self.apply(r)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(torch.cuda.current_stream())
            for _ in range(12):
                self.apply(r)
            e1.record(torch.cuda.current_stream())
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / 12

        # (bisected?, local ring stages, coarse tile-ring stages; 0 = default): fewer stages = less shared
        # memory per CTA, i.e. a third local CTA per SM / a local CTA on the chains' SMs
        cands = [(False, 0, 0), (True, 0, 0), (True, 4, 0), (True, 0, 2), (True, 4, 2)]
        ms = {}
        for cand in cands:
            self._set_tune(b0_split_on=cand[0], local_stages=cand[1], tile_stages=cand[2])
            ms[cand] = timed()
        best = min(ms, key=ms.get)
        if ms[best] > 0.92 * ms[cands[0]]:
            best = cands[0]
        self._set_tune(b0_split_on=best[0], local_stages=best[1], tile_stages=best[2])
        return {"b0_split_on": bool(best[0]), "local_stages": int(best[1]), "b0_tile_stages": int(best[2]),
                "apply_ms": {"%s,%d,%d" % ("bisected" if k[0] else "chain", k[1] or 6, k[2] or 4): round(v, 4)
                             for k, v in ms.items()}}

    def _getrs(self):
        """c -> getrs(lu, piv, c) (the reference's lu_solve, schwarz.py:56) with the
        same getrf factors; on the device when there is one (the factors are
        uploaded once per factorize), else LAPACK."""
        if getattr(self, "_getrs_fn", None) is not None:
            return self._getrs_fn
        lu, piv = self._b0_lu
        if getattr(self, "_host_only", False):
            fn = lambda c: scipy.linalg.lu_solve((lu, piv), c)  # noqa: E731
        else:
            torch = _torch()
            LU = torch.from_numpy(np.ascontiguousarray(lu)).cuda()
            pv = torch.from_numpy(np.asarray(piv, dtype=np.int32) + 1).cuda()  # LAPACK 1-based

            def fn(c):
                b = torch.from_numpy(np.ascontiguousarray(c, dtype=np.float64)).cuda()[:, None]
                return torch.linalg.lu_solve(LU, pv, b)[:, 0].cpu().numpy()
        self._getrs_fn = fn
        return fn

    def _tile_guard(self, solve, m, P, strict=True):
        """Max relative deviation of a B0 solve from getrs on 4 seeded vectors;
        raises SingularOperatorError above 1e-11 (B0 too ill-conditioned for the
        inverted diagonal blocks of the tile algorithm)."""
        rng = np.random.default_rng(0)
        dev = 0.0
        getrs = self._getrs()
        for _ in range(4):
            c = rng.standard_normal(m)
            want = getrs(c)
            dev = max(dev, float(np.abs(solve(c) - want).max() / max(np.abs(want).max(), 1e-300)))
        if dev > 1e-11 and strict:
            raise SingularOperatorError(
                "coarse tile factorisation deviates from getrs by %.2e (B0 too ill-conditioned for "
                "inverted %dx%d diagonal blocks)" % (dev, P, P))
        return dev

    def _check_coarse_solve(self, strict=True):
        """The guard of the tiled coarse solve, run on the device chain kernel itself."""
        torch = _torch()

        def dev_solve(c):
            cd = torch.from_numpy(c).cuda()
            y = torch.empty_like(cd)
            _lib.check(_lib.load().hg_precond_coarse_solve(self._handle, _vp(cd), _vp(y), _stream()),
                       "hg_precond_coarse_solve")
            return y.cpu().numpy()

        res = self._tile_guard(dev_solve, self.m, self.b0_tiles.P, strict)
        if strict:
            self._getrs_fn = None  # the device copy of the factors is not kept
        return res

    def _create(self, arrays, meta):
        """hg_precond_create from an image (``_image`` or the setup cache)."""
        lib = _lib.load()
        torch = _torch()  # CUDA context present before the first allocation
        d = _lib.HgPrecondDesc()
        for name, ctype in _lib.HgPrecondDesc._fields_:
            if issubclass(ctype, ctypes._Pointer):  # array field (numpy host array or CUDA tensor)
                a = arrays.get(name)
                if a is None:
                    setattr(d, name, None)
                elif isinstance(a, torch.Tensor):
                    setattr(d, name, ctypes.cast(ctypes.c_void_p(a.data_ptr()), ctype))
                else:
                    setattr(d, name, a.ctypes.data_as(ctype))
            else:
                setattr(d, name, int(meta.get(name, 0)))
        h = ctypes.c_void_p()
        _lib.check(lib.hg_precond_create(ctypes.byref(d), ctypes.byref(h)), "hg_precond_create")
        self._handle = h
        self._meta = meta
        self.m = int(meta["m"])
        tune = meta.get("tune")
        if tune and meta.get("b0_split"):  # a cached image: the schedule its setup chose
            self._set_tune(b0_split_on=tune["b0_split_on"], local_stages=tune["local_stages"],
                           tile_stages=tune.get("b0_tile_stages", 0))
        self.local_sizes = [int(x) for x in arrays["local_n"]] if "local_n" in arrays else []
        self.xs_len = int(np.asarray(arrays["local_idx_off"])[-1]) if "local_idx_off" in arrays else 0
        self.local_bands = [tuple(b) for b in meta["local_bands"]]
        self.cblock_shapes = [tuple(c) for c in meta["cblock_shapes"]]
        self.b0_bytes = int(meta["b0_bytes"])
        self.b0_bytes_multi = int(meta.get("b0_bytes_multi", meta["b0_bytes"]))
        self.b0_mode = int(meta["b0_mode"])
        self.b0_dense = bool(meta["b0_dense"])
        self.b0_dense_dev = meta.get("b0_dense_dev")
        self.b0_tile_dev = meta.get("b0_tile_dev")
        self.b0_split = bool(meta.get("b0_split"))
        self.split_bytes = int(meta.get("split_bytes", 0))
        self.n_split = int(meta.get("n_split", 0))
        self.panel_active = bool(lib.hg_precond_stat(h, _lib.STAT_PANEL_ACTIVE) == 1.0)
        self.panel_deviation = float(lib.hg_precond_stat(h, _lib.STAT_PANEL_DEVIATION))
        # factor bytes one batched local solve streams (16-row panel records, hg_local_panel.cu)
        self.panel_bytes = int(lib.hg_precond_stat(h, _lib.STAT_PANEL_BYTES)) if self.panel_active else None

    # ------------------------------------------------------------------ API
    @property
    def has_coarse(self):
        return self.m > 0

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
        # the C ABI takes column c at F + c n: a column-major (Fortran-ordered) F is passed as it is,
        # a row-major one is transposed on the host first (a strided 8 n nrhs-byte copy)
        Fc = F.T if F.T.flags.c_contiguous else np.ascontiguousarray(F.T)
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
        return Xc.T, _reports(hist, info, None)  # (n, nrhs), column-major: no host transpose

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


def host_image(forms, dec, coarse=None):
    """(arrays, meta) of the device image the GPU factorize would upload,
    computed on the host only (no device, no handle): the cache format's
    contents (cache.save_image), testable without a GPU."""
    pre = TwoLevelPreconditioner.__new__(TwoLevelPreconditioner)
    pre._host_only = True
    TwoLevelPreconditioner.__init__(pre, forms, dec, coarse, keep_image=True)
    return pre._image_arrays, pre._meta


def factorize(forms, dec, coarse=None, keep_image=False):
    """GPU ``factorize`` (schwarz.py:74-101): host factorisations + upload.
    ``keep_image``: keep the uploaded host arrays so that
    cache.save_preconditioner can write them (the on-disk setup cache)."""
    return TwoLevelPreconditioner(forms, dec, coarse, keep_image=keep_image)
