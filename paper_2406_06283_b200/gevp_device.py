"""Local H_k-GenEO eigenproblems on the device.

All coarse subdomains' pencils B_i p = lambda C_i p (eigencoarse.py:83-101,
C_i = W D_k W) are solved at once, in the shift-invert restatement of §8c
that coarse.solve_gevp_lanczos runs on the host with ARPACK:

    mu = 1 / (lambda + g),   A_i = R_I (B_i + g C_i)^{-1} C_i E_I,

A_i self-adjoint in <x, y> = x^T C_II y; the lowest lambda are the largest
mu.  Here one thick-restart (Krylov-Schur) Lanczos per subdomain runs in
lock step over the batch:

  * (B_i + g C_i)^{-1} for every subdomain in ONE device apply: the shifted
    blocks are uploaded as the block-diagonal "global" matrix of a
    preconditioner handle whose one-level blocks are exactly those blocks
    (device band LU, hg_factor.cu; band solves, hg_local_*.cu), so the
    one-level apply is the block-diagonal inverse;
  * C_i x for every subdomain as one device SpMV of the block-diagonal C;
  * per-subdomain C inner products, two-pass classical Gram-Schmidt against
    the subdomain's own basis and the Krylov-Schur restarts as batched
    tensor contractions over a padded [basis][subdomain][dof] layout.

Eigenpairs leave when the residual |b^T y| <= tol * max(theta) for the
n_wanted + 1 largest Ritz values of every subdomain (ARPACK's criterion with
tol at rounding level, as the host path asks with tol = 0).  Eigenvectors
map back exactly as the host path does (eigencoarse.py:201-204):
p = (B + g C)^{-1} C E_I q / mu, C-normalised.  A subdomain whose wanted
spectrum reaches below -g (a negative mu) is re-solved by the host path
with its widened shift.
"""

import types

import numpy as np
import scipy.sparse as sp

from .coarse import LocalGevpResult, solve_gevp_lanczos, assemble_local_gevp
from .errors import EigensolveError


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("gevp_device needs a CUDA device")
    return torch


def solve_local_gevps_device(forms, dec, n_wanted, shift=2.0, tol=1e-15, max_restarts=200, seed=7919,
                             keep_extra=20, verbose=False):
    """[LocalGevpResult] for every coarse subdomain (partial spectra: the
    lowest ``n_wanted + 1`` finite eigenvalues), as coarse.solve_gevp_lanczos
    returns them."""
    torch = _torch()
    from .schwarz import factorize

    nb = dec.n_coarse
    gevps = [assemble_local_gevp(i, forms, dec, dense=False) for i in range(nb)]
    sizes = np.array([g.b_mat.shape[0] for g in gevps])
    offs = np.concatenate([[0], np.cumsum(sizes)])
    N = int(offs[-1])
    Ms, Cs = [], []
    for g in gevps:
        Ms.append(sp.csr_matrix(g.b_mat + shift * g.c_mat))
        Cs.append(sp.csr_matrix(g.c_mat))
    Mbig = sp.block_diag(Ms, format="csr")
    Cbig = sp.block_diag(Cs, format="csr")
    forms_bd = types.SimpleNamespace(helmholtz=Mbig, dk=Cbig, n_dofs=N, k=None)
    subs = [types.SimpleNamespace(idof=np.arange(offs[i], offs[i + 1]), diameter=np.nan) for i in range(nb)]
    dec_bd = types.SimpleNamespace(fine_flat=lambda: ((i, 0, subs[i]) for i in range(nb)))
    import os

    saved = os.environ.get("HG_LOCAL_PANEL")
    os.environ["HG_LOCAL_PANEL"] = "0"  # single-vector applies only: no batched panel records
    try:
        pre = factorize(forms_bd, dec_bd, None)  # device band LU of every B_i + g C_i
    finally:
        if saved is None:
            del os.environ["HG_LOCAL_PANEL"]
        else:
            os.environ["HG_LOCAL_PANEL"] = saved

    dev = torch.device("cuda")
    f64 = torch.float64
    L = int(sizes.max())
    # padded [subdomain][dof] layout <-> the handle's concatenated layout
    pad_idx = torch.full((nb, L), N, dtype=torch.long)
    imask = torch.zeros((nb, L), dtype=torch.bool)
    for i, g in enumerate(gevps):
        pad_idx[i, : sizes[i]] = torch.arange(offs[i], offs[i + 1])
        imask[i, torch.as_tensor(np.asarray(g.idof_in_ov), dtype=torch.long)] = True
    pad_idx, imask = pad_idx.to(dev), imask.to(dev)
    valid = pad_idx < N
    flat_pos = pad_idx[valid]

    def to_flat(X):  # (nb, L) -> (N,)
        out = torch.zeros(N, dtype=f64, device=dev)
        out[flat_pos] = X[valid]
        return out

    def to_pad(x):  # (N,) -> (nb, L)
        X = torch.zeros((nb, L), dtype=f64, device=dev)
        X[valid] = x[flat_pos]
        return X

    def cmul(X):  # C_i X per subdomain
        return to_pad(pre.spmv(to_flat(X), "Dk"))

    def amul(X):  # A_i X = R_I (B + gC)^{-1} C E_I X
        Y = to_pad(pre.apply(pre.spmv(to_flat(X), "Dk")))
        return torch.where(imask, Y, torch.zeros_like(Y))

    def cdot(X, CY):  # per-subdomain <X, Y>_C given CY = C Y
        return (X * CY).sum(dim=-1)

    nev = int(min(n_wanted + 1, int(imask.sum(1).min().item()) - 1))
    mmax = min(2 * nev + 10, int(imask.sum(1).min().item()))
    kk = min(nev + keep_extra, mmax - 2)
    V = torch.zeros((mmax + 1, nb, L), dtype=f64, device=dev)
    S = torch.zeros((nb, mmax + 1, mmax), dtype=f64, device=dev)
    gen = torch.Generator(device="cpu").manual_seed(seed)
    v0 = torch.randn((nb, L), generator=gen, dtype=f64).to(dev)
    v0 = torch.where(imask, v0, torch.zeros_like(v0))
    v0 = v0 / torch.sqrt(cdot(v0, cmul(v0)))[:, None]
    V[0] = v0
    j0 = 0
    done = torch.zeros(nb, dtype=torch.bool, device=dev)
    theta = Y = None
    for restart in range(max_restarts):
        for j in range(j0, mmax):
            w = amul(V[j])
            for _ in range(2):  # CGS2 in the C inner product, per subdomain
                Cw = cmul(w)
                h = torch.einsum("kbl,bl->bk", V[: j + 1], Cw)
                w = w - torch.einsum("bk,kbl->bl", h, V[: j + 1])
                S[:, : j + 1, j] += h
            beta = torch.sqrt(torch.clamp(cdot(w, cmul(w)), min=0.0))
            S[:, j + 1, j] = beta
            V[j + 1] = w / torch.where(beta > 0, beta, torch.ones_like(beta))[:, None]
        # Rayleigh-Ritz on the projected matrix of each subdomain
        Sm = S[:, :mmax, :mmax]
        theta, Y = torch.linalg.eigh(0.5 * (Sm + Sm.transpose(1, 2)))
        if restart == 0:  # a spectrum reaching below -g shows as a large negative Ritz value at once
            theta_min = theta[:, 0].clone()
        order = torch.argsort(theta, dim=1, descending=True)
        theta = torch.gather(theta, 1, order)
        Y = torch.gather(Y, 2, order[:, None, :].expand(-1, mmax, -1))
        res = torch.abs(torch.einsum("bj,bji->bi", S[:, mmax, :mmax], Y))
        scale = theta.abs().max(dim=1).values
        done = (res[:, :nev] <= tol * scale[:, None]).all(dim=1)
        if verbose:
            print("gevp_device restart %d: %d/%d subdomains converged, worst residual %.2e" % (
                restart, int(done.sum()), nb, float((res[:, :nev] / scale[:, None]).max())))
        if bool(done.all()):
            break
        # Krylov-Schur restart: keep the kk largest Ritz pairs
        Vk = torch.einsum("jbl,bjk->kbl", V[:mmax], Y[:, :, :kk])
        bvec = torch.einsum("bj,bjk->bk", S[:, mmax, :mmax], Y[:, :, :kk])
        vlast = V[mmax].clone()
        V.zero_()
        V[:kk] = Vk
        V[kk] = vlast
        S.zero_()
        idx = torch.arange(kk, device=dev)
        S[:, idx, idx] = theta[:, :kk]
        S[:, kk, :kk] = bvec  # A V_k = V_k Theta + v_kk b^T; column kk's couplings come from its CGS
        j0 = kk
    else:
        raise EigensolveError("device Lanczos did not converge in %d restarts" % max_restarts)

    # eigenvectors: q = V y (idof part), p = (B + gC)^{-1} C E_I q / mu, C-normalised
    mu = theta[:, :nev]
    Q = torch.einsum("jbl,bjk->kbl", V[:mmax], Y[:, :, :nev])  # (nev, nb, L)
    results = [None] * nb
    neg = ((mu <= 0).any(dim=1) | (-theta_min >= mu[:, -1])).cpu().numpy()
    P = torch.empty_like(Q)
    for k in range(nev):
        Pk = to_pad(pre.apply(pre.spmv(to_flat(Q[k]), "Dk"))) / mu[:, k][:, None]
        nrm = torch.sqrt(cdot(Pk, cmul(Pk)))
        P[k] = Pk / nrm[:, None]
    mu_h = mu.cpu().numpy()
    P_h = P.permute(1, 2, 0).cpu().numpy()  # (nb, L, nev)
    for i in range(nb):
        if neg[i]:  # spectrum below -g: the host path widens the shift (rare)
            results[i] = solve_gevp_lanczos(gevps[i], n_wanted)
            continue
        lam = 1.0 / mu_h[i] - shift
        order = np.argsort(lam, kind="stable")
        n_i = sizes[i]
        vecs = np.ascontiguousarray(P_h[i, :n_i, order].T)
        nI = int(np.asarray(gevps[i].idof_in_ov).size)
        results[i] = LocalGevpResult(gevps[i].subdomain_index, lam[order], vecs, int(np.sum(lam <= 0.0)),
                                     int(n_i - nI), float(shift), True, nI)
    pre.close()
    return results
