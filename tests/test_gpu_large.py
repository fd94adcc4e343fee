"""BASELINE configs 4 and 5 at full size (0.5M / 1M dofs) on the device,
checked against the REFERENCE's own solve (default-on).

The reference package is absent on the GPU box, so its results travel as
committed fixtures: tests/golden/large_<cfg>.npz, written by
oracle/gen_large.py, which runs helmdd's own TwoLevelPreconditioner
(schwarz.py:37-71, SuperLU + getrf factors) and helmdd.wgmres.weighted_gmres
(wgmres.py:74-203) on this package's host setup of the config — the solve
block of cli.run_single (cli.py:297-307).  Here the same setup is rebuilt
(seeded, deterministic) and the device path must match:

  * apply of the seeded r (and rhs_p = M^{-1} f) on the fixture's 1/16 dof
    sample, rel. to the vector's max norm <= 1e-10 — this also proves the
    rebuilt setup is the fixture's;
  * the full GMRES solve of rhs column 0, single RHS, both orthogonalisations
    (dcgs2 — the one bench.py times — and measured): iterations within +-1,
    history <= 1e-8 beta on the common prefix, x rel <= 1e-8 when the counts
    agree, and x rel <= 1e-8 in fixed-iteration mode (rtol = 0, maxit = the
    reference's count) regardless;
  * column 0 of the 16-RHS block solve (weighted_gmres_batch, the bench step)
    and of the C-ABI host path (hg_solve_host_batch, the bench's e2e);
  * size-independent properties: determinism, linearity, zero -> zero, each
    batched-apply column equal to the single apply, and the W-orthonormality
    of the hundreds-of-vectors Krylov basis (test_wgmres.py:35-52 at scale).
"""

import gc
import os

import numpy as np
import pytest

import paper_2406_06283_b200 as hg

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CONFIGS = ["4", "5-8", "5-16", "5-32"]
APPLY_RTOL, SOL_RTOL = 1e-10, 1e-8


def fixture(name):
    path = os.path.join(ROOT, "tests", "golden", "large_%s.npz" % name)
    if not os.path.exists(path):
        pytest.fail("fixture %s missing: run python -m oracle.gen_large %s where /root/reference exists" % (path, name))
    return np.load(path)


def rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300))


def check_solve(x, rep, fx, what):
    it_ref = int(fx["iterations"])
    h_ref = fx["history"]
    assert abs(rep.iterations - it_ref) <= 1, "%s: %d iterations vs the reference's %d" % (what, rep.iterations, it_ref)
    k = min(rep.iterations, it_ref) + 1
    dh = np.abs(rep.residual_history[:k] - h_ref[:k]).max()
    assert dh <= 1e-8 * h_ref[0], "%s: history deviates by %.3e beta" % (what, dh / h_ref[0])
    if rep.iterations == it_ref:
        assert rel(x, fx["x"]) <= SOL_RTOL, "%s: x rel %.3e" % (what, rel(x, fx["x"]))
    return rel(x, fx["x"]) if rep.iterations == it_ref else None


@pytest.mark.parametrize("name", CONFIGS)
def test_full_size_parity_vs_reference(name):
    import torch

    fx = fixture(name)
    P = hg.build_problem(name, cstab="cache")
    # setup fingerprint: the rebuilt coarse space is the fixture's
    assert list(P.selection.m_per_subdomain) == list(fx["m_per"])
    assert P.coarse.m_total == int(fx["m_total"])
    last = np.array([r.eigenvalues[m - 1] for r, m in zip(P.results, P.selection.m_per_subdomain)])
    assert np.abs(last - fx["lam_last"]).max() <= 1e-9 * np.abs(fx["lam_last"]).max()

    pre = hg.factorize(P.forms, P.dec, P.coarse)
    print("%s: panel local solve active %s (deviation %.2e)" % (name, pre.panel_active, pre.panel_deviation))
    n = pre.n
    sub = fx["sub"]
    B, Dk = P.forms.helmholtz, P.forms.dk
    F = P.rhs if P.rhs.ndim == 2 else P.rhs[:, None]
    f = np.ascontiguousarray(F[:, 0])
    rng = np.random.default_rng(int(fx["r_seed"]))
    r = rng.standard_normal(n)

    # ---- applies vs the reference (schwarz.py:51-61)
    got = pre.apply(r)
    err_apply = float(np.abs(got[sub] - fx["apply_r_sub"]).max() / float(fx["apply_r_max"]))
    assert err_apply <= APPLY_RTOL, "apply rel %.3e" % err_apply
    assert abs(np.linalg.norm(got) - float(fx["apply_r_nrm"])) <= 1e-10 * float(fx["apply_r_nrm"])
    rhs_p = pre.apply(f)
    err_rhs = float(np.abs(rhs_p[sub] - fx["rhs_p_sub"]).max() / float(fx["rhs_p_max"]))
    assert err_rhs <= APPLY_RTOL, "rhs_p rel %.3e" % err_rhs

    # ---- size-independent properties
    assert np.array_equal(pre.apply(r), got)
    u = np.random.default_rng(7).standard_normal(n)
    lin = pre.apply(0.5 * r - 2.0 * u)
    assert np.abs(lin - (0.5 * got - 2.0 * pre.apply(u))).max() <= 1e-12 * np.abs(lin).max()
    assert np.all(pre.apply(np.zeros(n)) == 0.0)
    R = np.stack([r, u] + [F[:, c] for c in range(min(F.shape[1], 6))], axis=1)
    Rm = pre.apply_multi(R)
    for c in range(R.shape[1]):
        assert rel(Rm[:, c], pre.apply(R[:, c])) <= 1e-11  # panel local solve (hg_local_panel.cu)

    # ---- full single-RHS solves, both orthogonalisations (wgmres.py:74-203)
    op = pre.as_operator("T")
    it_ref = int(fx["iterations"])
    errs = {}
    for orth in ("dcgs2", "measured"):
        x, rep = hg.weighted_gmres(op, rhs_p, weight=Dk, rtol=P.config.rtol, maxit=P.config.maxit, orth=orth)
        assert rep.converged
        errs[orth] = check_solve(x, rep, fx, "%s single %s" % (name, orth))
        xf, repf = hg.weighted_gmres(op, rhs_p, weight=Dk, rtol=0.0, maxit=it_ref, orth=orth)
        assert repf.iterations == it_ref
        assert rel(xf, fx["x"]) <= SOL_RTOL, "%s fixed-iteration %s: x rel %.3e" % (name, orth, rel(xf, fx["x"]))

    # W-orthonormality of the full basis of the last dcgs2 solve (on the device)
    x, rep = hg.weighted_gmres(op, rhs_p, weight=Dk, rtol=P.config.rtol, maxit=P.config.maxit, orth="dcgs2")
    m = rep.iterations
    Q = op.basis(m)
    WQ = torch.stack([pre.spmv(Q[i], "Dk") for i in range(m)])
    gram = Q @ WQ.T
    ortho = float((gram - torch.eye(m, dtype=gram.dtype, device=gram.device)).abs().max())
    del Q, WQ, gram
    assert ortho <= 1e-10, "basis W-orthonormality %.3e over %d vectors" % (ortho, m)
    op.release()

    # ---- the bench's block solve (16 columns in lock step) and its C-ABI host path
    Fd = torch.from_numpy(np.ascontiguousarray(F.T)).cuda()
    Rp = pre.apply_multi(Fd)
    X, reps = hg.weighted_gmres_batch(op, Rp, weight=Dk, rtol=P.config.rtol, maxit=P.config.maxit, orth="dcgs2")
    assert all(rp.converged for rp in reps)
    check_solve(X[0].cpu().numpy(), reps[0], fx, "%s block column 0" % name)
    del X, Rp
    op.release()
    Xh, reps_h = pre.solve_host_batch(F, rtol=P.config.rtol, maxit=P.config.maxit)
    check_solve(Xh[:, 0], reps_h[0], fx, "%s hg_solve_host_batch column 0" % name)
    print("%s: reference %d iterations; apply rel %.2e, rhs_p rel %.2e, x rel %s, basis orthonormality %.1e"
          % (name, it_ref, err_apply, err_rhs, errs, ortho))
    del op, pre
    gc.collect()
    torch.cuda.empty_cache()
