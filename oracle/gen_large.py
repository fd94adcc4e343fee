"""Full-size parity fixtures for BASELINE configs 4 and 5 (TEST INFRASTRUCTURE).

Run in the build container, where /root/reference exists:

    python -m oracle.gen_large 5-16 [4 5-8 5-32 ...]

For each configuration the setup is this package's host restatement
(problems.build_problem; the reference's own setup takes hours at these
sizes), and the SOLVE is the reference's own code, imported
read-only from /root/reference/pkg/src:

  * helmdd.schwarz.TwoLevelPreconditioner (schwarz.py:37-71) built from
    SuperLU factors of every fine block (schwarz.py:104-110, without the
    report-only _smallest_eigenvalue) and lu_factor(B0) (schwarz.py:88-90);
  * helmdd.wgmres.weighted_gmres (wgmres.py:74-203) on
    op = lambda v: precond.apply(forms.helmholtz @ v), rhs_p = precond.apply(f),
    weight = forms.dk — the solve block of cli.run_single (cli.py:297-307).

Written to tests/golden/large_<name>.npz (the GPU box has no /root/reference,
so the test reads these):

  x, history, iterations, converged   the reference's converged solve of rhs column 0
  sub, apply_r_sub, apply_r_max       M^{-1} r for r = N(0,1) seed 2406 on a seeded
                                      1/16 sample of the dofs (+ global max |.|, norm)
  rhs_p_sub, rhs_p_max                M^{-1} f on the same sample
  m_per, tau, lam_last, lam_next, ... setup fingerprints: if the box's setup drifts
                                      from this one, the apply check says so first
"""

import os
import platform
import sys
import time

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/pkg/src"
OUT = os.path.join(ROOT, "tests", "golden")
R_SEED = 2406
SAMPLE_SEED = 11


def fixture_path(name):
    return os.path.join(OUT, "large_%s.npz" % name)


def sample_indices(n):
    """The seeded 1/16 dof sample the apply checks compare on."""
    return np.sort(np.random.default_rng(SAMPLE_SEED).choice(n, size=max(1, n // 16), replace=False))


def _reference_preconditioner(h, forms, dec, coarse):
    """helmdd's own TwoLevelPreconditioner from SuperLU + getrf factors."""
    import scipy.linalg
    from helmdd.schwarz import LocalSolver, TwoLevelPreconditioner

    Bc = forms.helmholtz.tocsc()
    solvers = []
    for i, j, sub in dec.fine_flat():
        idof = np.asarray(sub.idof)
        lu = spla.splu(Bc[idof][:, idof].tocsc()) if idof.size else None
        solvers.append(LocalSolver(i, j, idof, lu, True, getattr(sub, "diameter", np.nan), np.nan))
    b0_piv = scipy.linalg.lu_factor(np.asarray(coarse.B0))
    return TwoLevelPreconditioner(forms, solvers, Z=sp.csc_matrix(coarse.Z), b0_piv=b0_piv)


def setup_fingerprint(P):
    """Cheap numbers that pin the setup a fixture was generated from."""
    sel = P.selection
    last, nxt = [], []
    for res, m in zip(P.results, sel.m_per_subdomain):
        ev = res.eigenvalues
        last.append(ev[m - 1] if m >= 1 else np.nan)
        nxt.append(ev[m] if m < ev.size else np.nan)
    z_abs = sum(float(np.abs(b).sum()) for _, b in P.coarse.blocks)
    return dict(
        m_per=np.asarray(sel.m_per_subdomain), m_total=P.coarse.m_total, tau=sel.tau, cstab=P.cstab,
        tau_target=P.tau_target, lam_last=np.asarray(last), lam_next=np.asarray(nxt), z_abs=z_abs,
        b0_fro=float(np.linalg.norm(P.coarse.B0)), b0_trace=float(np.trace(P.coarse.B0)),
    )


def gen(name, workers=None):
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import helmdd  # noqa: F401
    from helmdd.wgmres import weighted_gmres

    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)
    from paper_2406_06283_b200.problems import build_problem

    t0 = time.perf_counter()
    P = build_problem(name, cstab="cache", workers=workers, verbose=True)
    t_setup = time.perf_counter() - t0
    forms = P.forms
    n = forms.n_dofs
    t0 = time.perf_counter()
    pre = _reference_preconditioner(helmdd, forms, P.dec, P.coarse)
    t_factor = time.perf_counter() - t0
    F = P.rhs if P.rhs.ndim == 2 else P.rhs[:, None]
    f = np.ascontiguousarray(F[:, 0])
    r = np.random.default_rng(R_SEED).standard_normal(n)
    sub = sample_indices(n)
    t0 = time.perf_counter()
    ar = pre.apply(r)
    t_apply = time.perf_counter() - t0
    rhs_p = pre.apply(f)
    # the solve block of cli.run_single (cli.py:297-307)
    op = lambda v: pre.apply(forms.helmholtz @ v)  # noqa: E731
    t0 = time.perf_counter()
    x, rep = weighted_gmres(op, rhs_p, weight=forms.dk, rtol=P.config.rtol, maxit=P.config.maxit)
    t_solve = time.perf_counter() - t0
    print("%s: reference solve %d iterations in %.1f s (apply %.2f s)" % (name, rep.iterations, t_solve, t_apply),
          flush=True)
    np.savez_compressed(
        fixture_path(name),
        name=name, n=n, r_seed=R_SEED, sample_seed=SAMPLE_SEED, sub=sub,
        apply_r_sub=ar[sub], apply_r_max=np.abs(ar).max(), apply_r_nrm=np.linalg.norm(ar),
        rhs_p_sub=rhs_p[sub], rhs_p_max=np.abs(rhs_p).max(), rhs_p_nrm=np.linalg.norm(rhs_p),
        x=x, history=rep.residual_history, iterations=rep.iterations, converged=rep.converged,
        breakdown=bool(getattr(rep, "breakdown", False)),
        t_setup=t_setup, t_factor=t_factor, t_apply=t_apply, t_solve=t_solve,
        host=platform.processor() or platform.machine(), **setup_fingerprint(P),
    )
    print("wrote", fixture_path(name), flush=True)


if __name__ == "__main__":
    names = sys.argv[1:] or ["4", "5-8", "5-16", "5-32"]
    for nm in names:
        gen(nm)
