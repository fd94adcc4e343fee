"""Regenerate tests/golden/*.npz from the REFERENCE package (TEST INFRASTRUCTURE).

Run in the build container, where /root/reference exists:

    python -m oracle.gen_golden

Every number stored here is produced by helmdd itself (imported read-only
from /root/reference/pkg/src); inputs are seeded so tests can rebuild them.
Files:
  config1.npz   BASELINE config 1 through the reference pipeline of
                cli.run_single (cli.py:224-307): C_stab, tau, Z, B0, apply /
                apply_T / apply_coarse on seeded vectors, GMRES x + history.
  small.npz     the pipelines of pkg/tests/test_schwarz.py (_pipeline and
                the one-level / degenerate cases) with applies on seeded r.
  wgmres.npz    reference weighted_gmres on the seeded random systems of
                pkg/tests/test_wgmres.py.
  analysis.npz  helmdd.analysis check_tf_stability / check_prop26_identity on
                the setups of pkg/tests/test_analysis.py:300-323 and
                check_t0_stability on the test_schwarz pipeline (n=16, k=10).
"""

import os
import sys

import numpy as np
import scipy.sparse as sp

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def _ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import helmdd

    return helmdd


def _pipeline(h, n, M, q, k, tau_target=1.0, layers=1):
    mesh = h.build_unit_square_mesh(n)
    space = h.build_fe_space(mesh)
    forms = h.assemble_forms(mesh, space, h.coefficient_field(mesh), k=k)
    dec = h.build_two_level(mesh, space, M, q, layers, layers)
    res = [h.solve_indefinite_gevp(h.assemble_local_gevp(i, forms, dec)) for i in range(dec.n_coarse)]
    sel = h.select_modes(res, tau_target)
    return forms, dec, h.build_coarse_space(res, sel, dec, forms)


def gen_config1(h):
    from helmdd import analysis

    mesh = h.build_unit_square_mesh(80)
    space = h.build_fe_space(mesh)
    forms = h.assemble_forms(mesh, space, h.coefficient_field(mesh), 10.0)
    rhs = h.assemble_rhs(mesh, space, lambda x, y: np.ones_like(x))
    cstab = analysis.estimate_cstab(forms)
    dec = h.build_two_level(mesh, space, 4, 1, 2, 2)
    res = [h.solve_indefinite_gevp(h.assemble_local_gevp(i, forms, dec)) for i in range(dec.n_coarse)]
    tau_target = 2e-5 * (1.0 + cstab) ** 2 * 10.0**2
    sel = h.select_modes(res, tau_target, [30] * dec.n_coarse)
    coarse = h.build_coarse_space(res, sel, dec, forms)
    pre = h.factorize(forms, dec, coarse)
    rng = np.random.default_rng(0)
    r = rng.standard_normal(forms.n_dofs)
    u = rng.standard_normal(forms.n_dofs)
    op = lambda v: pre.apply(forms.helmholtz @ v)
    rhs_p = pre.apply(rhs)
    x, rep = h.weighted_gmres(op, rhs_p, weight=forms.dk, rtol=1e-6, maxit=1000)
    x_fixed, rep_fixed = h.weighted_gmres(op, rhs_p, weight=forms.dk, rtol=0.0, maxit=rep.iterations)
    pre1 = h.factorize(forms, dec, None)
    x1, rep1 = h.weighted_gmres(lambda v: pre1.apply(forms.helmholtz @ v), pre1.apply(rhs), weight=forms.dk,
                                rtol=1e-6, maxit=1000)
    Z = sp.csc_matrix(coarse.Z)
    B = forms.helmholtz
    np.savez_compressed(
        os.path.join(OUT, "config1.npz"),
        B_indptr=B.indptr, B_indices=B.indices, B_data=B.data, Dk_data=forms.dk.data,
        rhs=rhs, cstab=cstab, tau_target=tau_target, tau=sel.tau, m_per=np.array(sel.m_per_subdomain),
        eig_low=np.concatenate([rr.eigenvalues[:8] for rr in res]),
        Z_indptr=Z.indptr, Z_indices=Z.indices, Z_data=Z.data, B0=coarse.B0,
        r=r, u=u, apply_r=pre.apply(r), apply_T_u=pre.apply_T(u), apply_coarse_r=pre.apply_coarse(r),
        apply_one_level_r=pre1.apply(r), Bu=B @ u, Dku=forms.dk @ u,
        rhs_p=rhs_p, x=x, history=rep.residual_history, iterations=rep.iterations,
        x_fixed=x_fixed, history_fixed=rep_fixed.residual_history,
        x_one_level=x1, iterations_one_level=rep1.iterations,
    )


def gen_small(h):
    out = {}
    rng = np.random.default_rng(5)
    # test_schwarz._pipeline cases (n, M, q, k)
    for tag, (n, M, q, k) in {"p8": (8, 2, 2, 5.0), "p16": (16, 2, 2, 10.0)}.items():
        forms, dec, coarse = _pipeline(h, n, M, q, k)
        pre = h.factorize(forms, dec, coarse)
        r = rng.standard_normal(forms.n_dofs)
        out[tag + "_r"] = r
        out[tag + "_apply"] = pre.apply(r)
        out[tag + "_apply_coarse"] = pre.apply_coarse(r)
        out[tag + "_m"] = coarse.m_total
        out[tag + "_B0"] = coarse.B0
    # one-level 4 subdomains (test_one_level_matches_dense_oracle)
    mesh = h.build_unit_square_mesh(8)
    space = h.build_fe_space(mesh)
    forms = h.assemble_forms(mesh, space, h.coefficient_field(mesh), k=4.0)
    dec = h.build_two_level(mesh, space, 2, 1)
    pre = h.factorize(forms, dec, None)
    r = rng.standard_normal(forms.n_dofs)
    out["one_r"] = r
    out["one_apply"] = pre.apply(r)
    # degenerate M = q = 1 (test_exact_degenerate_case)
    forms = h.assemble_forms(mesh, space, h.coefficient_field(mesh), k=3.0)
    dec = h.build_two_level(mesh, space, 1, 1)
    pre = h.factorize(forms, dec, None)
    v = np.random.default_rng(0).standard_normal(space.n_dofs)
    out["deg_v"] = v
    out["deg_apply_Bv"] = pre.apply(forms.helmholtz @ v)
    np.savez_compressed(os.path.join(OUT, "small.npz"), **out)


def gen_wgmres(h):
    out = {}
    rng = np.random.default_rng(1)
    A = rng.standard_normal((30, 30)) + 30 * np.eye(30)
    b = rng.standard_normal(30)
    out["A30"], out["b30"] = A, b
    for m in (5, 12, 25):
        x, rep = h.weighted_gmres(A, b, weight=None, rtol=0.0, maxit=m)
        out["x30_%d" % m], out["h30_%d" % m] = x, rep.residual_history
    rng = np.random.default_rng(3)
    A = rng.standard_normal((50, 50)) + 50 * np.eye(50)
    b = rng.standard_normal(50)
    G = rng.standard_normal((50, 50))
    W = G @ G.T + 50 * np.eye(50)
    x, rep = h.weighted_gmres(A, b, weight=W, rtol=1e-10, maxit=50)
    out.update(A50=A, b50=b, W50=W, x50=x, h50=rep.residual_history, it50=rep.iterations)
    np.savez_compressed(os.path.join(OUT, "wgmres.npz"), **out)


ANALYSIS_T0_THEORY = dict(k=10.0, lambda_overlap=1, theta=1e-6, cstab_estimate=1.0)


def gen_analysis(h):
    """helmdd.analysis lemma checks on the reference's own test setups
    (test_analysis.py:300-323) plus a coarse-stability case with a theory
    whose hypothesis holds (so every trial is asserted)."""
    import types

    from helmdd import analysis

    out = {}

    def store(tag, chk):
        out[tag + "_trials"] = chk.trials
        out[tag + "_violations"] = chk.violations
        out[tag + "_worst"] = chk.worst_margin
        out[tag + "_witness"] = chk.witness

    mesh = h.build_unit_square_mesh(8)
    space = h.build_fe_space(mesh)
    forms = h.assemble_forms(mesh, space, h.coefficient_field(mesh), 0.5)
    dec = h.build_two_level(mesh, space, 2, 2)
    store("tf", analysis.check_tf_stability(forms, dec, h.factorize(forms, dec, None), trials=10,
                                            rng=np.random.default_rng(5)))
    forms = h.assemble_forms(mesh, space, h.coefficient_field(mesh), 5.0)
    store("prop26", analysis.check_prop26_identity(forms, h.factorize(forms, dec, None), trials=20,
                                                   rng=np.random.default_rng(6)))
    forms, dec, coarse = _pipeline(h, 16, 2, 2, 10.0)
    theory = types.SimpleNamespace(**ANALYSIS_T0_THEORY)
    store("t0", analysis.check_t0_stability(forms, coarse, h.factorize(forms, dec, coarse), theory, trials=20,
                                            rng=np.random.default_rng(7)))
    np.savez_compressed(os.path.join(OUT, "analysis.npz"), **out)


def main():
    os.makedirs(OUT, exist_ok=True)
    h = _ref()
    gen_small(h)
    gen_wgmres(h)
    gen_config1(h)
    gen_analysis(h)
    print("golden vectors written to", OUT)


if __name__ == "__main__":
    main()
