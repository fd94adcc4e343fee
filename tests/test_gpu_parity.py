"""Parity of the device solve phase against the reference (golden vectors)
and the CPU oracle.  Bars (BASELINE north star): apply rel. error <= 1e-10,
GMRES iterations within +-1, solution rel. error <= 1e-8; SpMV bitwise."""

import numpy as np
import pytest
import scipy.sparse as sp

import paper_2406_06283_b200 as hg
from _helpers import golden_coarse
from oracle.schwarz_oracle import OraclePreconditioner
from oracle.wgmres_oracle import weighted_gmres as oracle_gmres

pytestmark = pytest.mark.gpu

APPLY_RTOL = 1e-10
SOL_RTOL = 1e-8


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.fixture(scope="module")
def cfg1(golden):
    g = golden("config1")
    P = hg.build_problem("1", workers=1, one_level=True)
    coarse = golden_coarse(g, P.forms.n_dofs)
    pre = hg.factorize(P.forms, P.dec, coarse)
    return P, g, coarse, pre


ORTHS = ["dcgs2", "measured"]


def test_spmv_bitwise(cfg1):
    P, g, _, pre = cfg1
    assert np.array_equal(pre.spmv(g["u"], "B"), g["Bu"])
    assert np.array_equal(pre.spmv(g["u"], "Dk"), g["Dku"])


def test_apply_matches_reference(cfg1):
    P, g, _, pre = cfg1
    assert rel(pre.apply(g["r"]), g["apply_r"]) <= APPLY_RTOL
    assert rel(pre.apply_T(g["u"]), g["apply_T_u"]) <= APPLY_RTOL
    assert rel(pre.apply_coarse(g["r"]), g["apply_coarse_r"]) <= APPLY_RTOL


def test_one_level_matches_reference(cfg1):
    P, g, _, _ = cfg1
    pre1 = hg.factorize(P.forms, P.dec, None)
    assert not pre1.has_coarse
    assert rel(pre1.apply(g["r"]), g["apply_one_level_r"]) <= APPLY_RTOL
    assert np.all(pre1.apply_coarse(g["r"]) == 0.0)


def test_zero_maps_to_zero(cfg1):
    _, _, _, pre = cfg1
    assert np.all(pre.apply(np.zeros(pre.n)) == 0.0)


def test_apply_deterministic_and_linear(cfg1):
    _, g, _, pre = cfg1
    rng = np.random.default_rng(8)
    u, v = rng.standard_normal(pre.n), rng.standard_normal(pre.n)
    a1, a2 = pre.apply(u), pre.apply(u)
    assert np.array_equal(a1, a2)
    lhs = pre.apply(0.3 * u - 1.7 * v)
    rhs = 0.3 * a1 - 1.7 * pre.apply(v)
    assert np.abs(lhs - rhs).max() <= 1e-12 * np.abs(rhs).max()


def test_torch_tensors_stay_on_device(cfg1):
    import torch

    _, g, _, pre = cfg1
    t = torch.from_numpy(g["r"]).cuda()
    out = pre.apply(t)
    assert isinstance(out, torch.Tensor) and out.is_cuda
    assert rel(out.cpu().numpy(), g["apply_r"]) <= APPLY_RTOL


def test_empty_coarse_equals_one_level_bitwise(cfg1):
    P = cfg1[0]
    empty = type("C", (), {"m_total": 0, "Z": sp.csc_matrix((P.forms.n_dofs, 0)), "B0": np.zeros((0, 0)),
                           "column_meta": []})()
    a = hg.factorize(P.forms, P.dec, empty)
    b = hg.factorize(P.forms, P.dec, None)
    r = np.random.default_rng(7).standard_normal(P.forms.n_dofs)
    assert np.array_equal(a.apply(r), b.apply(r))


def test_local_solves_match_lapack(cfg1):
    _, _, _, pre = cfg1
    rng = np.random.default_rng(10)
    for ls in pre.local_solvers:
        r = rng.standard_normal(ls.idof.size)
        got = ls.lu.solve(r)
        want = ls.lu.host.solve(r)
        assert rel(got, want) <= 1e-12


def test_local_solves_mixed_bandwidth():
    """BASELINE config 4 (one level): boundary blocks are narrower (kl 47 vs
    49, kv 94 vs 98) than the launch's register tiles; their zero-padded
    records must give the host band LU's solution on every block."""
    P = hg.build_problem("4", one_level=True)
    pre = hg.factorize(P.forms, P.dec, None)
    bands = {(f.lu.host.kl, f.lu.host.kv) for f in pre.local_solvers}
    assert len(bands) > 1
    rng = np.random.default_rng(40)
    for ls in pre.local_solvers:
        r = rng.standard_normal(ls.idof.size)
        assert rel(ls.lu.solve(r), ls.lu.host.solve(r)) <= 1e-12
    r = rng.standard_normal(pre.n)
    orc = OraclePreconditioner(P.forms, P.dec, None)
    assert rel(pre.apply(r), orc.apply(r)) <= APPLY_RTOL


@pytest.mark.parametrize("orth", ORTHS)
def test_gmres_matches_reference(cfg1, orth):
    P, g, _, pre = cfg1
    rhs_p = pre.apply(P.rhs)
    assert rel(rhs_p, g["rhs_p"]) <= APPLY_RTOL
    x, rep = hg.weighted_gmres(pre.as_operator("T"), rhs_p, weight=P.forms.dk, rtol=1e-6, maxit=1000, orth=orth)
    assert rep.converged
    assert abs(rep.iterations - int(g["iterations"])) <= 1
    assert rel(x, g["x"]) <= SOL_RTOL
    h = g["history"]
    k = min(h.size, rep.residual_history.size)
    assert np.abs(rep.residual_history[:k] - h[:k]).max() <= 1e-8 * h[0]
    # fixed-iteration mode: no stopping-rule slack can hide drift
    xf, repf = hg.weighted_gmres(pre.as_operator("T"), rhs_p, weight=P.forms.dk, rtol=0.0,
                                 maxit=int(g["iterations"]), orth=orth)
    assert repf.iterations == int(g["iterations"])
    assert rel(xf, g["x_fixed"]) <= SOL_RTOL


def test_solve_host_end_to_end(cfg1):
    P, g, _, pre = cfg1
    x, rep = pre.solve_host(P.rhs, rtol=1e-6, maxit=1000)
    assert abs(rep.iterations - int(g["iterations"])) <= 1
    assert rel(x, g["x"]) <= SOL_RTOL


@pytest.mark.parametrize("orth", ORTHS)
def test_one_level_gmres_iterations(cfg1, golden, orth):
    P, g, _, _ = cfg1
    pre1 = hg.factorize(P.forms, P.dec, None)
    x, rep = hg.weighted_gmres(pre1.as_operator("T"), pre1.apply(P.rhs), weight=P.forms.dk, rtol=1e-6, maxit=1000,
                               orth=orth)
    assert abs(rep.iterations - int(g["iterations_one_level"])) <= 1
    assert rel(x, g["x_one_level"]) <= SOL_RTOL


def test_small_pipelines(golden):
    g = golden("small")
    for tag, (n, M, q, k) in {"p8": (8, 2, 2, 5.0), "p16": (16, 2, 2, 10.0)}.items():
        mesh = hg.build_unit_square_mesh(n)
        space = hg.build_fe_space(mesh)
        forms = hg.assemble_forms(mesh, space, hg.coefficient_field(mesh), k)
        dec = hg.build_two_level(mesh, space, M, q)
        res = [hg.solve_indefinite_gevp(hg.assemble_local_gevp(i, forms, dec)) for i in range(dec.n_coarse)]
        coarse = hg.build_coarse_space(res, hg.select_modes(res, 1.0), dec, forms)
        pre = hg.factorize(forms, dec, coarse)
        assert rel(pre.apply(g[tag + "_r"]), g[tag + "_apply"]) <= 1e-10
        assert rel(pre.apply_coarse(g[tag + "_r"]), g[tag + "_apply_coarse"]) <= 1e-10
    mesh = hg.build_unit_square_mesh(8)
    space = hg.build_fe_space(mesh)
    forms = hg.assemble_forms(mesh, space, hg.coefficient_field(mesh), 4.0)
    pre = hg.factorize(forms, hg.build_two_level(mesh, space, 2, 1), None)
    assert rel(pre.apply(g["one_r"]), g["one_apply"]) <= 1e-12
    forms = hg.assemble_forms(mesh, space, hg.coefficient_field(mesh), 3.0)
    pre = hg.factorize(forms, hg.build_two_level(mesh, space, 1, 1), None)
    got = pre.apply_T(g["deg_v"])
    assert np.abs(got - g["deg_v"]).max() <= 1e-10 * np.abs(g["deg_v"]).max()
    assert rel(got, g["deg_apply_Bv"]) <= 1e-10


@pytest.mark.parametrize("orth", ORTHS)
def test_gmres_seeded_systems(golden, orth):
    g = golden("wgmres")
    for m in (5, 12, 25):
        x, rep = hg.weighted_gmres(g["A30"], g["b30"], rtol=0.0, maxit=m, orth=orth)
        assert rep.iterations == m
        assert np.abs(x - g["x30_%d" % m]).max() <= 1e-10 * max(np.abs(g["x30_%d" % m]).max(), 1.0)
        assert np.abs(rep.residual_history - g["h30_%d" % m]).max() <= 1e-10 * g["h30_%d" % m][0]
    x, rep = hg.weighted_gmres(g["A50"], g["b50"], weight=sp.csr_matrix(g["W50"]), rtol=1e-10, maxit=50, orth=orth)
    assert rep.converged and abs(rep.iterations - int(g["it50"])) <= (0 if orth == "measured" else 1)
    assert rel(x, g["x50"]) <= 1e-10
    hist = rep.residual_history
    assert np.all(np.diff(hist) <= 1e-14 * hist[0])
    r = g["b50"] - g["A50"] @ x
    assert abs(np.sqrt(r @ (g["W50"] @ r)) - hist[-1]) <= 1e-8 * hist[0]


@pytest.mark.parametrize("orth", ORTHS)
def test_gmres_edge_cases(orth):
    rng = np.random.default_rng(0)
    b = rng.standard_normal(40)
    gm = lambda *a, **k: hg.weighted_gmres(*a, orth=orth, **k)  # noqa: E731
    x, rep = gm(np.eye(40), b, rtol=1e-12, maxit=10)
    assert rep.iterations == 1 and rep.converged and np.abs(x - b).max() <= 1e-12
    A = np.diag([2.0, 2.0, 5.0])
    x, rep = gm(A, np.ones(3), rtol=1e-13, maxit=10)
    assert rep.iterations <= 2 and rep.converged and np.abs(A @ x - 1.0).max() <= 1e-12
    x, rep = gm(np.eye(4), np.zeros(4), maxit=4)
    assert rep.converged and rep.iterations == 0 and np.all(x == 0.0)
    A = rng.standard_normal((40, 40)) + 40 * np.eye(40)
    x, rep = gm(A, b, rtol=1e-14, maxit=3)
    assert rep.iterations == 3 and not rep.converged
    x0 = rng.standard_normal(40)
    x, rep = gm(A, b, rtol=1e-12, maxit=40, x0=x0)
    assert rep.converged and np.abs(A @ x - b).max() <= 1e-9 * np.abs(b).max()
    x, rep = gm(A, b, rtol=1e-10, maxit=20, gamma=0.5)
    assert rep.elman_envelope.size == rep.iterations + 1
    with pytest.raises(TypeError):
        hg.weighted_gmres(lambda v: v, b)


@pytest.mark.parametrize("name", ["2", "3"])
@pytest.mark.parametrize("orth", ORTHS)
def test_config_parity_vs_oracle(name, orth):
    P = hg.build_problem(name)
    pre = hg.factorize(P.forms, P.dec, P.coarse)
    orc = OraclePreconditioner(P.forms, P.dec, P.coarse)
    r = np.random.default_rng(11).standard_normal(P.forms.n_dofs)
    assert rel(pre.apply(r), orc.apply(r)) <= APPLY_RTOL
    B, Dk = P.forms.helmholtz, P.forms.dk
    rhs = P.rhs
    x, rep = hg.weighted_gmres(pre.as_operator("T"), pre.apply(rhs), weight=Dk, rtol=1e-6, maxit=1000, orth=orth)
    xo, info = oracle_gmres(lambda v: orc.apply(B @ v), orc.apply(rhs), weight=Dk, rtol=1e-6, maxit=1000)
    assert rep.converged and info["converged"]
    assert abs(rep.iterations - info["iterations"]) <= 1
    assert rel(x, xo) <= SOL_RTOL


def _small_pipeline(n, M, q, k):
    mesh = hg.build_unit_square_mesh(n)
    space = hg.build_fe_space(mesh)
    forms = hg.assemble_forms(mesh, space, hg.coefficient_field(mesh), k)
    return forms, hg.build_two_level(mesh, space, M, q)


def test_spd_flags_for_small_k():
    """test_schwarz.py:118-124 on the device factorisation."""
    forms, dec = _small_pipeline(8, 2, 2, 1.0)
    pre = hg.factorize(forms, dec, None)
    assert all(ls.spd_flag for ls in pre.local_solvers)
    assert all(ls.min_eig > 0 for ls in pre.local_solvers)


def test_factorization_consistency_device_solves():
    """test_schwarz.py:127-138 through the device local solves (ls.lu.solve)."""
    forms, dec = _small_pipeline(8, 2, 2, 5.0)
    pre = hg.factorize(forms, dec, None)
    B = forms.helmholtz.tocsr()
    rng = np.random.default_rng(10)
    for ls in pre.local_solvers:
        block = B[ls.idof][:, ls.idof]
        x = rng.standard_normal(ls.idof.size)
        back = ls.lu.solve(np.asarray(block @ x))
        assert np.abs(back - np.asarray(block @ ls.lu.solve(x))).max() <= 1e-9
        y = ls.lu.solve(x)
        assert np.abs(np.asarray(block @ y) - x).max() <= 1e-10 * np.abs(x).max()


@pytest.mark.parametrize("orth", ORTHS)
def test_weighted_basis_orthonormality(orth):
    """test_wgmres.py:35-52: the Krylov basis is W-orthonormal to 1e-10 over
    50 iterations (basis read back through hg_op_basis)."""
    rng = np.random.default_rng(2)
    n = 60
    A = rng.standard_normal((n, n)) + n * np.eye(n)  # the reference's _random_system
    b = rng.standard_normal(n)
    G = rng.standard_normal((n, n))
    W = sp.csr_matrix(G @ G.T + n * np.eye(n))
    op = hg.CsrOperator(A)
    x, rep = hg.weighted_gmres(op, b, weight=W, rtol=0.0, maxit=50, orth=orth)
    assert rep.iterations == 50
    V = op.basis(50).cpu().numpy().T
    gram = V.T @ (W @ V)
    assert np.abs(gram - np.eye(50)).max() <= 1e-10
    B = np.stack([b, rng.standard_normal(n)], axis=1)
    X, reps = hg.weighted_gmres_batch(op, B, weight=W, rtol=0.0, maxit=40, orth=orth)
    for c in range(2):
        Vc = op.basis(40, col=c).cpu().numpy().T
        assert np.abs(Vc.T @ (W @ Vc) - np.eye(40)).max() <= 1e-10


def test_local_solutions_match_block_solves(cfg1):
    """hg_precond_local_solutions: every block's x_s = B_s^{-1} R_s r before assembly equals the
    block-by-block LocalSolver.lu.solve (schwarz.py:58-60), and summing them is the one-level apply."""
    import ctypes

    import torch

    from paper_2406_06283_b200 import _lib

    P, g, coarse, pre = cfg1
    r = np.random.default_rng(8).standard_normal(pre.n)
    rd = torch.from_numpy(r).cuda()
    xs = torch.empty(pre.xs_len, dtype=torch.float64, device="cuda")
    _lib.check(_lib.load().hg_precond_local_solutions(pre._handle, ctypes.c_void_p(rd.data_ptr()),
                                                      ctypes.c_void_p(xs.data_ptr()), None), "local_solutions")
    xs = xs.cpu().numpy()
    pos = 0
    acc = np.zeros(pre.n)
    for ls in pre.local_solvers:
        n = ls.idof.size
        assert np.array_equal(xs[pos:pos + n], ls.lu.solve(r[ls.idof]))
        np.add.at(acc, ls.idof, xs[pos:pos + n])
        pos += n
    assert pos == pre.xs_len
