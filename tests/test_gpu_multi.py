"""Multi-RHS (batched) solve phase, SURVEY §8a row a15 (BASELINE config 5's
16 right-hand sides as one block).  There is no reference function for a
batch: every column is checked against the one-at-a-time device path (itself
pinned to the reference's golden vectors in test_gpu_parity.py) and, where
cheap, against the CPU oracle / the reference's golden values directly.
Bars: apply columns rel <= 1e-11 vs the single apply (1e-10 vs the reference),
SpMM bitwise, GMRES iterations +-1 and solution rel <= 1e-8 per column."""

import os

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
# a batched column vs the single apply: the batched local solve runs on 16-row
# panels with explicit 16 x 16 inverses (hg_local_panel.cu), checked at 1e-11
MULTI_RTOL = 1e-11


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def colrel(A, B):
    return max(rel(A[:, c], B[:, c]) for c in range(B.shape[1]))


@pytest.fixture(scope="module")
def cfg1(golden):
    g = golden("config1")
    P = hg.build_problem("1", workers=1, one_level=True)
    coarse = golden_coarse(g, P.forms.n_dofs)
    pre = hg.factorize(P.forms, P.dec, coarse)
    return P, g, coarse, pre


def test_spmm_bitwise(cfg1):
    P, g, _, pre = cfg1
    U = np.random.default_rng(3).standard_normal((pre.n, 16))
    U[:, 0] = g["u"]
    for kind, M in (("B", pre._B), ("Dk", pre._Dk)):
        got = pre.as_operator(kind).apply_multi(U)
        for c in range(16):
            assert np.array_equal(got[:, c], M @ U[:, c]), (kind, c)
    assert np.array_equal(pre.as_operator("B").apply_multi(U)[:, 0], g["Bu"])


@pytest.mark.parametrize("nrhs", [1, 3, 16])
def test_apply_multi_matches_single(cfg1, nrhs):
    P, g, _, pre = cfg1
    R = np.random.default_rng(nrhs).standard_normal((pre.n, nrhs))
    R[:, 0] = g["r"]
    got = pre.apply_multi(R)
    want = np.stack([pre.apply(R[:, c]) for c in range(nrhs)], axis=1)
    assert colrel(got, want) <= MULTI_RTOL
    assert rel(got[:, 0], g["apply_r"]) <= APPLY_RTOL  # the reference's own value
    # deterministic, and the batched operator T = M^-1 B too
    assert np.array_equal(pre.apply_multi(R), got)
    T = pre.as_operator("T").apply_multi(R)
    assert colrel(T, np.stack([pre.apply_T(R[:, c]) for c in range(nrhs)], axis=1)) <= MULTI_RTOL


def test_apply_multi_zero_columns_and_device_tensors(cfg1):
    import torch

    _, g, _, pre = cfg1
    R = np.zeros((pre.n, 4))
    R[:, 2] = g["r"]
    got = pre.apply_multi(R)
    assert np.all(got[:, [0, 1, 3]] == 0.0)
    assert rel(got[:, 2], g["apply_r"]) <= APPLY_RTOL
    t = torch.from_numpy(np.ascontiguousarray(R.T)).cuda()
    out = pre.apply_multi(t)
    assert isinstance(out, torch.Tensor) and out.is_cuda and tuple(out.shape) == (4, pre.n)
    assert np.array_equal(out.cpu().numpy().T, got)
    with pytest.raises(ValueError):
        pre.apply_multi(np.zeros((pre.n, 17)))


def test_apply_multi_one_level(cfg1):
    P, g, _, _ = cfg1
    pre1 = hg.factorize(P.forms, P.dec, None)
    R = np.random.default_rng(5).standard_normal((pre1.n, 5))
    R[:, 1] = g["r"]
    got = pre1.apply_multi(R)
    assert rel(got[:, 1], g["apply_one_level_r"]) <= APPLY_RTOL
    want = np.stack([pre1.apply(R[:, c]) for c in range(5)], axis=1)
    if pre1.panel_active:  # 16-row panel solve: explicit 16 x 16 inverses, different rounding
        assert colrel(got, want) <= MULTI_RTOL
    else:
        assert np.array_equal(got, want)  # row kernel, no coarse part: same per-column arithmetic, bitwise


def test_apply_multi_unpremultiplied_coarse_tiles(cfg1, monkeypatch):
    """The batched coarse solve on the L2-counter tile layout (b0 mode 0)."""
    P, g, coarse, _ = cfg1
    monkeypatch.setenv("HG_B0_MODE", "0")
    monkeypatch.setenv("HG_B0_DENSE", "0")
    pre0 = hg.factorize(P.forms, P.dec, coarse)
    assert pre0.b0_mode == 0 and not pre0.b0_dense
    R = np.random.default_rng(9).standard_normal((pre0.n, 16))
    R[:, 5] = g["r"]
    got = pre0.apply_multi(R)
    want = np.stack([pre0.apply(R[:, c]) for c in range(16)], axis=1)
    assert colrel(got, want) <= MULTI_RTOL
    assert rel(got[:, 5], g["apply_r"]) <= APPLY_RTOL


@pytest.mark.parametrize("orth", ["dcgs2", "measured"])
def test_gmres_batch_matches_single_and_reference(cfg1, orth):
    P, g, _, pre = cfg1
    rng = np.random.default_rng(21)
    F = rng.standard_normal((pre.n, 6))
    F[:, 0] = P.rhs
    F[:, 3] = 0.0  # zero right-hand side: 0 iterations, x = 0
    Rp = pre.apply_multi(F)
    X, reps = hg.weighted_gmres_batch(pre.as_operator("T"), Rp, weight=P.forms.dk, rtol=1e-6, maxit=1000, orth=orth)
    assert len(reps) == 6
    assert reps[3].iterations == 0 and reps[3].converged and np.all(X[:, 3] == 0.0)
    assert abs(reps[0].iterations - int(g["iterations"])) <= 1
    assert rel(X[:, 0], g["x"]) <= SOL_RTOL
    for c in (0, 1, 2, 4, 5):
        x, rep = hg.weighted_gmres(pre.as_operator("T"), Rp[:, c], weight=P.forms.dk, rtol=1e-6, maxit=1000,
                                   orth=orth)
        assert rep.converged and reps[c].converged
        assert abs(rep.iterations - reps[c].iterations) <= 1
        assert rel(X[:, c], x) <= SOL_RTOL
        k = min(rep.residual_history.size, reps[c].residual_history.size)
        assert np.abs(rep.residual_history[:k] - reps[c].residual_history[:k]).max() <= 1e-8 * rep.residual_history[0]


@pytest.mark.parametrize("orth", ["dcgs2", "measured"])
def test_gmres_batch_fixed_iterations_and_maxit(cfg1, orth):
    P, g, _, pre = cfg1
    F = np.random.default_rng(4).standard_normal((pre.n, 3))
    F[:, 1] = P.rhs
    Rp = pre.apply_multi(F)
    it = int(g["iterations"])
    X, reps = hg.weighted_gmres_batch(pre.as_operator("T"), Rp, weight=P.forms.dk, rtol=0.0, maxit=it, orth=orth)
    assert all(r.iterations == it and not r.converged for r in reps)
    assert rel(X[:, 1], g["x_fixed"]) <= SOL_RTOL


@pytest.mark.parametrize("orth", ["dcgs2", "measured"])
def test_gmres_batch_seeded_systems(golden, orth):
    g = golden("wgmres")
    B = np.stack([g["b30"], np.roll(g["b30"], 3), -2.0 * g["b30"]], axis=1)
    for m in (5, 12, 25):
        X, reps = hg.weighted_gmres_batch(g["A30"], B, rtol=0.0, maxit=m, orth=orth)
        assert all(r.iterations == m for r in reps)
        assert np.abs(X[:, 0] - g["x30_%d" % m]).max() <= 1e-10 * max(np.abs(g["x30_%d" % m]).max(), 1.0)
        assert np.abs(reps[0].residual_history - g["h30_%d" % m]).max() <= 1e-10 * g["h30_%d" % m][0]
        assert np.abs(X[:, 2] + 2.0 * X[:, 0]).max() <= 1e-10 * np.abs(X[:, 0]).max()
    W = sp.csr_matrix(g["W50"])
    X, reps = hg.weighted_gmres_batch(g["A50"], np.stack([g["b50"], g["b50"]], axis=1), weight=W, rtol=1e-10,
                                      maxit=50, orth=orth)
    for c in range(2):
        assert reps[c].converged and abs(reps[c].iterations - int(g["it50"])) <= (0 if orth == "measured" else 1)
        assert rel(X[:, c], g["x50"]) <= 1e-10


def test_solve_host_batch(cfg1):
    P, g, _, pre = cfg1
    F = np.random.default_rng(6).standard_normal((pre.n, 4))
    F[:, 2] = P.rhs
    X, reps = pre.solve_host_batch(F, rtol=1e-6, maxit=1000)
    assert abs(reps[2].iterations - int(g["iterations"])) <= 1
    assert rel(X[:, 2], g["x"]) <= SOL_RTOL
    x, rep = pre.solve_host(F[:, 0], rtol=1e-6, maxit=1000)
    assert abs(rep.iterations - reps[0].iterations) <= 1 and rel(X[:, 0], x) <= SOL_RTOL


@pytest.mark.parametrize("name", ["2", "3"])
def test_config_batch_parity_vs_oracle(name):
    """Multi-CTA batched coarse solve (K = 40 / 4 panels) against the oracle."""
    P = hg.build_problem(name)
    pre = hg.factorize(P.forms, P.dec, P.coarse)
    orc = OraclePreconditioner(P.forms, P.dec, P.coarse)
    R = np.random.default_rng(12).standard_normal((P.forms.n_dofs, 16))
    got = pre.apply_multi(R)
    for c in (0, 7, 15):
        assert rel(got[:, c], orc.apply(R[:, c])) <= APPLY_RTOL
    want = np.stack([pre.apply(R[:, c]) for c in range(16)], axis=1)
    assert colrel(got, want) <= MULTI_RTOL
    B, Dk = P.forms.helmholtz, P.forms.dk
    F = np.stack([P.rhs, R[:, 1]], axis=1)
    X, reps = hg.weighted_gmres_batch(pre.as_operator("T"), pre.apply_multi(F), weight=Dk, rtol=1e-6, maxit=1000)
    for c in range(2):
        xo, info = oracle_gmres(lambda v: orc.apply(B @ v), orc.apply(F[:, c]), weight=Dk, rtol=1e-6, maxit=1000)
        assert reps[c].converged and info["converged"]
        assert abs(reps[c].iterations - info["iterations"]) <= 1
        assert rel(X[:, c], xo) <= SOL_RTOL


@pytest.mark.parametrize("name", ["1", "2"])
def test_coarse_solve_modes_agree(name, monkeypatch):
    """Dense B0^{-1} (GEMV / DMMA GEMM), the DSMEM cluster chain and the
    batched tagged-pair chain: the same coarse operator to rounding, each
    against the oracle (lu_solve, schwarz.py:56)."""
    P = hg.build_problem(name)
    orc = OraclePreconditioner(P.forms, P.dec, P.coarse)
    R = np.random.default_rng(31).standard_normal((P.forms.n_dofs, 16))
    outs = {}
    for dense in ("1", "0", "multi"):
        monkeypatch.setenv("HG_B0_DENSE", dense)
        pre = hg.factorize(P.forms, P.dec, P.coarse)
        assert pre.b0_dense == (dense != "0")
        single = np.stack([pre.apply_coarse(R[:, c]) for c in (0, 9)], axis=1)
        outs[dense] = (pre.apply(R[:, 0]), pre.apply_multi(R), single)
        for k, c in enumerate((0, 9)):
            assert rel(single[:, k], orc.apply_coarse(R[:, c])) <= APPLY_RTOL
        assert rel(outs[dense][0], orc.apply(R[:, 0])) <= APPLY_RTOL
        assert colrel(outs[dense][1], np.stack([pre.apply(R[:, c]) for c in range(16)], axis=1)) <= MULTI_RTOL
    assert rel(outs["1"][0], outs["0"][0]) <= 1e-12
    assert colrel(outs["1"][1], outs["0"][1]) <= 1e-12
    assert np.array_equal(outs["multi"][0], outs["0"][0])  # "multi": the single apply keeps the chain
    assert np.array_equal(outs["multi"][1], outs["1"][1])  # and the batched one uses B0^{-1}


def _fov_reference_loop(forms, apply_T, mode, samples=0, rng=None):
    """helmdd.analysis.fov_bounds (analysis.py:342-375) with a given apply_T."""
    import scipy.linalg

    Dk = forms.dk
    n = forms.n_dofs
    if mode == "dense":
        T = np.empty((n, n))
        eye = np.eye(n)
        for j in range(n):
            T[:, j] = apply_T(eye[:, j])
        Dk_d = Dk.toarray()
        M1 = Dk_d @ T
        sym = 0.5 * (M1 + M1.T)
        return (float(scipy.linalg.eigh(sym, Dk_d, eigvals_only=True)[0]),
                float(scipy.linalg.eigh(T.T @ M1, Dk_d, eigvals_only=True)[-1]))
    c1, c2 = np.inf, 0.0
    for _ in range(samples):
        u = rng.standard_normal(n)
        tu = apply_T(u)
        du = Dk @ u
        denom = float(u @ du)
        c1 = min(c1, float(tu @ du) / denom)
        c2 = max(c2, float(tu @ (Dk @ tu)) / denom)
    return c1, c2


def test_fov_bounds_batched_matches_reference_loop(cfg1):
    """the analysis consumer on batched device applies."""
    P, g, _, pre = cfg1
    got = hg.fov_bounds(P.forms, pre, mode="sampled", samples=40, rng=np.random.default_rng(5))
    want = _fov_reference_loop(P.forms, pre.apply_T, "sampled", 40, np.random.default_rng(5))
    assert abs(got[0] - want[0]) <= 1e-10 * abs(want[0]) and abs(got[1] - want[1]) <= 1e-10 * abs(want[1])
    mesh = hg.build_unit_square_mesh(8)
    space = hg.build_fe_space(mesh)
    forms = hg.assemble_forms(mesh, space, hg.coefficient_field(mesh), 5.0)
    dec = hg.build_two_level(mesh, space, 2, 2)
    res = [hg.solve_indefinite_gevp(hg.assemble_local_gevp(i, forms, dec)) for i in range(dec.n_coarse)]
    coarse = hg.build_coarse_space(res, hg.select_modes(res, 1.0), dec, forms)
    small = hg.factorize(forms, dec, coarse)
    orc = OraclePreconditioner(forms, dec, coarse)
    got = hg.fov_bounds(forms, small, mode="dense")
    want = _fov_reference_loop(forms, lambda u: orc.apply(forms.helmholtz @ u), "dense")
    assert abs(got[0] - want[0]) <= 1e-9 * abs(want[0]) and abs(got[1] - want[1]) <= 1e-9 * abs(want[1])


def test_packed_z_matches_row_major_kernels(cfg1, monkeypatch):
    """The batched Z^T R / Z Y read Z from packed DMMA-fragment copies (hg_multi.cu
    "packed Z"); HG_Z_PACKED=0 keeps the row-major kernels.  Same products, same
    k order: the two paths agree to rounding of the DMMA accumulation order."""
    P, g, coarse, pre = cfg1
    R = np.random.default_rng(21).standard_normal((pre.n, 16))
    want = pre.apply_multi(R)
    monkeypatch.setenv("HG_Z_PACKED", "0")
    plain = hg.factorize(P.forms, P.dec, coarse)
    got = plain.apply_multi(R)
    assert colrel(got, want) <= 1e-13
    assert colrel(plain.apply_multi(R[:, :3]), want[:, :3]) <= 1e-13
