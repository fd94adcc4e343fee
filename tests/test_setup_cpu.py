"""Setup-phase restatement vs the reference's golden outputs (CPU)."""

import numpy as np
import pytest
import scipy.sparse as sp

import paper_2406_06283_b200 as hg
from paper_2406_06283_b200 import coarse as hc
from paper_2406_06283_b200 import factor


@pytest.fixture(scope="module")
def cfg1():
    return hg.build_problem("1", workers=1)


def test_forms_bitwise(cfg1, golden):
    g = golden("config1")
    B, Dk = cfg1.forms.helmholtz, cfg1.forms.dk
    assert np.array_equal(B.indptr, g["B_indptr"]) and np.array_equal(B.indices, g["B_indices"])
    assert np.array_equal(B.data, g["B_data"])
    assert np.array_equal(Dk.data, g["Dk_data"])
    assert np.array_equal(cfg1.rhs, g["rhs"])


def test_cstab_sparse_matches_dense(cfg1, golden):
    g = golden("config1")
    assert abs(cfg1.cstab - float(g["cstab"])) <= 1e-9 * float(g["cstab"])


def test_mode_selection_and_coarse(cfg1, golden):
    g = golden("config1")
    assert list(cfg1.selection.m_per_subdomain) == list(g["m_per"])
    assert abs(cfg1.selection.tau - float(g["tau"])) <= 1e-10
    low = np.concatenate([r.eigenvalues[:8] for r in cfg1.results])
    assert np.abs(low - g["eig_low"]).max() <= 1e-9
    B0 = cfg1.coarse.B0
    assert np.abs(B0 - g["B0"]).max() <= 1e-10 * np.abs(g["B0"]).max()


def test_lanczos_matches_dense_on_config1(cfg1):
    for i in (0, 5, 10):
        gs = hc.assemble_local_gevp(i, cfg1.forms, cfg1.dec, dense=False)
        rl = hc.solve_gevp_lanczos(gs, 12)
        rd = cfg1.results[i]
        assert np.abs(rl.eigenvalues[:12] - rd.eigenvalues[:12]).max() <= 1e-9


def test_select_modes_cap_semantics():
    res = [hc.LocalGevpResult(0, np.array([-1.0, 0.1, 0.2, 0.3, 5.0]), np.eye(5), 1, 0, 1.0)]
    with pytest.raises(hg.ModeCapError):
        hc.select_modes(res, 1.0, [2])
    sel = hc.select_modes(res, 1.0, [2], truncate=True)
    assert sel.m_per_subdomain == [2] and sel.tau == 0.2
    sel = hc.select_modes(res, 1.0)
    assert sel.m_per_subdomain == [4] and sel.tau == 5.0


def test_decomposition_divisibility_errors():
    mesh = hg.build_unit_square_mesh(10)
    space = hg.build_fe_space(mesh)
    with pytest.raises(hg.ConfigError):
        hg.build_two_level(mesh, space, 3, 1)
    with pytest.raises(hg.ConfigError):
        hg.build_two_level(mesh, space, 2, 1, 0, 1)


def test_pou_partition_of_unity():
    mesh = hg.build_unit_square_mesh(24)
    space = hg.build_fe_space(mesh)
    dec = hg.build_two_level(mesh, space, 3, 2, 2, 1)
    tot = np.zeros(space.n_dofs)
    for sub in dec.coarse:
        tot[sub.ovdof] += sub.pou
    assert np.abs(tot - 1.0).max() <= 1e-14


def test_b0_band_packing_roundtrip(cfg1):
    lu, piv = factor.lu_b0(cfg1.coarse.B0)
    perm, kl, ku, lband, uband = factor.pack_b0(lu, piv)
    m = lu.shape[0]
    L = np.eye(m)
    U = np.zeros((m, m))
    for i in range(m):
        for t in range(kl):
            j = i - kl + t
            if j >= 0:
                L[i, j] = lband[i, t]
        for t in range(ku + 1):
            if i + t < m:
                U[i, i + t] = uband[i, t]
    assert np.array_equal(np.tril(lu, -1) + np.eye(m), L)
    assert np.array_equal(np.triu(lu), U)
    c = np.random.default_rng(0).standard_normal(m)
    import scipy.linalg

    want = scipy.linalg.lu_solve((lu, piv), c)
    got = scipy.linalg.solve_triangular(U, scipy.linalg.solve_triangular(L, c[perm], lower=True, unit_diagonal=True))
    assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()
