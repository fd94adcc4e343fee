"""The CPU oracle (oracle/) pinned against golden vectors produced by the
reference package itself (oracle/gen_golden.py)."""

import numpy as np
import pytest

import paper_2406_06283_b200 as hg
from _helpers import golden_coarse
from oracle import dense
from oracle.schwarz_oracle import OraclePreconditioner
from oracle.wgmres_oracle import weighted_gmres as oracle_gmres


@pytest.fixture(scope="module")
def cfg1_oracle(golden):
    g = golden("config1")
    P = hg.build_problem("1", workers=1, one_level=True)
    coarse = golden_coarse(g, P.forms.n_dofs)
    return P, g, OraclePreconditioner(P.forms, P.dec, coarse)


def test_oracle_apply_matches_reference(cfg1_oracle):
    P, g, orc = cfg1_oracle
    for got, want in ((orc.apply(g["r"]), g["apply_r"]), (orc.apply_T(g["u"]), g["apply_T_u"]),
                      (orc.apply_coarse(g["r"]), g["apply_coarse_r"])):
        assert np.abs(got - want).max() <= 1e-13 * np.abs(want).max()


def test_oracle_gmres_matches_reference(cfg1_oracle):
    P, g, orc = cfg1_oracle
    B, Dk = P.forms.helmholtz, P.forms.dk
    rhs_p = orc.apply(P.rhs)
    assert np.abs(rhs_p - g["rhs_p"]).max() <= 1e-13 * np.abs(g["rhs_p"]).max()
    x, info = oracle_gmres(lambda v: orc.apply(B @ v), rhs_p, weight=Dk, rtol=1e-6, maxit=1000)
    assert info["iterations"] == int(g["iterations"])
    assert np.abs(x - g["x"]).max() <= 1e-11 * np.abs(g["x"]).max()
    assert np.abs(info["history"] - g["history"]).max() <= 1e-11 * g["history"][0]


def test_oracle_small_pipelines(golden):
    g = golden("small")
    for tag, (n, M, q, k) in {"p8": (8, 2, 2, 5.0), "p16": (16, 2, 2, 10.0)}.items():
        mesh = hg.build_unit_square_mesh(n)
        space = hg.build_fe_space(mesh)
        forms = hg.assemble_forms(mesh, space, hg.coefficient_field(mesh), k)
        dec = hg.build_two_level(mesh, space, M, q)
        res = [hg.solve_indefinite_gevp(hg.assemble_local_gevp(i, forms, dec)) for i in range(dec.n_coarse)]
        sel = hg.select_modes(res, 1.0)
        coarse = hg.build_coarse_space(res, sel, dec, forms)
        assert coarse.m_total == int(g[tag + "_m"])
        orc = OraclePreconditioner(forms, dec, coarse)
        want = g[tag + "_apply"]
        assert np.abs(orc.apply(g[tag + "_r"]) - want).max() <= 1e-11 * np.abs(want).max()
        M2 = dense.dense_two_level(forms, dec, coarse.Z)
        assert np.abs(M2 @ g[tag + "_r"] - want).max() <= 1e-10 * np.abs(want).max()


def test_oracle_gmres_seeded_systems(golden):
    g = golden("wgmres")
    for m in (5, 12, 25):
        x, info = oracle_gmres(g["A30"], g["b30"], rtol=0.0, maxit=m)
        assert np.abs(x - g["x30_%d" % m]).max() <= 1e-12 * max(np.abs(g["x30_%d" % m]).max(), 1.0)
        xt, ht = dense.textbook_gmres(g["A30"], g["b30"], m)
        assert np.abs(x - xt).max() <= 1e-10 * max(np.abs(xt).max(), 1.0)
    x, info = oracle_gmres(g["A50"], g["b50"], weight=g["W50"], rtol=1e-10, maxit=50)
    assert info["iterations"] == int(g["it50"])
    assert np.abs(x - g["x50"]).max() <= 1e-12 * np.abs(g["x50"]).max()
