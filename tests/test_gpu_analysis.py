"""Analysis consumers on the device applies:
check_tf_stability, check_t0_stability and check_prop26_identity against the
reference's own outcomes on the same setups (tests/golden/analysis.npz,
written by oracle/gen_golden.py from helmdd.analysis; the setups are
pkg/tests/test_analysis.py:300-323 and the test_schwarz pipeline).  The
random draws follow the reference's order, so the trial counts, violations
and witnesses agree and the worst margins agree to rounding."""

import types

import numpy as np
import pytest

import paper_2406_06283_b200 as hg
from oracle.gen_golden import ANALYSIS_T0_THEORY

pytestmark = pytest.mark.gpu


def _forms(k):
    mesh = hg.build_unit_square_mesh(8)
    space = hg.build_fe_space(mesh)
    return mesh, space, hg.assemble_forms(mesh, space, hg.coefficient_field(mesh), k)


def test_tf_stability_matches_reference(golden):
    g = golden("analysis")
    mesh, space, forms = _forms(0.5)
    dec = hg.build_two_level(mesh, space, 2, 2)
    assert dec.Hf * 0.5 <= np.sqrt(2.0) / 2.0
    chk = hg.check_tf_stability(forms, dec, hg.factorize(forms, dec, None), trials=10, rng=np.random.default_rng(5))
    assert chk.trials == int(g["tf_trials"]) == 10 * 16
    assert chk.violations == int(g["tf_violations"]) == 0
    assert chk.witness == int(g["tf_witness"])
    assert abs(chk.worst_margin - float(g["tf_worst"])) <= 1e-9 * abs(float(g["tf_worst"]))


def test_prop26_identity_matches_reference(golden):
    g = golden("analysis")
    mesh, space, forms = _forms(5.0)
    dec = hg.build_two_level(mesh, space, 2, 2)
    chk = hg.check_prop26_identity(forms, hg.factorize(forms, dec, None), trials=20, rng=np.random.default_rng(6))
    assert chk.trials == int(g["prop26_trials"]) and chk.violations == int(g["prop26_violations"]) == 0
    # margins are 1e-12 |lhs| minus rounding noise: same scale as the reference's
    assert 0.5 * float(g["prop26_worst"]) <= chk.worst_margin <= 2.0 * float(g["prop26_worst"])


def test_t0_stability_matches_reference(golden):
    g = golden("analysis")
    mesh = hg.build_unit_square_mesh(16)
    space = hg.build_fe_space(mesh)
    forms = hg.assemble_forms(mesh, space, hg.coefficient_field(mesh), 10.0)
    dec = hg.build_two_level(mesh, space, 2, 2, 1, 1)
    res = [hg.solve_indefinite_gevp(hg.assemble_local_gevp(i, forms, dec)) for i in range(dec.n_coarse)]
    coarse = hg.build_coarse_space(res, hg.select_modes(res, 1.0), dec, forms)
    pre = hg.factorize(forms, dec, coarse)
    theory = types.SimpleNamespace(**ANALYSIS_T0_THEORY)
    chk = hg.check_t0_stability(forms, coarse, pre, theory, trials=20, rng=np.random.default_rng(7))
    assert chk.extra["hypothesis_value"] <= 0.5
    assert chk.trials == int(g["t0_trials"]) == 20 and chk.violations == int(g["t0_violations"])
    assert chk.witness == int(g["t0_witness"])
    assert abs(chk.worst_margin - float(g["t0_worst"])) <= 1e-9 * abs(float(g["t0_worst"]))
