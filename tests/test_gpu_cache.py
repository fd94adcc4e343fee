"""On-disk setup cache, device side: a handle created
from the cache (factorize_from_cache -> hg_precond_create on the stored
arrays, no host setup) applies and solves bitwise like the freshly
factorised one, and the config-level entry point hits on its second call."""

import numpy as np
import pytest

import paper_2406_06283_b200 as hg
from paper_2406_06283_b200 import cache
from _helpers import golden_coarse

pytestmark = pytest.mark.gpu


def test_cached_handle_is_bitwise_the_fresh_one(golden, tmp_path):
    g = golden("config1")
    P = hg.build_problem("1", workers=1, one_level=True)
    coarse = golden_coarse(g, P.forms.n_dofs)
    fresh = hg.factorize(P.forms, P.dec, coarse, keep_image=True)
    path = cache.save_preconditioner(fresh, str(tmp_path / "cfg1"), extra_arrays={"rhs": P.rhs})
    pre = cache.factorize_from_cache(path)
    assert pre.n == fresh.n and pre.m == fresh.m and pre.has_coarse
    assert np.array_equal(pre.apply(g["r"]), fresh.apply(g["r"]))
    assert np.array_equal(pre.apply_T(g["u"]), fresh.apply_T(g["u"]))
    assert np.array_equal(pre.apply_coarse(g["r"]), fresh.apply_coarse(g["r"]))
    R = np.stack([g["r"], g["u"], g["rhs_p"]], axis=1)
    assert np.array_equal(pre.apply_multi(R), fresh.apply_multi(R))
    s = 3
    r_loc = g["r"][pre.local_solvers[s].idof]
    assert np.array_equal(pre.local_solvers[s].lu.solve(r_loc), fresh.local_solvers[s].lu.solve(r_loc))
    x1, rep1 = hg.weighted_gmres(pre.as_operator("T"), g["rhs_p"], weight=pre.forms.dk, rtol=1e-6, maxit=1000)
    x0, rep0 = hg.weighted_gmres(fresh.as_operator("T"), g["rhs_p"], weight=P.forms.dk, rtol=1e-6, maxit=1000)
    assert rep1.iterations == rep0.iterations == int(g["iterations"])
    assert np.array_equal(x1, x0)
    assert np.array_equal(rep1.residual_history, rep0.residual_history)


def test_solver_for_config_misses_then_hits(tmp_path):
    pre0, P0, info0 = cache.solver_for_config("1", cache_dir=str(tmp_path), workers=1)
    pre1, P1, info1 = cache.solver_for_config("1", cache_dir=str(tmp_path), workers=1)
    assert not info0["hit"] and info1["hit"] and info1["path"] == info0["path"]
    assert np.array_equal(P1.rhs, P0.rhs)
    r = np.random.default_rng(3).standard_normal(pre0.n)
    assert np.array_equal(pre1.apply(r), pre0.apply(r))
    x0, rep0 = hg.weighted_gmres(pre0.as_operator("T"), pre0.apply(P0.rhs), weight=P0.forms.dk, rtol=1e-6, maxit=500)
    x1, rep1 = hg.weighted_gmres(pre1.as_operator("T"), pre1.apply(P1.rhs), weight=P1.forms.dk, rtol=1e-6, maxit=500)
    assert rep0.iterations == rep1.iterations and np.array_equal(x0, x1)
