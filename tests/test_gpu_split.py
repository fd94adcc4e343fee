"""Split local blocks (include/helmgpu.h "Split local blocks"; factor.split_block):
a subdomain's band solve cut into P chunks + separators + spikes is the SAME
local operator ls.lu.solve (schwarz.py:58-60).  Checked against the unsplit
device preconditioner (itself pinned to the reference's golden vectors and
the oracle in test_gpu_parity.py), against the CPU oracle directly, batched
vs single, through a GMRES solve, and through the setup cache."""

import numpy as np
import pytest

import paper_2406_06283_b200 as hg
from paper_2406_06283_b200 import cache
from oracle.schwarz_oracle import OraclePreconditioner
from oracle.wgmres_oracle import weighted_gmres as oracle_gmres

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.fixture(scope="module")
def cfg3():
    P = hg.build_problem("3", workers=1)
    plain = hg.factorize(P.forms, P.dec, P.coarse)
    return P, plain


@pytest.mark.parametrize("nchunk", [2, 4])
def test_split_apply_matches_unsplit_and_oracle(cfg3, nchunk, monkeypatch):
    P, plain = cfg3
    monkeypatch.setenv("HG_LOCAL_SPLIT", str(nchunk))
    pre = hg.factorize(P.forms, P.dec, P.coarse)
    assert pre.n_split == len(pre.local_solvers) and pre.split_bytes > 0
    rng = np.random.default_rng(11)
    r = rng.standard_normal(pre.n)
    want = plain.apply(r)
    got = pre.apply(r)
    assert rel(got, want) <= 1e-11
    assert rel(pre.apply_T(r), plain.apply_T(r)) <= 1e-11
    oracle = OraclePreconditioner(P.forms, P.dec, P.coarse)
    assert rel(got, oracle.apply(r)) <= 1e-10
    # batched: every column vs the single split apply and vs the unsplit batch
    R = rng.standard_normal((pre.n, 16))
    R[:, 3] = r
    M = pre.apply_multi(R)
    assert rel(M[:, 3], got) <= 1e-11
    assert max(rel(M[:, c], plain.apply(R[:, c])) for c in (0, 7, 15)) <= 1e-11
    assert rel(pre.apply_multi(R[:, :5]), M[:, :5]) <= 1e-13
    # invariants: zero -> zero, determinism, linearity
    assert not pre.apply(np.zeros(pre.n)).any()
    assert np.array_equal(pre.apply(r), got)
    s = rng.standard_normal(pre.n)
    assert rel(pre.apply(2.0 * r - 3.0 * s), 2.0 * got - 3.0 * pre.apply(s)) <= 1e-12
    # LocalSolver.lu.solve of a split block (schwarz.py:26-34) against the unsplit block's device solve
    for s in (0, len(pre.local_solvers) - 1):
        rl = rng.standard_normal(pre.local_solvers[s].idof.size)
        assert rel(pre.local_solvers[s].lu.solve(rl), plain.local_solvers[s].lu.solve(rl)) <= 1e-11


def test_split_gmres_matches_oracle(cfg3, monkeypatch):
    P, plain = cfg3
    monkeypatch.setenv("HG_LOCAL_SPLIT", "4")
    pre = hg.factorize(P.forms, P.dec, P.coarse)
    f = np.asarray(P.rhs, dtype=float)
    rhs_p = pre.apply(f)
    op = pre.as_operator("T")
    x, rep = hg.weighted_gmres(op, rhs_p, weight=P.forms.dk, rtol=P.config.rtol, maxit=P.config.maxit)
    oracle = OraclePreconditioner(P.forms, P.dec, P.coarse)
    B = P.forms.helmholtz
    xo, info = oracle_gmres(lambda v: oracle.apply(B @ v), oracle.apply(f), weight=P.forms.dk, rtol=P.config.rtol,
                            maxit=P.config.maxit)
    its = info["iterations"]
    assert rep.converged and info["converged"]
    assert abs(rep.iterations - its) <= 1
    assert rel(x, xo) <= 1e-8
    # the 16-column block through the split path
    F = np.repeat(f[:, None], 4, axis=1) * np.array([1.0, -2.0, 0.5, 3.0])
    X, reps = hg.weighted_gmres_batch(op, pre.apply_multi(F), weight=P.forms.dk, rtol=P.config.rtol,
                                      maxit=P.config.maxit)
    for c, sc in enumerate([1.0, -2.0, 0.5, 3.0]):
        assert abs(reps[c].iterations - its) <= 1
        assert rel(X[:, c], sc * xo) <= 1e-8


def test_split_cache_round_trip(cfg3, monkeypatch, tmp_path):
    P, _ = cfg3
    monkeypatch.setenv("HG_LOCAL_SPLIT", "2")
    pre = hg.factorize(P.forms, P.dec, P.coarse, keep_image=True)
    path = str(tmp_path / "img")
    cache.save_preconditioner(pre, path)
    again = cache.factorize_from_cache(path)
    r = np.random.default_rng(5).standard_normal(pre.n)
    assert np.array_equal(pre.apply(r), again.apply(r))
    R = np.random.default_rng(6).standard_normal((pre.n, 16))
    assert np.array_equal(pre.apply_multi(R), again.apply_multi(R))


def test_inconsistent_split_descriptors_are_refused(monkeypatch):
    """hg_precond_create validates the split-block description (helmgpu.h): positions out of the
    solution scratch, a split that does not name a separator pseudo block, a spike past its data."""
    from paper_2406_06283_b200 import schwarz
    from paper_2406_06283_b200.schwarz import TwoLevelPreconditioner

    P = hg.build_problem("1", workers=1, one_level=True)
    monkeypatch.setenv("HG_LOCAL_SPLIT", "2")
    A, M = schwarz.host_image(P.forms, P.dec, None)
    assert M["n_split"] > 0
    good = TwoLevelPreconditioner.from_image(dict(A), dict(M))
    r = np.random.default_rng(1).standard_normal(good.n)
    assert np.isfinite(good.apply(r)).all()

    def broken(name, mutate):
        arrays = {k: np.array(v, copy=True) for k, v in A.items()}
        mutate(arrays)
        with pytest.raises(hg.DeviceError, match=name):
            TwoLevelPreconditioner.from_image(arrays, dict(M))

    broken("position out of range", lambda a: a["split_f_pos"].__setitem__(0, int(a["local_idx_off"][-1]) + 5))
    broken("pseudo block", lambda a: a["split_blk"].__setitem__(0, 0))
    broken("spike", lambda a: a["spike_off"].__setitem__(len(a["spike_off"]) - 1, int(M["spike_len"])))
