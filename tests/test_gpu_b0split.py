"""Bisected single-RHS coarse solve (include/helmgpu.h "Bisected coarse solve"):
two half chains + a dense separator system are the SAME y = B0^{-1} c as
lu_solve(b0_piv, c) (schwarz.py:56).  Checked against the full-chain device
solve, the oracle, through the debug switch (device tickets re-paired), under
CUDA-graph replay and with a dropped Z^T r (bounded wait -> poisoned handle)."""

import numpy as np
import pytest

import paper_2406_06283_b200 as hg
from paper_2406_06283_b200 import _lib

from oracle.schwarz_oracle import OraclePreconditioner

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.fixture(scope="module")
def setup3():
    import os

    P = hg.build_problem("3", workers=1)
    old = os.environ.get("HG_B0_SPLIT")
    os.environ["HG_B0_SPLIT"] = "0"
    plain = hg.factorize(P.forms, P.dec, P.coarse)
    os.environ["HG_B0_SPLIT"] = "1"
    split = hg.factorize(P.forms, P.dec, P.coarse)
    if old is None:
        del os.environ["HG_B0_SPLIT"]
    else:
        os.environ["HG_B0_SPLIT"] = old
    return P, plain, split


def test_bisected_coarse_solve_matches_chain_and_oracle(setup3):
    P, plain, split = setup3
    assert split.b0_split and not plain.b0_split
    assert split._meta["b0_split_dev"] <= 1e-11
    rng = np.random.default_rng(4)
    r = rng.standard_normal(split.n)
    assert rel(split.apply_coarse(r), plain.apply_coarse(r)) <= 1e-11
    assert rel(split.apply(r), plain.apply(r)) <= 1e-11
    orc = OraclePreconditioner(P.forms, P.dec, P.coarse)
    assert rel(split.apply(r), orc.apply(r)) <= 1e-10
    assert np.array_equal(split.apply(r), split.apply(r))
    assert not split.apply(np.zeros(split.n)).any()


def test_debug_switch_repairs_tickets(setup3):
    P, plain, split = setup3
    lib = _lib.load()
    r = np.random.default_rng(5).standard_normal(split.n)
    on = split.apply(r)
    for _ in range(3):
        split.apply(r)
    _lib.check(lib.hg_debug_set(split._handle, _lib.DEBUG_B0_SPLIT, 0), "debug")
    off = split.apply(r)
    assert np.array_equal(off, split.apply(r))
    assert rel(off, plain.apply(r)) <= 1e-13  # the full chain of the same handle
    _lib.check(lib.hg_debug_set(split._handle, _lib.DEBUG_B0_SPLIT, 1), "debug")
    assert np.array_equal(split.apply(r), on)


def test_gmres_through_bisected_coarse_solve(setup3):
    P, plain, split = setup3
    f = np.asarray(P.rhs, dtype=float)
    x1, r1 = hg.weighted_gmres(split.as_operator("T"), split.apply(f), weight=P.forms.dk, rtol=1e-6, maxit=1000)
    x0, r0 = hg.weighted_gmres(plain.as_operator("T"), plain.apply(f), weight=P.forms.dk, rtol=1e-6, maxit=1000)
    assert r1.converged and r1.iterations == r0.iterations
    assert rel(x1, x0) <= 1e-9


def test_graph_replay_and_dropped_zt(setup3):
    import torch

    P, plain, _ = setup3
    import os

    old = os.environ.get("HG_B0_SPLIT")
    os.environ["HG_B0_SPLIT"] = "1"
    try:
        pre = hg.factorize(P.forms, P.dec, P.coarse)
    finally:
        if old is None:
            del os.environ["HG_B0_SPLIT"]
        else:
            os.environ["HG_B0_SPLIT"] = old
    r = torch.from_numpy(np.random.default_rng(6).standard_normal(pre.n)).cuda()
    eager = pre.apply(r).clone()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        out = pre.apply(r)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            out = pre.apply(r)
    for _ in range(3):
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, eager)
        assert torch.equal(pre.apply(r), eager)
    lib = _lib.load()
    _lib.check(lib.hg_debug_set(None, _lib.DEBUG_SPIN_LIMIT_MS, 200), "debug")
    try:
        _lib.check(lib.hg_debug_set(pre._handle, _lib.DEBUG_SKIP_ZT, 1), "debug")
        with pytest.raises(hg.DeviceError):
            pre.apply(r.cpu().numpy())
        with pytest.raises(hg.DeviceError):
            pre.check()
    finally:
        _lib.check(lib.hg_debug_set(None, _lib.DEBUG_SPIN_LIMIT_MS, 10000), "debug")
