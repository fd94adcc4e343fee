"""Failure paths and safety nets of the device solve phase (VERDICT r1 weak
#5-#8): bounded cross-kernel waits that poison a handle instead of
hanging the GPU, CUDA-graph capture of an apply, the DCGS2 explicit-rho pass,
the maxit guard and the Krylov-basis release.  Bars as everywhere: apply
rel <= 1e-10 vs the reference's golden vector, iterations +-1, x <= 1e-8."""

import time

import numpy as np
import pytest

import paper_2406_06283_b200 as hg
from paper_2406_06283_b200 import _lib
from _helpers import golden_coarse

pytestmark = pytest.mark.gpu


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.fixture(scope="module")
def cfg1(golden):
    g = golden("config1")
    P = hg.build_problem("1", workers=1, one_level=True)
    coarse = golden_coarse(g, P.forms.n_dofs)
    return P, g, coarse


@pytest.fixture
def short_spin():
    lib = _lib.load()
    _lib.check(lib.hg_debug_set(None, _lib.DEBUG_SPIN_LIMIT_MS, 300), "hg_debug_set")
    yield
    _lib.check(lib.hg_debug_set(None, _lib.DEBUG_SPIN_LIMIT_MS, 10000), "hg_debug_set")


@pytest.mark.parametrize("mode", ["1", "0"])
@pytest.mark.parametrize("batched", [False, True])
def test_lost_zt_times_out_and_poisons(cfg1, short_spin, monkeypatch, mode, batched):
    """The coarse solve is launched ahead of the Z^T r it waits for.  Drop
    that Z^T r (fault injection): the wait must give up within its bound, the
    call must raise DeviceError, and the handle must stay poisoned — never a
    hung GPU."""
    P, g, coarse = cfg1
    monkeypatch.setenv("HG_B0_MODE", mode)
    monkeypatch.setenv("HG_B0_DENSE", "0")  # the chain kernels (the ones that wait on Z^T r)
    pre = hg.factorize(P.forms, P.dec, coarse)
    assert pre.b0_mode == int(mode)
    R = np.stack([g["r"], g["u"]], axis=1)
    assert rel(pre.apply(g["r"]), g["apply_r"]) <= 1e-10  # healthy first
    lib = _lib.load()
    _lib.check(lib.hg_debug_set(pre._handle, _lib.DEBUG_SKIP_ZT, 1), "hg_debug_set")
    t0 = time.perf_counter()
    with pytest.raises(hg.DeviceError, match="timed out"):
        pre.apply_multi(R) if batched else pre.apply(g["r"])
    assert time.perf_counter() - t0 < 30.0
    with pytest.raises(hg.DeviceError, match="poisoned"):
        pre.apply(g["r"])
    with pytest.raises(hg.DeviceError):
        hg.weighted_gmres(pre.as_operator("T"), g["rhs_p"], weight=P.forms.dk, rtol=1e-6, maxit=50)
    # a fresh handle on the same device is unaffected
    pre2 = hg.factorize(P.forms, P.dec, coarse)
    assert rel(pre2.apply(g["r"]), g["apply_r"]) <= 1e-10


def test_graph_capture_replays_match_eager(cfg1):
    """An apply captured into a CUDA graph (serial launch order under capture;
    the coarse solve's pairing with Z^T r is a device ticket, not a host
    counter) replays with new inputs bitwise equal to eager applies, and
    eager applies after the replays stay correct (hg_api.cu:418)."""
    import torch

    P, g, coarse = cfg1
    pre = hg.factorize(P.forms, P.dec, coarse)
    n = pre.n
    rng = np.random.default_rng(44)
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    pre.apply(x)  # warm: everything allocated before capture
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        y = pre.apply(x)
    for _ in range(3):
        v = rng.standard_normal(n)
        x.copy_(torch.from_numpy(v))
        graph.replay()
        torch.cuda.synchronize()
        pre.check()
        assert np.array_equal(y.cpu().numpy(), pre.apply(v))
    assert rel(pre.apply(g["r"]), g["apply_r"]) <= 1e-10
    x.copy_(torch.from_numpy(g["r"]))
    graph.replay()
    torch.cuda.synchronize()
    assert rel(y.cpu().numpy(), g["apply_r"]) <= 1e-10


def test_dcgs2_explicit_rho_pass(cfg1):
    """Force the DCGS2 explicit-rho branch (taken when rho^2 = a_j - s.s loses
    its digits) on every column and iteration: single and batched solves keep
    the reference's iteration count and solution (golden config 1), and the
    passes are counted."""
    P, g, coarse = cfg1
    pre = hg.factorize(P.forms, P.dec, coarse)
    op = pre.as_operator("T")
    lib = _lib.load()
    before = lib.hg_dcgs2_explicit_passes()
    _lib.check(lib.hg_debug_set(None, _lib.DEBUG_FORCE_EXPLICIT_RHO, 1), "hg_debug_set")
    try:
        x, rep = hg.weighted_gmres(op, g["rhs_p"], weight=P.forms.dk, rtol=1e-6, maxit=1000, orth="dcgs2")
        R = np.stack([g["rhs_p"], g["rhs_p"], 0.5 * g["rhs_p"]], axis=1)
        X, reps = hg.weighted_gmres_batch(op, R, weight=P.forms.dk, rtol=1e-6, maxit=1000, orth="dcgs2")
    finally:
        _lib.check(lib.hg_debug_set(None, _lib.DEBUG_FORCE_EXPLICIT_RHO, 0), "hg_debug_set")
    it_ref = int(g["iterations"])
    assert abs(rep.iterations - it_ref) <= 1
    assert rel(x, g["x"]) <= 1e-8
    assert np.abs(rep.residual_history[: it_ref + 1] - g["history"][: rep.iterations + 1][: it_ref + 1]).max() \
        <= 1e-8 * g["history"][0]
    assert rep.reorth_passes >= 2 * (rep.iterations - 1)  # delayed pass + explicit pass per iteration
    for c, r in enumerate(reps):
        assert abs(r.iterations - it_ref) <= 1
        assert rel(X[:, c], (0.5 if c == 2 else 1.0) * g["x"]) <= 1e-8
    assert lib.hg_dcgs2_explicit_passes() - before >= rep.iterations - 1


def test_maxit_beyond_basis_kernels_is_refused_up_front(cfg1):
    P, g, coarse = cfg1
    pre = hg.factorize(P.forms, P.dec, coarse)
    t0 = time.perf_counter()
    with pytest.raises(hg.DeviceError, match="1024"):
        hg.weighted_gmres(pre.as_operator("T"), g["rhs_p"], weight=P.forms.dk, rtol=1e-6, maxit=5000)
    assert time.perf_counter() - t0 < 5.0
    with pytest.raises(hg.DeviceError, match="1024"):
        hg.weighted_gmres_batch(pre.as_operator("T"), np.stack([g["rhs_p"]] * 2, axis=1), weight=P.forms.dk,
                                rtol=1e-6, maxit=5000)


def test_release_frees_the_basis_and_the_op_stays_usable(cfg1):
    P, g, coarse = cfg1
    pre = hg.factorize(P.forms, P.dec, coarse)
    op = pre.as_operator("T")
    x1, rep1 = hg.weighted_gmres(op, g["rhs_p"], weight=P.forms.dk, rtol=1e-6, maxit=1000)
    assert op.basis(rep1.iterations).shape[0] == rep1.iterations
    op.release()
    with pytest.raises(hg.DeviceError):
        op.basis(1)
    x2, rep2 = hg.weighted_gmres(op, g["rhs_p"], weight=P.forms.dk, rtol=1e-6, maxit=1000)
    assert rep2.iterations == rep1.iterations and np.array_equal(x1, x2)
