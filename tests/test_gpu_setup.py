"""Setup on the device: the coarse operator B0 = Z^T B Z
(eigencoarse.py:286-287), its LU with partial pivoting (schwarz.py:90,
getrf semantics) and the rank certificate, built by hg_coarse_setup, against
the host build (numpy / LAPACK, what the reference runs)."""

import numpy as np
import pytest
import scipy.linalg

import paper_2406_06283_b200 as hg
from paper_2406_06283_b200 import coarse as C

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300))


@pytest.fixture(scope="module")
def cfg2():
    P = hg.build_problem("2")
    sel = P.selection
    host = C.build_coarse_space(P.results, sel, P.dec, P.forms, device=False)
    dev = C.build_coarse_space(P.results, sel, P.dec, P.forms, device=True)
    return P, host, dev


def test_device_b0_matches_host(cfg2):
    P, host, dev = cfg2
    assert dev.m_total == host.m_total == 2560 and dev.removed == host.removed == []
    assert rel(dev.B0, host.B0) <= 1e-13
    assert np.array_equal(dev.B0, dev.B0.T)  # symmetrised exactly


def test_device_getrf_matches_lapack(cfg2):
    P, host, dev = cfg2
    blocks = host.blocks
    pairs = C._interaction_pairs(P.forms, [i for i, _ in blocks])
    B0, (lu, piv), info, (lmax, inv_max) = C.coarse_operator_device(P.forms, blocks, pairs)
    assert info == 0
    lu_h, piv_h = scipy.linalg.lu_factor(host.B0)
    assert np.array_equal(piv, piv_h)  # same row interchanges as LAPACK
    assert rel(lu, lu_h) <= 1e-11
    c = np.random.default_rng(3).standard_normal(B0.shape[0])
    assert rel(scipy.linalg.lu_solve((lu, piv), c), scipy.linalg.lu_solve((lu_h, piv_h), c)) <= 1e-11
    # certificate estimates (power / inverse iteration: from below, trusted with a margin) against the
    # dense eigenvalues
    ev = np.abs(np.linalg.eigvalsh(host.B0))
    assert 0.9 * ev.max() <= lmax <= ev.max() * (1 + 1e-12)
    assert 0.9 / ev.min() <= inv_max <= (1 + 1e-12) / ev.min()


def test_preconditioner_from_device_coarse(cfg2):
    P, host, dev = cfg2
    pre_h = hg.factorize(P.forms, P.dec, host)
    pre_d = hg.factorize(P.forms, P.dec, dev)
    r = np.random.default_rng(5).standard_normal(pre_h.n)
    assert rel(pre_d.apply(r), pre_h.apply(r)) <= 1e-11
