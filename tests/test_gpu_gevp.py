"""Local H_k-GenEO eigenproblems on the device (SURVEY §8f item 3,
gevp_device.py): the batched thick-restart Lanczos against the host ARPACK
restatement (coarse.solve_gevp_lanczos, eigencoarse.py:152-217 semantics):
the same lowest eigenvalues, the same selected coarse space (the apply only
depends on span(Z)), hence the same preconditioner."""

import numpy as np
import pytest

import paper_2406_06283_b200 as hg
from paper_2406_06283_b200 import problems

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300))


@pytest.mark.parametrize("name", ["2", "prof-512"])
def test_device_gevp_matches_host_lanczos(name):
    cfg = problems.CONFIGS[name]
    P = hg.build_problem(name, cstab=None if name == "prof-512" else "cache", one_level=True)
    n_wanted = cfg.cap + 1
    host = problems.solve_local_gevps(P.forms, P.dec, "lanczos", n_wanted=n_wanted)
    dev = problems.solve_local_gevps(P.forms, P.dec, "device", n_wanted=n_wanted)
    worst = 0.0
    for h, d in zip(host, dev):
        k = min(h.eigenvalues.size, d.eigenvalues.size)
        assert k >= n_wanted
        lam_h, lam_d = h.eigenvalues[:k], d.eigenvalues[:k]
        worst = max(worst, float(np.abs(lam_d - lam_h).max() / np.abs(lam_h).max()))
        # C-normalised eigenvectors span the same space (signs free)
        gp = hg.assemble_local_gevp(h.subdomain_index, P.forms, P.dec, dense=False)
        Ch = gp.c_mat @ h.eigenvectors[:, :n_wanted - 1]
        M = d.eigenvectors[:, :n_wanted - 1].T @ Ch  # C-inner products: orthogonal if the spans agree
        s = np.linalg.svd(M, compute_uv=False)
        assert s.min() >= 1.0 - 1e-8, (h.subdomain_index, s.min())
    assert worst <= 1e-10, worst


@pytest.mark.parametrize("name", ["3", "2"])
def test_preconditioner_from_device_gevps(name):
    """Against the host Lanczos restatement (same shifted operator) the
    preconditioners agree to 1e-10.  Against the reference's dense path
    (gamma = 2 k^2 squeezes the finite spectrum into a relative width of
    ~1e-3, so its eigenvectors are the less accurate ones) they agree to
    1e-9."""
    P_lz = hg.build_problem(name, cstab="cache", gevp="lanczos")
    P_dev = hg.build_problem(name, cstab="cache", gevp="device")
    P_dense = hg.build_problem(name, cstab="cache", gevp="dense")
    assert P_dev.selection.m_per_subdomain == P_lz.selection.m_per_subdomain == P_dense.selection.m_per_subdomain
    r = np.random.default_rng(8).standard_normal(P_lz.forms.n_dofs)
    y_lz = hg.factorize(P_lz.forms, P_lz.dec, P_lz.coarse).apply(r)
    y_dev = hg.factorize(P_dev.forms, P_dev.dec, P_dev.coarse).apply(r)
    y_dense = hg.factorize(P_dense.forms, P_dense.dec, P_dense.coarse).apply(r)
    print("%s: device vs host Lanczos %.2e, device vs dense %.2e, host Lanczos vs dense %.2e"
          % (name, rel(y_dev, y_lz), rel(y_dev, y_dense), rel(y_lz, y_dense)))
    assert rel(y_dev, y_lz) <= 1e-10
    assert rel(y_dev, y_dense) <= 1e-9
