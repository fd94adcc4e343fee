"""Device factorisation of the local blocks (VERDICT r1
item 7): the band LU the GPU builds (hg_factor.cu, dgbtrf semantics) against
LAPACK dgbtrf on the host (factor.band_lu, what the reference's SuperLU
factorisation is restated as, schwarz.py:104-131): identical pivots, factors
equal to rounding, the same applies (golden vectors of the reference), and
the reference's singular-block test naming the (i, j) pair."""

import numpy as np
import pytest

import paper_2406_06283_b200 as hg
from _helpers import golden_coarse

pytestmark = pytest.mark.gpu


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def compare_records(dev, host):
    A, B = dev._image_arrays, host._image_arrays
    for name in ("local_n", "local_kl", "local_kv", "local_fstride", "local_bstride", "local_fwd_off",
                 "local_bwd_off", "local_idx"):
        assert np.array_equal(A[name], B[name]), name
    worst_l = worst_u = 0.0
    piv_diff = swaps = 0
    for s in range(len(A["local_n"])):
        n, fs, bs = int(A["local_n"][s]), int(A["local_fstride"][s]), int(A["local_bstride"][s])
        klp, kvp = int(A["local_kl"][s]), int(A["local_kv"][s])
        if n == 0:
            continue
        fo, bo = int(A["local_fwd_off"][s]), int(A["local_bwd_off"][s])
        fd = np.asarray(A["local_fwd"][fo:fo + n * fs]).reshape(n, fs)
        fh = np.asarray(B["local_fwd"][fo:fo + n * fs]).reshape(n, fs)
        bd = np.asarray(A["local_bwd"][bo:bo + n * bs]).reshape(n, bs)
        bh = np.asarray(B["local_bwd"][bo:bo + n * bs]).reshape(n, bs)
        piv_diff += int(np.sum(fd[:, klp] != fh[:, klp]))
        swaps += int(np.sum(fh[:, klp] != np.arange(n)))
        worst_l = max(worst_l, rel(fd[:, :klp], fh[:, :klp]))
        worst_u = max(worst_u, rel(bd[:, :kvp], bh[:, :kvp]), rel(bd[:, kvp], bh[:, kvp]))
        assert np.all(fd[:, klp + 1:] == 0.0) and np.all(bd[:, kvp + 1:] == 0.0)  # record padding
    return piv_diff, worst_l, worst_u, swaps


@pytest.fixture(scope="module")
def cfg1(golden):
    g = golden("config1")
    P = hg.build_problem("1", workers=1, one_level=True)
    return P, g, golden_coarse(g, P.forms.n_dofs)


def test_device_band_lu_matches_dgbtrf_config1(cfg1, monkeypatch):
    P, g, coarse = cfg1
    dev = hg.factorize(P.forms, P.dec, coarse, keep_image=True)
    assert dev.device_factor
    monkeypatch.setenv("HG_HOST_FACTOR", "1")
    host = hg.factorize(P.forms, P.dec, coarse, keep_image=True)
    assert not host.device_factor
    piv_diff, wl, wu, _ = compare_records(dev, host)
    assert piv_diff == 0 and wl <= 1e-12 and wu <= 1e-12, (piv_diff, wl, wu)
    assert rel(dev.apply(g["r"]), g["apply_r"]) <= 1e-10
    assert rel(dev.apply(g["r"]), host.apply(g["r"])) <= 1e-12
    x, rep = hg.weighted_gmres(dev.as_operator("T"), g["rhs_p"], weight=P.forms.dk, rtol=1e-6, maxit=1000)
    assert rep.iterations == int(g["iterations"]) and rel(x, g["x"]) <= 1e-8


@pytest.mark.parametrize("name", ["2", "3"])
def test_device_band_lu_matches_dgbtrf_configs_2_3(name, monkeypatch):
    """64 blocks of ~1200 dofs, pivoting blocks included (k = 40)."""
    P = hg.build_problem(name, one_level=True)
    dev = hg.factorize(P.forms, P.dec, None, keep_image=True)
    monkeypatch.setenv("HG_HOST_FACTOR", "1")
    host = hg.factorize(P.forms, P.dec, None, keep_image=True)
    piv_diff, wl, wu, swaps = compare_records(dev, host)
    assert piv_diff == 0 and wl <= 1e-11 and wu <= 1e-11, (piv_diff, wl, wu)
    if name == "2":
        assert swaps > 0  # partial pivoting exercised (pivots occur at k = 40, constant coefficient)
    r = np.random.default_rng(1).standard_normal(dev.n)
    assert rel(dev.apply(r), host.apply(r)) <= 1e-11


def test_device_factor_names_the_singular_block():
    # k^2 exactly on a Dirichlet eigenvalue of the first fine block (test_schwarz.py:164-180)
    import scipy.linalg

    mesh = hg.build_unit_square_mesh(8)
    space = hg.build_fe_space(mesh)
    probe = hg.assemble_forms(mesh, space, hg.coefficient_field(mesh), 1.0)
    dec = hg.build_two_level(mesh, space, 2, 2)
    idof = dec.fine[0][0].idof
    mu = scipy.linalg.eigh(probe.stiffness[idof][:, idof].toarray(), probe.mass[idof][:, idof].toarray(),
                           eigvals_only=True)[0]
    forms = hg.assemble_forms(mesh, space, hg.coefficient_field(mesh), np.sqrt(mu))
    with pytest.raises(hg.SingularOperatorError, match=r"\(0, 0\)"):
        pre = hg.factorize(forms, dec, None)
        assert pre.device_factor
