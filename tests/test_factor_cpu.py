"""Band LU records: the packed layout, interpreted with the kernel's exact
semantics, reproduces LAPACK dgbtrs and a dense solve (CPU)."""

import numpy as np
import pytest
import scipy.sparse as sp

import paper_2406_06283_b200 as hg
from paper_2406_06283_b200 import factor
from _helpers import emulate_band_records


def _banded(rng, n, w, weak_diag=False):
    A = np.zeros((n, n))
    for i in range(n):
        for j in range(max(0, i - w), min(n, i + w + 1)):
            A[i, j] = rng.standard_normal()
    if weak_diag:
        A[np.arange(n), np.arange(n)] *= 1e-3  # forces row interchanges
    return sp.csr_matrix(A)


@pytest.mark.parametrize("n,w,weak", [(5, 1, False), (7, 2, False), (50, 5, True), (97, 24, True), (130, 40, False)])
def test_records_match_dgbtrs(n, w, weak):
    rng = np.random.default_rng(n)
    A = _banded(rng, n, w, weak)
    f = factor.band_lu(A)
    assert f.kl == w and f.ku == w
    if weak:
        assert np.any(f.piv != np.arange(n))
    fwd, bwd, fs, bs, klp, kvp = factor.pack_band_records(f)
    assert fs % 2 == 0 and bs % 2 == 0 and fs >= klp + 1 and bs >= kvp + 1
    assert klp >= max(f.kl, 3) and kvp >= max(f.kv, 3)
    b = rng.standard_normal(n)
    x_rec = emulate_band_records(fwd, bwd, n, klp, kvp, b)
    x_lap = f.solve(b)
    x_dense = np.linalg.solve(A.toarray(), b)
    assert np.abs(x_rec - x_lap).max() <= 1e-12 * np.abs(x_lap).max()
    assert np.abs(x_rec - x_dense).max() <= 1e-9 * np.abs(x_dense).max()


def test_helmholtz_blocks_match_superlu(golden):
    P = hg.build_problem("1", workers=1, one_level=True)
    B = P.forms.helmholtz.tocsc()
    import scipy.sparse.linalg as spla

    for i, j, sub in list(P.dec.fine_flat())[:4]:
        blk = B[sub.idof][:, sub.idof]
        f = factor.band_lu(blk, label=(i, j))
        fwd, bwd, _, _, klp, kvp = factor.pack_band_records(f)
        r = np.random.default_rng(i).standard_normal(sub.idof.size)
        x = emulate_band_records(fwd, bwd, f.n, klp, kvp, r)
        ref = spla.splu(blk.tocsc()).solve(r)
        assert np.abs(x - ref).max() <= 1e-11 * np.abs(ref).max()


def test_singular_block_is_named():
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
    blk = forms.helmholtz.tocsc()[idof][:, idof]
    with pytest.raises(hg.SingularOperatorError, match=r"\(0, 0\)"):
        factor.band_lu(blk, label=(0, 0))


def test_record_floor_padding():
    """Narrow blocks are zero padded to the launch's record floor: the padded
    records still solve exactly (zero multipliers) and meet the floor."""
    import numpy as np
    import scipy.sparse as sp

    from _helpers import emulate_band_records

    assert factor.register_tiles(98) == 5 and factor.record_floor(98) == 95
    assert factor.record_floor(24) <= 24 and factor.record_floor(2) == 0
    rng = np.random.default_rng(3)
    n, kl = 60, 4
    A = sp.diags([rng.standard_normal(n - abs(d)) for d in range(-kl, kl + 1)], list(range(-kl, kl + 1))).tocsr()
    A = A + sp.eye(n) * 3.0
    f = factor.band_lu(A)
    fwd, bwd, fs, bs, klp, kvp = factor.pack_band_records(f, kl_floor=31, kv_floor=40)
    assert klp == 31 and kvp == 40 and fs >= 32 and bs >= 41
    r = rng.standard_normal(n)
    got = emulate_band_records(fwd.reshape(n, fs), bwd.reshape(n, bs), n, klp, kvp, r)
    assert np.abs(got - f.solve(r)).max() <= 1e-12 * np.abs(f.solve(r)).max()


def test_split_block_is_the_same_local_operator():
    """factor.split_block (chunks + separators + spikes) against dgbtrs of the
    whole block, and the descriptor arrays the device consumes (helmgpu.h
    "Split local blocks") interpreted exactly as hg_split.cu does."""
    import os

    import paper_2406_06283_b200 as hg
    from paper_2406_06283_b200 import factor, schwarz
    from _helpers import emulate_band_records

    P = hg.build_problem("1", workers=1, one_level=True)
    B = P.forms.helmholtz.tocsr()
    subs = [np.asarray(sub.idof) for _, _, sub in P.dec.fine_flat()]
    rng = np.random.default_rng(2)
    blk = factor.submatrix(B, subs[5], subs[5])
    whole = factor.band_lu(blk)
    r = rng.standard_normal(blk.shape[0])
    for nchunk in (2, 3):
        sb = factor.split_block(blk, nchunk)
        assert len(sb.chunks) == nchunk and sb.sep_rows.size == (nchunk - 1) * whole.kl
        assert np.abs(sb.solve(r) - whole.solve(r)).max() <= 1e-12 * np.abs(whole.solve(r)).max()
    assert factor.split_block(blk, 6) is None  # chunks shorter than four band widths: declined

    old = os.environ.get("HG_LOCAL_SPLIT")
    os.environ["HG_LOCAL_SPLIT"] = "2"
    try:
        A, M = schwarz.host_image(P.forms, P.dec, None)
    finally:
        if old is None:
            del os.environ["HG_LOCAL_SPLIT"]
        else:
            os.environ["HG_LOCAL_SPLIT"] = old
    assert M["n_split"] == len(subs) and M["n_local"] == 3 * len(subs)
    rg = rng.standard_normal(B.shape[0])
    xs = np.zeros(int(A["local_idx_off"][-1]))
    off, idx = A["local_idx_off"], A["local_idx"]
    for b in range(M["n_local"]):  # chunk solves from the packed records
        n = int(A["local_n"][b])
        if n == 0:
            continue
        fs, bs = int(A["local_fstride"][b]), int(A["local_bstride"][b])
        fw = A["local_fwd"][A["local_fwd_off"][b]:A["local_fwd_off"][b] + n * fs].reshape(n, fs)
        bw = A["local_bwd"][A["local_bwd_off"][b]:A["local_bwd_off"][b] + n * bs].reshape(n, bs)
        xs[off[b]:off[b] + n] = emulate_band_records(fw, bw, n, int(A["local_kl"][b]), int(A["local_kv"][b]),
                                                    rg[idx[off[b]:off[b] + n]])
    xsep = np.zeros(int(A["split_row_off"][-1]))
    for s in range(M["n_split"]):  # separators
        r0, r1 = int(A["split_row_off"][s]), int(A["split_row_off"][s + 1])
        pb = int(A["split_blk"][s])
        t = rg[idx[off[pb]:off[pb + 1]]].copy()
        for k in range(r1 - r0):
            a, e = int(A["split_f_indptr"][r0 + k]), int(A["split_f_indptr"][r0 + k + 1])
            t[k] -= A["split_f_val"][a:e] @ xs[A["split_f_pos"][a:e]]
        ns = r1 - r0
        so = int(A["split_sinv_off"][s])
        xsep[r0:r1] = A["split_sinv"][so:so + ns * ns].reshape(ns, ns) @ t
        xs[off[pb]:off[pb] + ns] = xsep[r0:r1]
    for i in range(M["n_spike"]):  # spikes, from the packed fragment blocks
        b, s = int(A["spike_blk"][i]), int(A["spike_split"][i])
        n, w, c0 = int(A["local_n"][b]), int(A["spike_w"][i]), int(A["spike_col0"][i])
        mt = (n + 7) // 8
        pk = A["spike_data"][A["spike_off"][i]:A["spike_off"][i] + mt * 8 * w].reshape(mt, w // 8, 8, 4, 2)
        W = pk.transpose(0, 2, 1, 4, 3).reshape(mt * 8, w)[:n]  # (mt, g, kb, h, q)
        r0 = int(A["split_row_off"][s])
        ns = int(A["split_row_off"][s + 1]) - r0
        xv = np.zeros(w)
        k = min(w, ns - c0)
        xv[:k] = xsep[r0 + c0:r0 + c0 + k]
        xs[off[b]:off[b] + n] -= W @ xv
    # assemble in block order and compare with the sum of whole-block solves
    got = np.zeros(B.shape[0])
    for b in range(M["n_local"]):
        np.add.at(got, idx[off[b]:off[b + 1]], xs[off[b]:off[b + 1]])
    want = np.zeros(B.shape[0])
    for idof in subs:
        want[idof] += factor.band_lu(factor.submatrix(B, idof, idof)).solve(rg[idof])
    assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()
