"""Shared test helpers (not collected)."""

import types

import numpy as np
import scipy.sparse as sp


def golden_coarse(g, n):
    """A reference-shaped CoarseSpace from config1.npz (Z, B0, column_meta)."""
    Z = sp.csc_matrix((g["Z_data"], g["Z_indices"], g["Z_indptr"]), shape=(n, g["B0"].shape[0]))
    meta = [(i, l) for i, m in enumerate(g["m_per"]) for l in range(int(m))]
    return types.SimpleNamespace(Z=Z, B0=g["B0"], m_total=Z.shape[1], column_meta=meta)


def emulate_band_records(fwd, bwd, n, kl, kv, r):
    """Interpret the packed band-LU records exactly as the device kernel does
    (include/helmgpu.h): pivoted forward sweep, then reversed backward sweep."""
    b = np.array(r, dtype=float, copy=True)
    for j in range(n):
        rec = fwd[j]
        l = int(round(rec[kl]))
        if l != j:
            b[j], b[l] = b[l], b[j]
        t1 = min(kl, n - 1 - j)
        if t1 > 0:
            b[j + 1 : j + 1 + t1] -= rec[0:t1] * b[j]
    for rr in range(n):
        j = n - 1 - rr
        rec = bwd[rr]
        b[j] = b[j] * rec[kv]
        t1 = min(kv, j)
        if t1 > 0:
            b[j - t1 : j][::-1] -= rec[0:t1] * b[j]
    return b
