"""Component-wise parity diagnosis at a BASELINE config (GPU box):
SpMV, every local solve vs the host band LU, the coarse part and the whole
apply vs the CPU oracle.   python tools/diag_parity.py [config ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np

import paper_2406_06283_b200 as hg
from oracle.schwarz_oracle import OraclePreconditioner


def rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300))


for name in sys.argv[1:] or ["4"]:
    t0 = time.time()
    P = hg.build_problem(name, cstab="cache")
    pre = hg.factorize(P.forms, P.dec, P.coarse)
    print("[%s] setup %.0f s, n=%d, m=%d, b0_mode=%d, bands rf/rb from kl/kv max %s" % (
        name, time.time() - t0, pre.n, pre.m, pre.b0_mode,
        (max(k for k, _ in pre.local_bands), max(v for _, v in pre.local_bands))), flush=True)
    rng = np.random.default_rng(1)
    r = rng.standard_normal(pre.n)
    print("  spmv B bitwise:", np.array_equal(pre.spmv(r, "B"), P.forms.helmholtz @ r), flush=True)
    worst, bad = 0.0, []
    for s, ls in enumerate(pre.local_solvers):
        x = rng.standard_normal(ls.idof.size)
        e = rel(ls.lu.solve(x), ls.lu.host.solve(x))
        worst = max(worst, e)
        if e > 1e-10:
            bad.append((s, ls.idof.size, ls.lu.host.kl, ls.lu.host.kv, e))
    print("  local solves: worst %.2e, bad %d %s" % (worst, len(bad), bad[:5]), flush=True)
    orc = OraclePreconditioner(P.forms, P.dec, P.coarse, b0_lu=pre.b0_piv)
    print("  apply_coarse vs oracle: %.2e" % rel(pre.apply_coarse(r), orc.apply_coarse(r)), flush=True)
    print("  apply vs oracle: %.2e" % rel(pre.apply(r), orc.apply(r)), flush=True)
    R = np.stack([r, rng.standard_normal(pre.n)], axis=1)
    M = pre.apply_multi(R)
    print("  apply_multi col0 vs oracle: %.2e" % rel(M[:, 0], orc.apply(r)), flush=True)
