"""Small end-to-end run for compute-sanitizer (memcheck / racecheck / initcheck):
config 2 (65k dofs, 8x8 subdomains) with its local blocks split in two, one
single apply, one batched apply, a short single solve and a short block solve.

    compute-sanitizer --tool memcheck python tools/sanitize_small.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("HG_LOCAL_SPLIT", "2")
os.environ.setdefault("HG_SPLIT_WORKERS", "1")

import numpy as np

import paper_2406_06283_b200 as hg

P = hg.build_problem(sys.argv[1] if len(sys.argv) > 1 else "2", workers=1)
pre = hg.factorize(P.forms, P.dec, P.coarse)
rng = np.random.default_rng(0)
r = rng.standard_normal(pre.n)
R = rng.standard_normal((pre.n, 16))
a = pre.apply(r)
M = pre.apply_multi(R)
print("apply ok, |a| %.3e; batch col 0 vs single %.2e" % (np.abs(a).max(), np.abs(M[:, 0] - pre.apply(R[:, 0])).max()))
op = pre.as_operator("T")
x, rep = hg.weighted_gmres(op, pre.apply(np.asarray(P.rhs, dtype=float)), weight=P.forms.dk, rtol=0.0, maxit=5)
X, reps = hg.weighted_gmres_batch(op, pre.apply_multi(R), weight=P.forms.dk, rtol=0.0, maxit=4)
x2, rep2 = hg.weighted_gmres(op, pre.apply(np.asarray(P.rhs, dtype=float)), weight=P.forms.dk, rtol=0.0, maxit=5,
                             orth="measured")
print("solves ok:", rep.iterations, [q.iterations for q in reps][:3], rep2.iterations, "split blocks", pre.n_split)
