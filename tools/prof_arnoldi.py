"""Arnoldi-only profiling driver: the batched DCGS2 kernels at config 5's
size (n = 1,046,529, 16 columns) on a diagonal CSR operator and a diagonal
weight, so the profiled region holds nothing but the Krylov machinery.
    python tools/prof_arnoldi.py [maxit]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import scipy.sparse as sp
import torch

import paper_2406_06283_b200 as hg

its = int(sys.argv[1]) if len(sys.argv) > 1 else 40
n = 1_046_529
rng = np.random.default_rng(0)
A = sp.diags(rng.uniform(1.0, 2.0, n)).tocsr()
W = sp.diags(rng.uniform(0.5, 1.5, n)).tocsr()
op = hg.CsrOperator(A)
wt = hg.CsrOperator(W)
F = torch.from_numpy(rng.standard_normal((16, n))).cuda()
for _ in range(2):
    hg.weighted_gmres_batch(op, F, weight=wt, rtol=0.0, maxit=its)
torch.cuda.synchronize()
torch.cuda.profiler.start()
X, reps = hg.weighted_gmres_batch(op, F, weight=wt, rtol=0.0, maxit=its)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("profiled: %d columns x %d iterations" % (len(reps), reps[0].iterations))
