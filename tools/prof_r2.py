"""Round-2 profiling driver: the preconditioner comes from the on-disk setup
cache (HG_CACHE_DIR; the first, plain run writes it, the ncu run loads it),
then, between cudaProfilerStart/Stop: `napply` single applies, `napply`
batched applies and ONE fixed-length 16-RHS block solve (rtol = 0).

    python tools/prof_r2.py [config] [iterations] [napply]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2406_06283_b200 as hg
from paper_2406_06283_b200 import cache

cfg = sys.argv[1] if len(sys.argv) > 1 else "5-16"
its = int(sys.argv[2]) if len(sys.argv) > 2 else 8
napply = int(sys.argv[3]) if len(sys.argv) > 3 else 2
pre, P, info = cache.solver_for_config(cfg)
print("setup cache hit" if info["hit"] else "setup built", "%.1f s" % info["seconds"], flush=True)
F = P.rhs if P.rhs.ndim == 2 else np.repeat(P.rhs[:, None], 16, axis=1)
Fd = torch.from_numpy(np.ascontiguousarray(F.T)).cuda()
op = pre.as_operator("T")
for _ in range(2):
    pre.apply(Fd[0])
    hg.weighted_gmres_batch(op, pre.apply_multi(Fd), weight=P.forms.dk, rtol=0.0, maxit=its, orth="dcgs2")
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(napply):
    pre.apply(Fd[0])
for _ in range(napply):
    pre.apply_multi(Fd)
X, reps = hg.weighted_gmres_batch(op, pre.apply_multi(Fd), weight=P.forms.dk, rtol=0.0, maxit=its, orth="dcgs2")
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("profiled: %d applies, %d batched applies, block solve %d columns x %d iterations" % (
    napply, napply, len(reps), reps[0].iterations))
