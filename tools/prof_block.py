"""Profiling driver for the batched (16-RHS block) solve: set up a config,
warm up, then run ONE fixed-length batched solve (rtol = 0, maxit from argv)
between cudaProfilerStart/Stop, so that `ncu --profile-from-start off`
captures exactly that solve's kernels.

    python tools/prof_block.py [config] [maxit] [orth]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2406_06283_b200 as hg

cfg = sys.argv[1] if len(sys.argv) > 1 else "5-16"
its = int(sys.argv[2]) if len(sys.argv) > 2 else 8
orth = sys.argv[3] if len(sys.argv) > 3 else "dcgs2"
P = hg.build_problem(cfg, cstab=None if cfg.startswith("prof") else "cache",
                     workers=int(os.environ.get("SETUP_WORKERS", "0")) or None)
pre = hg.factorize(P.forms, P.dec, P.coarse)
F = P.rhs if P.rhs.ndim == 2 else np.repeat(P.rhs[:, None], 16, axis=1)
Fd = torch.from_numpy(np.ascontiguousarray(F.T)).cuda()
op = pre.as_operator("T")
for _ in range(2):
    hg.weighted_gmres_batch(op, pre.apply_multi(Fd), weight=P.forms.dk, rtol=0.0, maxit=its, orth=orth)
torch.cuda.synchronize()
torch.cuda.profiler.start()
X, reps = hg.weighted_gmres_batch(op, pre.apply_multi(Fd), weight=P.forms.dk, rtol=0.0, maxit=its, orth=orth)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("profiled block solve: %d columns x %d iterations" % (len(reps), reps[0].iterations))
