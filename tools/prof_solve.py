"""Profiling driver: set up a config, warm up, then run ONE fixed-length GMRES
solve (rtol = 0, maxit from argv) between cudaProfilerStart/Stop, so that
`ncu --profile-from-start off` captures exactly that solve's kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2406_06283_b200 as hg

cfg = sys.argv[1] if len(sys.argv) > 1 else "5-16"
its = int(sys.argv[2]) if len(sys.argv) > 2 else 8
P = hg.build_problem(cfg, cstab=None if cfg.startswith("prof") else "cache",
                     workers=int(os.environ.get("SETUP_WORKERS", "0")) or None)
pre = hg.factorize(P.forms, P.dec, P.coarse)
f = P.rhs if P.rhs.ndim == 1 else P.rhs[:, 0]
fd = torch.from_numpy(np.ascontiguousarray(f)).cuda()
op = pre.as_operator("T")
for _ in range(2):
    hg.weighted_gmres(op, pre.apply(fd), weight=P.forms.dk, rtol=0.0, maxit=its)
torch.cuda.synchronize()
torch.cuda.profiler.start()
x, rep = hg.weighted_gmres(op, pre.apply(fd), weight=P.forms.dk, rtol=0.0, maxit=its)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("profiled solve: %d iterations, residual %.3e" % (rep.iterations, rep.residual_history[-1]))
