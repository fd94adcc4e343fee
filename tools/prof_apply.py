"""Profiling driver: set up one config, then run a few applies (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2406_06283_b200 as hg

cfg = sys.argv[1] if len(sys.argv) > 1 else "5-16"
n_apply = int(sys.argv[2]) if len(sys.argv) > 2 else 3
P = hg.build_problem(cfg, cstab=None if cfg.startswith("prof") else "cache", workers=int(os.environ.get("SETUP_WORKERS", "0")) or None)
pre = hg.factorize(P.forms, P.dec, P.coarse)
r = torch.from_numpy(np.random.default_rng(0).standard_normal(pre.n)).cuda()
for _ in range(n_apply):
    pre.apply(r)
torch.cuda.synchronize()
print("stages", pre.profile(r, iters=3))
