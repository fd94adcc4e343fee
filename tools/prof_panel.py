"""Batched apply at the profiler stand-in config (prof-512: 5-16's block
shape at a quarter of the size) for ncu captures of the batched kernels.
python tools/prof_panel.py [config] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2406_06283_b200 as hg

cfg = sys.argv[1] if len(sys.argv) > 1 else "prof-512"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
P = hg.build_problem(cfg, cstab=None if cfg == "prof-512" else "cache", workers=int(os.environ.get("HG_WORKERS", "0")) or None)
pre = hg.factorize(P.forms, P.dec, P.coarse)
print("panel active", pre.panel_active, "deviation %.2e" % pre.panel_deviation, "bytes %.3f GB" % (pre.panel_bytes / 1e9))
R = torch.from_numpy(np.random.default_rng(0).standard_normal((16, pre.n))).cuda()
for _ in range(reps):
    pre.apply_multi(R)
torch.cuda.synchronize()
print({k: round(v, 4) for k, v in pre.profile_multi(R, iters=3).items()})
