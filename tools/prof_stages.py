"""Apply timings and serialised stage profiles (single and batched) of a
BASELINE config, from the setup cache.  python tools/prof_stages.py [config]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2406_06283_b200 as hg
from paper_2406_06283_b200 import cache

cfg = sys.argv[1] if len(sys.argv) > 1 else "5-16"
pre, P, info = cache.solver_for_config(cfg)
R = torch.from_numpy(np.random.default_rng(0).standard_normal((16, pre.n))).cuda()


def timed(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


t1 = timed(lambda: pre.apply(R[0]), 50)
tm = timed(lambda: pre.apply_multi(R), 30)
env = {k: v for k, v in os.environ.items() if k.startswith("HG_") and k != "HG_CACHE_DIR"}
print("%s %s cache_hit=%s: apply %.4f ms, apply_multi(16) %.4f ms" % (cfg, env, info["hit"], t1, tm))
print("  single:", {k: round(v, 4) for k, v in pre.profile(R[0], iters=10).items()})
print("  multi :", {k: round(v, 4) for k, v in pre.profile_multi(R, iters=10).items()})
out = pre.apply_multi(R).cpu().numpy()
s = pre.apply(R[5]).cpu().numpy()
print("  col 5 multi vs single rel %.2e" % (np.abs(out[5] - s).max() / np.abs(s).max()))
