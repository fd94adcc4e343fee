import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2406_06283_b200 as hg
P = hg.build_problem("1", workers=1, one_level=False)
pre = hg.factorize(P.forms, P.dec, P.coarse)
print("mode", pre.b0_mode, "m", pre.m, flush=True)
r = np.random.default_rng(0).standard_normal(pre.n)
print("coarse", np.abs(pre.apply_coarse(r)).max(), flush=True)
print("profile", pre.profile(r, 2), flush=True)
print("apply", np.abs(pre.apply(r)).max(), flush=True)
