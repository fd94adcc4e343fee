"""Setup-phase timings of one configuration, host vs device paths.
python tools/prof_setup.py [config] [gevp: auto|device]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("HG_SETUP_TIMING", "1")

import numpy as np

import paper_2406_06283_b200 as hg

cfg = sys.argv[1] if len(sys.argv) > 1 else "5-16"
gevp = sys.argv[2] if len(sys.argv) > 2 else "device"
t0 = time.perf_counter()
P = hg.build_problem(cfg, cstab="cache", gevp=gevp, verbose=True)
print("build_problem %.1f s" % (time.perf_counter() - t0), {k: round(v, 2) for k, v in P.times.items()})
print("coarse", getattr(P.coarse, "build_seconds", None), "m", P.coarse.m_total, "removed", len(P.coarse.removed),
      "has lu", getattr(P.coarse, "_b0_lu", None) is not None)
t0 = time.perf_counter()
pre = hg.factorize(P.forms, P.dec, P.coarse)
print("factorize %.1f s" % (time.perf_counter() - t0), {k: round(v, 2) for k, v in pre.setup_times.items()},
      "device factor", pre.device_factor, "panel", pre.panel_active)
r = np.random.default_rng(0).standard_normal(pre.n)
x = pre.apply(r)
print("apply ok", float(np.abs(x).max()))
