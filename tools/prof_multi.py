"""Timing of the batched (multi-RHS) path at a BASELINE config: single vs
batched apply, batched stage profile, one batched GMRES solve with phase
stats.  python tools/prof_multi.py [config] [nrhs] [maxit]"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2406_06283_b200 as hg
from paper_2406_06283_b200 import _lib

cfg = sys.argv[1] if len(sys.argv) > 1 else "5-16"
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 16
maxit = int(sys.argv[3]) if len(sys.argv) > 3 else 1000
P = hg.build_problem(cfg, cstab="cache")
pre = hg.factorize(P.forms, P.dec, P.coarse)
F = P.rhs if P.rhs.ndim == 2 else np.repeat(P.rhs[:, None], nrhs, axis=1)
F = F[:, :nrhs]
R = torch.from_numpy(np.ascontiguousarray(F.T)).cuda()
lib = _lib.load()


def timed(fn, reps):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


t1 = timed(lambda: pre.apply(R[0]), 20)
tm = timed(lambda: pre.apply_multi(R), 10)
print("apply single %.3f ms; apply_multi(%d) %.3f ms = %.3f ms/column" % (t1, nrhs, tm, tm / nrhs))
print("stages single:", {k: round(v, 4) for k, v in pre.profile(R[0], iters=5).items()})
print("stages multi :", {k: round(v, 4) for k, v in pre.profile_multi(R, iters=5).items()})
out = pre.apply_multi(R).cpu().numpy()
for c in (0, nrhs - 1):
    s = pre.apply(R[c]).cpu().numpy()
    print("col %d multi vs single rel %.2e" % (c, np.abs(out[c] - s).max() / np.abs(s).max()))

op = pre.as_operator("T")
Rp = pre.apply_multi(R)
lib.hg_stats_enable(1)
lib.hg_stats_read(None, None, 1)
torch.cuda.synchronize()
t0 = time.perf_counter()
X, reps = hg.weighted_gmres_batch(op, Rp, weight=P.forms.dk, rtol=P.config.rtol, maxit=maxit, orth="dcgs2")
torch.cuda.synchronize()
dt = time.perf_counter() - t0
ms = np.zeros(_lib.NPHASES)
cnt = np.zeros(_lib.NPHASES, dtype=np.int64)
lib.hg_stats_read(_lib.ptr(ms, ctypes.c_double), _lib.ptr(cnt, ctypes.c_int64), 1)
its = [r.iterations for r in reps]
print("batched GMRES: %.2f s, iterations %s, total %d -> %.1f iters/s" % (dt, its, sum(its), sum(its) / dt))
print("phases (ms):", dict(zip(_lib.PHASES, np.round(ms, 1))), "sum %.1f" % ms.sum())
print("reorth:", [r.reorth_passes for r in reps])
lib.hg_stats_enable(0)

# single-RHS solves, both orthogonalisation schemes, with phase stats
f0 = pre.apply(R[0])
for orth in ("dcgs2", "measured", "dcgs2"):
    lib.hg_stats_enable(1)
    lib.hg_stats_read(None, None, 1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, rep = hg.weighted_gmres(op, f0, weight=P.forms.dk, rtol=P.config.rtol, maxit=maxit, orth=orth)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    lib.hg_stats_read(_lib.ptr(ms, ctypes.c_double), _lib.ptr(cnt, ctypes.c_int64), 1)
    print("single %-8s: %.3f s, %d iterations -> %.1f iters/s; phases %s sum %.1f" % (
        orth, dt, rep.iterations, rep.iterations / dt, dict(zip(_lib.PHASES, np.round(ms, 1))), ms.sum()))
lib.hg_stats_enable(0)
# batched again (workspace mapped now), both schemes
for orth in ("dcgs2", "measured"):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    X, reps = hg.weighted_gmres_batch(op, Rp, weight=P.forms.dk, rtol=P.config.rtol, maxit=maxit, orth=orth)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    its = [r.iterations for r in reps]
    print("batched %-8s: %.2f s, total %d iterations -> %.1f iters/s; its %s" % (orth, dt, sum(its), sum(its) / dt, its))
