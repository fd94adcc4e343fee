"""Times the C-ABI host path (hg_solve_host_batch) against the device-resident solve."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2406_06283_b200 as hg
from paper_2406_06283_b200 import cache
cfg = sys.argv[1] if len(sys.argv) > 1 else "4"
pre, P, info = cache.solver_for_config(cfg)
print(cfg, "tune", pre._meta.get("tune"))
rhs = P.rhs if P.rhs.ndim == 2 else P.rhs[:, None]
Fh = torch.from_numpy(np.ascontiguousarray(rhs.T)).pin_memory().numpy().T
for rep in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    X, reps = pre.solve_host_batch(Fh, rtol=1e-6, maxit=1000)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print("host path %.1f ms, iterations %s" % ((t1 - t0) * 1e3, [r.iterations for r in reps][:3]))
op = pre.as_operator("T")
Fd = torch.from_numpy(np.ascontiguousarray(rhs.T)).cuda()
for rep in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    X, reps = hg.weighted_gmres_batch(op, pre.apply_multi(Fd), weight=P.forms.dk, rtol=1e-6, maxit=1000)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print("device path %.1f ms" % ((t1 - t0) * 1e3))
