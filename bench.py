#!/usr/bin/env python
"""Benchmark of the B200 solve phase (two-level Schwarz / H_k-GenEO, weighted GMRES).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 5-16]

A step is one preconditioned solve of one right-hand side of the workload
(rhs_p = M^{-1} f, then full D_k-weighted GMRES to rtol 1e-6 from x0 = 0,
exactly cli.run_single's solve block, cli.py:297-307).  The workload is
BASELINE config 5 at 16x16 subdomains (the north star's ~1M-dof k=100
config): n = 1024 (1,046,529 dofs), k = 100, a(x) log-uniform [1, 10] on
64x64 cells (seed 5), overlap 4, cap 60 modes per subdomain (m = 15,360),
right-hand sides = the config's 16 seeded N(0,1) load vectors.

value   = GMRES iterations/s over the whole job, inputs resident in HBM
e2e     = the same metric through the C ABI hg_solve_host with host buffers
          (H2D of f and D2H of x inside the timed region)
roofline= the dominant kernel of the apply, timed live with CUDA events
cpu_baseline = the CPU oracle (oracle/, a restatement of the reference's
          SuperLU / LAPACK / numpy solve path) on a bounded sample.

Multi-GPU: one process per GPU (torchrun); ranks solve disjoint right-hand
sides (weak scaling, no data-path collective); time = max over ranks.
``--impl reference`` times the CPU oracle port on rank 0 only.
"""

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="5-16")
    ap.add_argument("--cpu-iters", type=int, default=6, help="GMRES iterations in the CPU baseline sample")
    ap.add_argument("--ref-iters", type=int, default=3, help="GMRES iterations per reference-arm step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cstab", default="cache", help="'cache' (recorded setup constant), 'auto' (recompute)")
    return ap.parse_args()


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------- distributed
class Dist:
    def __init__(self, backend):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        if self.world > 1:
            import torch.distributed as dist

            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group(backend)
            self.pg = dist

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def max(self, x):
        if not self.pg:
            return x
        import torch

        t = torch.tensor([float(x)], device="cuda" if self.pg.get_backend() == "nccl" else "cpu", dtype=torch.float64)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x):
        if not self.pg:
            return x
        import torch

        t = torch.tensor([float(x)], device="cuda" if self.pg.get_backend() == "nccl" else "cpu", dtype=torch.float64)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.SUM)
        return float(t.item())

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


def shard_columns(step, rank, world, nrhs):
    """Right-hand side column solved by `rank` at `step` (disjoint across ranks)."""
    return (step * world + rank) % nrhs


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(index), "--query-gpu=" + self.FIELDS, "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
                for nm, v in zip(names, r[4:8]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- byte model
def stage_bytes(pre):
    """Algorithmic HBM bytes of each apply stage."""
    nloc = pre.local_sizes
    loc = sum(8 * n * (kl + kv + 1) + 4 * n + 12 * n + 8 * n for n, (kl, kv) in zip(nloc, pre.local_bands))
    zt = zy = asm = b0 = 0
    if pre.has_coarse:
        zt = sum(8 * n * m + 12 * n for n, m in pre.cblock_shapes)
        zy = sum(8 * n * m + 8 * n for n, m in pre.cblock_shapes) + 8 * pre.m
        b0 = pre.b0_bytes
    asm = 8 * sum(nloc) + (8 * sum(n for n, _ in pre.cblock_shapes) if pre.has_coarse else 0) + 8 * pre.n
    return {"zt": zt, "b0_solve": b0, "zy": zy, "local": loc, "assemble": asm}


def solve_bytes(pre, nnz, iters):
    """Algorithmic bytes of one solve of `iters` iterations (SURVEY §8d model)."""
    n = pre.n
    s_spmv = 12 * nnz + 4 * (n + 1) + 16 * n
    s_apply = sum(stage_bytes(pre).values())
    total = s_apply  # rhs_p = M^{-1} f
    for j in range(iters):
        total += 2 * s_spmv + s_apply + (32 * (j + 1) + 64) * n
    total += 8 * n * iters  # x = V y
    return total


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json, burst copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel_key):
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(path):
        with open(path) as fh:
            return json.load(fh).get(kernel_key)
    return None


# ---------------------------------------------------------------- arms
def run_ours(args, dist):
    import torch

    import paper_2406_06283_b200 as hg
    from paper_2406_06283_b200 import _lib

    torch.cuda.set_device(dist.local)
    t0 = time.perf_counter()
    P = hg.build_problem(args.config, cstab=args.cstab, verbose=dist.rank == 0)
    t_setup = time.perf_counter() - t0
    t0 = time.perf_counter()
    pre = hg.factorize(P.forms, P.dec, P.coarse)
    t_fact = time.perf_counter() - t0
    setup = dict(P.times)
    setup["factorize_upload"] = t_fact
    log("setup %.1f s + factorize/upload %.1f s; device bytes %.2f GB" % (t_setup, t_fact, pre.device_bytes / 1e9))

    rhs_host = P.rhs if P.rhs.ndim == 2 else P.rhs[:, None]
    nrhs = rhs_host.shape[1]
    rhs_dev = torch.from_numpy(np.ascontiguousarray(rhs_host.T)).cuda()  # (nrhs, n), resident in HBM
    op = pre.as_operator("T")
    Dk = P.forms.dk
    rtol, maxit = P.config.rtol, P.config.maxit
    stream = torch.cuda.current_stream()

    def solve(col):
        rhs_p = pre.apply(rhs_dev[col])
        x, rep = hg.weighted_gmres(op, rhs_p, weight=Dk, rtol=rtol, maxit=maxit)
        return rep

    for s in range(args.warmup):
        rep = solve(shard_columns(s, dist.rank, dist.world, nrhs))
        log("warmup %d: %d iterations, converged=%s" % (s, rep.iterations, rep.converged))
    dist.barrier()
    torch.cuda.synchronize()
    launches0 = _lib.load().hg_kernel_launches()
    clocks = ClockSampler(dist.local)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters = 0
    ev0.record(stream)
    for s in range(args.steps):
        rep = solve(shard_columns(args.warmup + s, dist.rank, dist.world, nrhs))
        iters += rep.iterations
    ev1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    dist.barrier()
    launches = int(_lib.load().hg_kernel_launches() - launches0)
    ms_local = ev0.elapsed_time(ev1)
    ms = dist.max(ms_local)
    iters_all = dist.sum(iters)
    value = iters_all / (ms / 1e3)

    # applies/s (device-resident input), its stage profile and the kernel roofline
    r = rhs_dev[0]
    out = torch.empty_like(r)
    for _ in range(3):
        pre.apply(r)
    torch.cuda.synchronize()
    na = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(na):
        pre.apply(r)
    e1.record(stream)
    torch.cuda.synchronize()
    apply_ms = e0.elapsed_time(e1) / na
    stages = pre.profile(r, iters=5)
    sb = stage_bytes(pre)
    peak, peak_src = peaks()
    dom = max(stages, key=lambda k: stages[k])
    kern = {"local": "k_local_solve", "b0_solve": "k_b0_solve", "zt": "k_zt", "zy": "k_zy", "assemble": "k_assemble"}
    ach = sb[dom] / (stages[dom] / 1e3) / 1e9
    roofline = {"kernel": kern[dom], "bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                "frac": round(ach / peak, 4), "traffic": ncu_traffic(kern[dom]), "peak_source": peak_src,
                "algorithmic_bytes": sb[dom], "ms": round(stages[dom], 4)}
    per_stage = {k: {"ms": round(stages[k], 4), "bytes": sb[k],
                     "GBps": round(sb[k] / max(stages[k], 1e-9) / 1e6, 1)} for k in stages}
    it_per_solve = iters / max(args.steps, 1)
    sbytes = solve_bytes(pre, P.forms.helmholtz.nnz, int(round(it_per_solve)))
    solve_ms = ms_local / max(args.steps, 1)
    solve_roof = {"bytes_per_solve": sbytes, "achieved": round(sbytes / (solve_ms / 1e3) / 1e9, 1),
                  "frac": round(sbytes / (solve_ms / 1e3) / 1e9 / peak, 4), "unit": "GB/s"}

    # e2e through the C ABI with host buffers
    e2e = None
    if not args.no_e2e:
        fh = torch.from_numpy(np.ascontiguousarray(rhs_host[:, 0])).pin_memory().numpy()
        pre.solve_host(fh, rtol=rtol, maxit=maxit)
        torch.cuda.synchronize()
        dist.barrier()
        e0.record(stream)
        it_e2e = 0
        for s in range(args.steps):
            col = shard_columns(args.warmup + s, dist.rank, dist.world, nrhs)
            fh = torch.from_numpy(np.ascontiguousarray(rhs_host[:, col])).pin_memory().numpy()
            x, rep = pre.solve_host(fh, rtol=rtol, maxit=maxit)
            it_e2e += rep.iterations
        e1.record(stream)
        torch.cuda.synchronize()
        ms_e2e = dist.max(e0.elapsed_time(e1))
        e2e = {"value": round(dist.sum(it_e2e) / (ms_e2e / 1e3), 3), "unit": "iters/s",
               "h2d_bytes_per_step": 8 * pre.n, "d2h_bytes_per_step": 8 * pre.n + 8 * (maxit + 1),
               "path": "hg_solve_host (C ABI, host f in, host x out)"}

    cpu = None
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(P, pre, args.cpu_iters)
    n = pre.n
    line = {
        "metric": "GMRES iters/s (FP64, two-level Schwarz + H_k-GenEO, D_k-weighted)",
        "value": round(value, 3),
        "unit": "iters/s",
        "n_gpus": dist.world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms / max(args.steps, 1), 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic, seeded (coefficient seed %d, rhs seeds %d+c)" % (P.config.coeff_seed, P.config.rhs_seed),
        "config": {
            "workload": "BASELINE config %s: n=%d (%d dofs), k=%g, %dx%d subdomains, overlap %d, cap %d (m=%d), "
                        "a log-uniform[%g,%g] on %dx%d cells" % (
                            P.config.name, P.config.n, n, P.config.k, P.config.M, P.config.M, P.config.layers,
                            P.config.cap, pre.m, P.config.coeff_lo, P.config.coeff_hi, P.config.coeff_cells,
                            P.config.coeff_cells),
            "step": "rhs_p = M^-1 f; full weighted GMRES to rtol %g from x0=0 (one rhs per rank per step)" % rtol,
            "l2": "inputs larger than L2: %.2f GB device-resident factors/Z/B0 vs 126 MB L2" % (pre.device_bytes / 1e9),
            "iters_per_solve": round(it_per_solve, 2),
            "parallelism": "rhs-parallel replicas x%d" % dist.world,
        },
        "applies_per_s": round(1e3 / apply_ms, 2),
        "apply_ms": round(apply_ms, 4),
        "stage_ms_serialised": per_stage,
        "solve_roofline": solve_roof,
        "roofline": roofline,
        "setup_s": {k: round(v, 2) for k, v in setup.items()},
        "gpu_launches": launches,
        "clocks": clk,
    }
    if e2e:
        line["e2e"] = e2e
    if cpu:
        line["cpu_baseline"] = cpu
    return line


def cpu_baseline(P, pre, iters):
    """The oracle (restated reference solve path) on a bounded sample of the workload."""
    from oracle.schwarz_oracle import OraclePreconditioner
    from oracle.wgmres_oracle import weighted_gmres as oracle_gmres

    cores = len(os.sched_getaffinity(0))
    orc = OraclePreconditioner(P.forms, P.dec, P.coarse, b0_lu=pre.b0_piv)
    f = P.rhs if P.rhs.ndim == 1 else P.rhs[:, 0]
    B, Dk = P.forms.helmholtz, P.forms.dk
    t0 = time.perf_counter()
    rhs_p = orc.apply(f)
    x, info = oracle_gmres(lambda v: orc.apply(B @ v), rhs_p, weight=Dk, rtol=0.0, maxit=iters)
    dt = time.perf_counter() - t0
    t0 = time.perf_counter()
    orc.apply(f)
    t_apply = time.perf_counter() - t0
    return {"value": round(info["iterations"] / dt, 4), "unit": "iters/s", "cores": cores, "kind": "port",
            "sample": "rhs_p = M^-1 f + %d GMRES iterations (fixed-iteration mode) of the same workload, "
                      "oracle/ restatement on SuperLU/LAPACK/numpy, default BLAS threads" % info["iterations"],
            "seconds": round(dt, 2), "apply_s": round(t_apply, 3)}


def run_reference(args, dist):
    if dist.rank != 0:
        return None
    import paper_2406_06283_b200 as hg
    from oracle.schwarz_oracle import OraclePreconditioner
    from oracle.wgmres_oracle import weighted_gmres as oracle_gmres

    t0 = time.perf_counter()
    P = hg.build_problem(args.config, cstab=args.cstab, verbose=True)
    orc = OraclePreconditioner(P.forms, P.dec, P.coarse, b0_lu=getattr(P.coarse, "_b0_lu", None))
    log("reference-arm setup %.1f s" % (time.perf_counter() - t0))
    rhs = P.rhs if P.rhs.ndim == 2 else P.rhs[:, None]
    B, Dk = P.forms.helmholtz, P.forms.dk

    def step(s):
        f = rhs[:, s % rhs.shape[1]]
        x, info = oracle_gmres(lambda v: orc.apply(B @ v), orc.apply(f), weight=Dk, rtol=0.0, maxit=args.ref_iters)
        return info["iterations"]

    for s in range(args.warmup):
        step(s)
    t0 = time.perf_counter()
    it = 0
    for s in range(args.steps):
        it += step(args.warmup + s)
    dt = time.perf_counter() - t0
    value = it / dt
    cores = len(os.sched_getaffinity(0))
    return {
        "impl": "reference",
        "metric": "GMRES iters/s (FP64, two-level Schwarz + H_k-GenEO, D_k-weighted)",
        "value": round(value, 4),
        "unit": "iters/s",
        "n_gpus": dist.world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(dt / max(args.steps, 1) * 1e3, 2),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic, seeded",
        "config": {"workload": "BASELINE config %s (same as the ours arm)" % P.config.name,
                   "step": "rhs_p = M^-1 f + %d GMRES iterations, CPU oracle port" % args.ref_iters},
        "cpu_baseline": {"value": round(value, 4), "unit": "iters/s", "cores": cores, "kind": "port",
                         "sample": "%d GMRES iterations + 1 apply per step on the host cores" % args.ref_iters},
        "e2e": {"value": round(value, 4), "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    args = parse()
    if args.impl == "reference":
        dist = Dist("gloo")
        line = run_reference(args, dist)
    else:
        dist = Dist("nccl")
        line = run_ours(args, dist)
    if dist.rank == 0 and line is not None:
        print(json.dumps(line), flush=True)
    dist.close()


if __name__ == "__main__":
    main()
