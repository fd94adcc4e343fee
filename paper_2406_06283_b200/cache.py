"""On-disk setup cache (the reference has no
checkpointing).

The unit cached is the *device image* of a preconditioner: every array
hg_precond_create consumes (include/helmgpu.h HgPrecondDesc) — the global
CSR of B and D_k, per-block band-LU records with their pivots, idof lists,
the dense Z blocks and index sets, the B0 permutation, inverse diagonal
blocks and tiles — plus the scalars and the Python-side metadata
(TwoLevelPreconditioner._image).  Loading it feeds hg_precond_create
directly: no mesh, assembly, eigensolves or factorisations run, and the
handle is bitwise the one the fresh setup would build.

Format (version CACHE_VERSION): a directory with one uncompressed ``.npy``
per array (memory-mapped on load) and ``meta.json`` (written last: a
directory without it is incomplete and ignored).  Entries are keyed by a
hash of everything that determines the image: the problem configuration,
the C_stab it was built with, the coarse-solve knobs (HG_B0_MODE / PANEL /
DENSE / CTAS), the ABI version and this package's setup version.

Problem-level entries (``solver_for_config``) add the right-hand sides and
the setup phase times, so a driver can go straight to the solve.
"""

import hashlib
import json
import os
import shutil
import time
import types
from dataclasses import asdict

import numpy as np
import scipy.sparse as sp

CACHE_VERSION = 1
SETUP_VERSION = "r2c"  # bump when the host setup restatement changes its outputs
KNOBS = ("HG_B0_MODE", "HG_B0_PANEL", "HG_B0_DENSE", "HG_B0_CTAS", "HG_LOCAL_SPLIT", "HG_B0_SPLIT", "HG_B0_SPLIT_CS")


def default_dir():
    return os.environ.get("HG_CACHE_DIR", os.path.join(os.path.expanduser("~"), ".cache", "helmgpu"))


def image_key(config, cstab):
    """Hash of everything that determines a config's device image."""
    from . import _lib

    cfg = asdict(config) if hasattr(config, "__dataclass_fields__") else dict(config)
    blob = json.dumps({"config": cfg, "cstab": float(cstab), "knobs": {k: os.environ.get(k) for k in KNOBS},
                       "abi": _lib.ABI_VERSION, "setup": SETUP_VERSION, "cache": CACHE_VERSION},
                      sort_keys=True, default=str)
    return hashlib.sha256(blob.encode()).hexdigest()[:24]


def save_image(path, arrays, meta, extra_arrays=None):
    """Write an image directory (meta.json last, via rename: atomic)."""
    tmp = path + ".tmp%d" % os.getpid()
    shutil.rmtree(tmp, ignore_errors=True)
    os.makedirs(tmp)
    names = {}
    for group, arrs in (("desc", arrays), ("extra", extra_arrays or {})):
        for name, a in arrs.items():
            np.save(os.path.join(tmp, "%s.%s.npy" % (group, name)), np.ascontiguousarray(a))
            names.setdefault(group, []).append(name)
    m = dict(meta)
    m["_cache_version"] = CACHE_VERSION
    m["_arrays"] = names
    with open(os.path.join(tmp, "meta.json"), "w") as fh:
        json.dump(m, fh, default=_json_default)
    if os.path.exists(path):
        shutil.rmtree(path)
    os.rename(tmp, path)
    return path


def _json_default(o):
    if isinstance(o, (np.integer,)):
        return int(o)
    if isinstance(o, (np.floating,)):
        return float(o)
    raise TypeError(type(o))


def load_image(path, mmap=True):
    """(desc arrays, meta, extra arrays) of an image directory, or None if
    it is absent, incomplete or of another cache version."""
    mpath = os.path.join(path, "meta.json")
    if not os.path.exists(mpath):
        return None
    with open(mpath) as fh:
        meta = json.load(fh)
    if meta.get("_cache_version") != CACHE_VERSION:
        return None
    out = {}
    for group in ("desc", "extra"):
        out[group] = {name: np.load(os.path.join(path, "%s.%s.npy" % (group, name)), mmap_mode="r" if mmap else None)
                      for name in meta["_arrays"].get(group, [])}
    return out["desc"], meta, out["extra"]


def forms_from_image(arrays, meta):
    """Light stand-in for AssembledForms (helmholtz, dk, n_dofs, k) from the
    image's global CSR (B and D_k share the pattern)."""
    n = int(meta["n"])
    ip = np.asarray(arrays["indptr"], dtype=np.int32)
    ix = np.asarray(arrays["indices"], dtype=np.int32)
    B = sp.csr_matrix((np.asarray(arrays["b_data"]), ix, ip), shape=(n, n))
    Dk = sp.csr_matrix((np.asarray(arrays["dk_data"]), ix, ip), shape=(n, n)) if "dk_data" in arrays else None
    return types.SimpleNamespace(helmholtz=B, dk=Dk, n_dofs=n, k=meta.get("k"))


def save_preconditioner(pre, path, extra_arrays=None, extra_meta=None):
    """Cache a TwoLevelPreconditioner (it keeps its image when built with
    keep_image=True, see factorize)."""
    if getattr(pre, "_image_arrays", None) is None:
        raise ValueError("preconditioner was built without keep_image=True; nothing to cache")
    meta = dict(pre._meta)
    meta.update(extra_meta or {})
    return save_image(path, pre._image_arrays, meta, extra_arrays)


def factorize_from_cache(path, forms=None):
    """TwoLevelPreconditioner straight from a cached image (hg_precond_create
    on the stored arrays).  Raises FileNotFoundError if there is no valid
    entry at ``path``."""
    from .schwarz import TwoLevelPreconditioner

    got = load_image(path)
    if got is None:
        raise FileNotFoundError("no setup cache entry at %s" % path)
    arrays, meta, _ = got
    return TwoLevelPreconditioner.from_image(arrays, meta, forms)


def solver_for_config(name, cache_dir=None, cstab="cache", verbose=False, workers=None):
    """(preconditioner, problem view, info) for a BASELINE configuration, from
    the cache when a valid entry exists, else built (setup + factorize) and
    written.  The problem view has ``config``, ``forms``, ``rhs``, ``times``;
    ``info`` = {"hit": bool, "seconds": ..., "path": ...}."""
    from . import problems
    from .schwarz import TwoLevelPreconditioner, factorize

    cfg = problems.CONFIGS[name] if isinstance(name, str) else name
    cval = problems.cached_cstab(cfg) if cstab == "cache" else None
    root = cache_dir or default_dir()
    t0 = time.perf_counter()
    if cval is not None:
        path = os.path.join(root, "%s-%s" % (cfg.name, image_key(cfg, cval)))
        got = load_image(path)
        if got is not None:
            arrays, meta, extra = got
            pre = TwoLevelPreconditioner.from_image(arrays, meta)
            view = types.SimpleNamespace(config=cfg, forms=pre.forms, rhs=np.asarray(extra["rhs"]),
                                         times=dict(meta.get("setup_times", {})), cstab=cval, dec=None, coarse=None)
            return pre, view, {"hit": True, "seconds": time.perf_counter() - t0, "path": path}
    P = problems.build_problem(cfg, cstab=cstab, verbose=verbose, workers=workers)
    t1 = time.perf_counter()
    pre = factorize(P.forms, P.dec, P.coarse, keep_image=True)
    times = dict(P.times)
    times["factorize_upload"] = time.perf_counter() - t1
    path = os.path.join(root, "%s-%s" % (cfg.name, image_key(cfg, P.cstab)))
    os.makedirs(root, exist_ok=True)
    save_preconditioner(pre, path, extra_arrays={"rhs": P.rhs}, extra_meta={"setup_times": times, "k": cfg.k})
    P.times = times
    return pre, P, {"hit": False, "seconds": time.perf_counter() - t0, "path": path}
