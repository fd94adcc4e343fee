"""ctypes binding of libhelmgpu.so (include/helmgpu.h).

The shared library is built in-tree (``paper_2406_06283_b200/libhelmgpu.so``,
see csrc/Makefile).  There is no fallback: if the library is missing or no
CUDA device is present, the first call raises.
"""

import atexit
import ctypes
import os

from .errors import DeviceError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libhelmgpu.so")

_i32p = ctypes.POINTER(ctypes.c_int32)
_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)
_vp = ctypes.c_void_p


class HgPrecondDesc(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int32),
        ("nnz", ctypes.c_int64),
        ("indptr", _i32p),
        ("indices", _i32p),
        ("b_data", _f64p),
        ("dk_data", _f64p),
        ("n_local", ctypes.c_int32),
        ("local_n", _i32p),
        ("local_kl", _i32p),
        ("local_kv", _i32p),
        ("local_fstride", _i32p),
        ("local_bstride", _i32p),
        ("local_idx_off", _i64p),
        ("local_idx", _i32p),
        ("local_fwd_off", _i64p),
        ("local_fwd_len", ctypes.c_int64),
        ("local_fwd", _f64p),
        ("local_bwd_off", _i64p),
        ("local_bwd_len", ctypes.c_int64),
        ("local_bwd", _f64p),
        ("m", ctypes.c_int32),
        ("n_cblk", ctypes.c_int32),
        ("cblk_n", _i32p),
        ("cblk_m", _i32p),
        ("cblk_idx_off", _i64p),
        ("cblk_idx", _i32p),
        ("cblk_z_off", _i64p),
        ("z_len", ctypes.c_int64),
        ("z_data", _f64p),
        ("b0_perm", _i32p),
        ("b0_panel", ctypes.c_int32),
        ("b0_npanel", ctypes.c_int32),
        ("b0_dinv", _f64p),
        ("b0_tile_ptr", _i64p),
        ("b0_tile_col", _i32p),
        ("b0_ntile", ctypes.c_int64),
        ("b0_tiles", _f64p),
        ("b0_ctas", ctypes.c_int32),
        ("b0_mode", ctypes.c_int32),
        ("b0_cluster", ctypes.c_int32),
        ("b0_ring", ctypes.c_int32),
        ("b0_inv", _f64p),
        ("local_bw", _i32p),
        ("lcsr_indptr", _i64p),
        ("lcsr_cols", _i32p),
        ("lcsr_vals", _f64p),
        ("lcsr_nnz", ctypes.c_int64),
        ("factor_info", _i32p),
        ("factor_min_pivot", _f64p),
        ("b0_inv_batched_only", ctypes.c_int32),
        ("n_split", ctypes.c_int32),
        ("split_blk", _i32p),
        ("split_row_off", _i64p),
        ("split_f_indptr", _i64p),
        ("split_f_pos", _i64p),
        ("split_f_val", _f64p),
        ("split_sinv_off", _i64p),
        ("split_sinv_len", ctypes.c_int64),
        ("split_sinv", _f64p),
        ("n_spike", ctypes.c_int32),
        ("spike_blk", _i32p),
        ("spike_split", _i32p),
        ("spike_col0", _i32p),
        ("spike_w", _i32p),
        ("spike_off", _i64p),
        ("spike_len", ctypes.c_int64),
        ("spike_data", _f64p),
        ("b0_split", ctypes.c_int32),
        ("b0s_a", ctypes.c_int32),
        ("b0s_ns", ctypes.c_int32),
        ("b0s_wl", ctypes.c_int32),
        ("b0s_wr", ctypes.c_int32),
        ("b0h0_npanel", ctypes.c_int32),
        ("b0h0_ring", ctypes.c_int32),
        ("b0h0_cluster", ctypes.c_int32),
        ("b0h0_ntile", ctypes.c_int64),
        ("b0h0_perm", _i32p),
        ("b0h0_dinv", _f64p),
        ("b0h0_tile_ptr", _i64p),
        ("b0h0_tile_col", _i32p),
        ("b0h0_tiles", _f64p),
        ("b0h1_npanel", ctypes.c_int32),
        ("b0h1_ring", ctypes.c_int32),
        ("b0h1_cluster", ctypes.c_int32),
        ("b0h1_ntile", ctypes.c_int64),
        ("b0h1_perm", _i32p),
        ("b0h1_dinv", _f64p),
        ("b0h1_tile_ptr", _i64p),
        ("b0h1_tile_col", _i32p),
        ("b0h1_tiles", _f64p),
        ("b0s_f", _f64p),
        ("b0s_sinv", _f64p),
        ("b0s_w", _f64p),
    ]


# name -> (restype, argtypes); every symbol include/helmgpu.h declares
SIGNATURES = {
    "hg_abi_version": (ctypes.c_int, []),
    "hg_last_error": (ctypes.c_char_p, []),
    "hg_kernel_launches": (ctypes.c_int64, []),
    "hg_device_sync": (ctypes.c_int, []),
    "hg_shutdown": (ctypes.c_int, []),
    "hg_precond_create": (ctypes.c_int, [ctypes.POINTER(HgPrecondDesc), ctypes.POINTER(_vp)]),
    "hg_precond_destroy": (ctypes.c_int, [_vp]),
    "hg_precond_device_bytes": (ctypes.c_int64, [_vp]),
    "hg_precond_apply": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "hg_precond_apply_T": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "hg_precond_apply_coarse": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "hg_precond_spmv": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp, _vp]),
    "hg_precond_profile": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int32, _f64p, _vp]),
    "hg_local_solve": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp, _vp]),
    "hg_precond_local_solutions": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "hg_op_create_csr": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int64, _i32p, _i32p, _f64p, ctypes.POINTER(_vp)]),
    "hg_op_create_precond": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.POINTER(_vp)]),
    "hg_op_destroy": (ctypes.c_int, [_vp]),
    "hg_op_apply": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "hg_gmres": (
        ctypes.c_int,
        [_vp, _vp, _vp, _vp, _vp, ctypes.c_double, ctypes.c_int32, _f64p, _i32p, _vp],
    ),
    "hg_solve_host": (
        ctypes.c_int,
        [_vp, _f64p, _f64p, ctypes.c_double, ctypes.c_int32, _f64p, _i32p, _vp],
    ),
    "hg_precond_apply_multi": (ctypes.c_int, [_vp, _vp, ctypes.c_int64, _vp, ctypes.c_int64, ctypes.c_int32, _vp]),
    "hg_precond_profile_multi": (
        ctypes.c_int,
        [_vp, _vp, ctypes.c_int64, _vp, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, _f64p, _vp],
    ),
    "hg_op_apply_multi": (ctypes.c_int, [_vp, _vp, ctypes.c_int64, _vp, ctypes.c_int64, ctypes.c_int32, _vp]),
    "hg_gmres_batch": (
        ctypes.c_int,
        [_vp, _vp, _vp, ctypes.c_int64, _vp, ctypes.c_int64, ctypes.c_int32, ctypes.c_double, ctypes.c_int32,
         _f64p, _i32p, _vp],
    ),
    "hg_solve_host_batch": (
        ctypes.c_int,
        [_vp, _f64p, _f64p, ctypes.c_int32, ctypes.c_double, ctypes.c_int32, _f64p, _i32p, _vp],
    ),
    "hg_stats_enable": (ctypes.c_int, [ctypes.c_int]),
    "hg_op_basis": (ctypes.c_int, [_vp, ctypes.c_int32, ctypes.c_int32, _vp, _vp]),
    "hg_set_orthogonalization": (ctypes.c_int, [ctypes.c_int]),
    "hg_get_orthogonalization": (ctypes.c_int, []),
    "hg_stats_read": (ctypes.c_int, [_f64p, _i64p, ctypes.c_int]),
    "hg_precond_status": (ctypes.c_int, [_vp]),
    "hg_op_release": (ctypes.c_int, [_vp]),
    "hg_dcgs2_explicit_passes": (ctypes.c_int64, []),
    "hg_debug_set": (ctypes.c_int, [_vp, ctypes.c_int32, ctypes.c_int64]),
    "hg_precond_read": (ctypes.c_int, [_vp, ctypes.c_int32, _f64p, ctypes.c_int64]),
    "hg_precond_stat": (ctypes.c_double, [_vp, ctypes.c_int32]),
    "hg_precond_coarse_solve": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "hg_coarse_setup": (
        ctypes.c_int,
        [ctypes.POINTER(HgPrecondDesc), _i32p, _i32p, _f64p, _f64p, _i32p, _i32p, _f64p, ctypes.c_int32],
    ),
}
STAT_PANEL_ACTIVE, STAT_PANEL_DEVIATION, STAT_PANEL_BYTES = 1, 2, 3
FIELD_LOCAL_FWD, FIELD_LOCAL_BWD = 1, 2

ABI_VERSION = 5
DEBUG_SPIN_LIMIT_MS, DEBUG_SKIP_ZT, DEBUG_FORCE_EXPLICIT_RHO, DEBUG_B0_SPLIT, DEBUG_LOCAL_STAGES = 1, 2, 3, 4, 5
DEBUG_B0_TILE_STAGES = 6
MAX_BASIS = 1024  # Krylov vectors the basis kernels support (MAX_NV)
NPHASES = 7  # HG_NPHASES
ORTH = {"measured": 0, "dcgs2": 1}
PHASES = ("op_apply", "proj_dots", "cgs_update", "measure", "second_pass", "append", "w_spmv")
MAX_RHS = 16

_LIB = None


def load(path=LIB_PATH):
    """Load the library and bind every exported symbol (raises if absent)."""
    global _LIB
    if _LIB is not None and path == LIB_PATH:
        return _LIB
    if not os.path.exists(path):
        raise ImportError(
            "libhelmgpu.so not built (%s); run `make -C paper_2406_06283_b200/csrc` "
            "or __graft_entry__.build() — there is no CPU fallback" % path
        )
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.hg_abi_version() != ABI_VERSION:
        raise ImportError("libhelmgpu.so ABI mismatch")
    if path == LIB_PATH:
        _LIB = lib
        atexit.register(lib.hg_shutdown)
    return lib


def check(status, what=""):
    if status != 0:
        msg = load().hg_last_error().decode(errors="replace")
        raise DeviceError("%s failed (status %d): %s" % (what or "helmgpu call", status, msg))


def ptr(arr, ctype):
    """ctypes pointer into a numpy array (None for None / empty)."""
    if arr is None:
        return None
    return arr.ctypes.data_as(ctypes.POINTER(ctype))
