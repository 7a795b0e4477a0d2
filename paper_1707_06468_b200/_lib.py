"""ctypes binding of ``libproxsaga.so`` (the C ABI declared in include/proxsaga.h).

The library is built in-tree (``__graft_entry__.build()`` /
``make -C paper_1707_06468_b200/csrc``).  There is no fallback: if the
library or a CUDA device is missing, every solver entry point raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libproxsaga.so"
# A/B experiments: PROXSAGA_LIB points at another build of the same ABI
if os.environ.get("PROXSAGA_LIB"):
    LIB_PATH = Path(os.environ["PROXSAGA_LIB"])

PS_OK, PS_EINVAL, PS_ERANGE, PS_ECUDA, PS_ENOMEM = 0, 1, 2, 3, 4
LOSS = {"logistic": 0, "squared": 1}
PEN_ZERO, PEN_L1, PEN_GROUP, PEN_BOX = 0, 1, 2, 3
F32, F64 = 0, 1
I32, I64 = 0, 1
PART_SINGLETON, PART_CONTIG, PART_GENERAL = 0, 1, 2
# ps_sched_t.flags (include/proxsaga.h PS_FLAG_*)
FLAG_SCRAMBLE, FLAG_GENERIC, FLAG_DELTA_ZERO, FLAG_GROUP_WARP, FLAG_GROUP_LANE = 4, 16, 32, 64, 128
FLAG_MON_ENDS_IN_PLACE, FLAG_ZERO_IMMEDIATE, FLAG_GROUP_STORE_ZEROS = 65536, 131072, 262144
FLAG_NO_CLUSTER, FLAG_FAST_V1 = 2097152, 4194304
FLAG_MON_DEVICE_X = 524288
FLAG_LOCAL_VIEW = 134217728
ABI_VERSION = 3

# Every symbol include/proxsaga.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "ps_abi_version", "ps_last_error", "ps_device_count", "ps_prepare", "ps_scratch_bytes",
    "ps_launch_config", "ps_run", "ps_objective", "ps_smooth_gradient", "ps_fixed_point_residual",
    "ps_resync_average", "ps_prox", "ps_state_reset", "ps_hot_layout", "ps_coord_get", "ps_coord_set",
    "ps_coord_get_perm", "ps_coord_set_perm", "ps_atomic_gather",
    "ps_atomic_scatter_add", "ps_atomic_exchange", "ps_atomic_fetch_add_i64",
    "ps_atomic_add_repeat", "ps_gen_zipf_csr", "ps_gen_labels", "ps_timestamp",
    "ps_dual_objective", "ps_run_monitored", "ps_libsvm_index", "ps_libsvm_scan", "ps_libsvm_fill",
    "ps_fista_prox", "ps_fista_extrapolate", "ps_loss_deriv", "ps_loss_eval", "ps_batch_run", "ps_batch_run_rep", "ps_batch_field", "ps_batch_tune", "ps_batch_tune2", "ps_batch_last_grid", "ps_batch_state_doubles",
    "ps_batch_rep_doubles",
)

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_f64 = ctypes.c_double


class Csr(ctypes.Structure):
    _fields_ = [("n_rows", _i64), ("n_cols", _i64), ("nnz", _i64), ("row_ptr", _vp),
                ("col_idx", _vp), ("values", _vp), ("labels", _vp), ("row_ptr_type", _i32),
                ("value_type", _i32)]


class Part(ctypes.Structure):
    _fields_ = [("kind", _i32), ("G", _i32), ("n_blocks", _i64), ("block_of", _vp),
                ("blk_ptr", _vp), ("blk_coords", _vp), ("blk_count", _vp), ("blk_weight", _vp),
                ("row_blk", _vp), ("row_g", _vp), ("spos", _vp), ("max_slots", _i32), ("max_row_nnz", _i32)]


class Params(ctypes.Structure):
    _fields_ = [("loss", _i32), ("penalty", _i32), ("lambda1", _f64), ("lam2", _f64),
                ("lo", _f64), ("hi", _f64), ("gamma", _f64)]


class Stats(ctypes.Structure):
    _fields_ = [("max_count", _i64), ("n_dead", _i64), ("max_row_sqnorm", _f64),
                ("max_row_nnz", _i32), ("max_slots", _i32)]


class Sched(ctypes.Structure):
    _fields_ = [("samples", _vp), ("count", _i64), ("seed", ctypes.c_uint64),
                ("slot_base", ctypes.c_uint64), ("counter", _vp), ("batch", _i32),
                ("ctas", _i32), ("warps_per_cta", _i32), ("hot_cols", _i32), ("contention", _f64),
                ("hot_period", _i32), ("flags", _i32), ("hot_shift", _i32), ("reserved", _i32),
                ("trace_v", _vp), ("trace_dx", _vp)]


_P = ctypes.POINTER
_lib = None


class LibraryMissing(RuntimeError):
    pass


def load():
    """Load libproxsaga.so (raises LibraryMissing if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise LibraryMissing(f"{LIB_PATH} is not built; run __graft_entry__.build()")
    L = ctypes.CDLL(str(LIB_PATH))
    sig = {
        "ps_abi_version": (_i32, []),
        "ps_last_error": (ctypes.c_char_p, []),
        "ps_device_count": (_i32, []),
        "ps_prepare": (_i32, [_P(Csr), _P(Part), _vp, _P(Stats), _vp]),
        "ps_scratch_bytes": (_i64, [_P(Csr), _P(Part), _i32]),
        "ps_launch_config": (_i32, [_P(Csr), _P(Part), _P(Sched), _P(_i32), _P(_i32), _P(_i64)]),
        "ps_run": (_i32, [_P(Csr), _P(Part), _P(Params), _vp, _vp, _P(Sched), _vp, _vp]),
        "ps_objective": (_i32, [_P(Csr), _P(Part), _P(Params), _vp, _i32, _vp, _vp]),
        "ps_smooth_gradient": (_i32, [_P(Csr), _P(Params), _vp, _i32, _vp, _vp]),
        "ps_fixed_point_residual": (_i32, [_P(Csr), _P(Part), _P(Params), _vp, _vp, _vp, _vp]),
        "ps_resync_average": (_i32, [_P(Csr), _vp, _vp, _vp]),
        "ps_prox": (_i32, [_P(Params), _vp, _vp, _i64, _vp, _vp]),
        "ps_state_reset": (_i32, [_vp, _i64, _vp, _i64, _vp, _vp]),
        "ps_timestamp": (_i32, [_vp, _vp]),
        "ps_dual_objective": (_i32, [_P(Csr), _P(Part), _P(Params), _vp, _i32, _vp, _vp]),
        "ps_libsvm_index": (_i32, [_vp, _i64, _vp, _i64, _vp]),
        "ps_fista_prox": (_i32, [_P(Part), _P(Params), _vp, _vp, ctypes.c_double, _i64, _vp, _vp, _vp]),
        "ps_fista_extrapolate": (_i32, [_vp, _vp, ctypes.c_double, _i64, _vp, _vp]),
        "ps_loss_deriv": (_i32, [_i32, _i32, _vp, _vp, _i64, _vp, _vp]),
        "ps_loss_eval": (_i32, [_i32, _vp, _vp, _i64, _vp, _vp, _vp]),
        "ps_batch_run": (_i32, [_P(Csr), _P(Part), _P(Params), _vp, _i32, _vp, _vp, _P(Sched), _vp]),
        "ps_batch_run_rep": (_i32, [_P(Csr), _P(Part), _P(Params), _vp, _i32, _vp, _vp, _P(Sched), _vp, _i32, _i32, _vp]),
        "ps_batch_field": (_i32, [_vp, _i64, _i32, _i32, _i32, _i32, _i32, _vp, _i32, _vp]),
        "ps_batch_tune": (_i32, [_i64, _i64]),
        "ps_batch_tune2": (_i32, [_i32, _i64, _i32, _i32]),
        "ps_batch_last_grid": (_i32, [_P(_i32), _P(_i32)]),
        "ps_batch_state_doubles": (_i64, [_i64, _i32, _i32]),
        "ps_batch_rep_doubles": (_i64, [_i32, _i32, _i32, _i32]),
        "ps_libsvm_scan": (_i32, [_vp, _i64, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
        "ps_libsvm_fill": (_i32, [_vp, _i64, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
        "ps_run_monitored": (_i32, [_P(Csr), _P(Part), _P(Params), _vp, _vp, _P(Sched), _vp, _vp, _i64, _i32,
                                    _vp, _P(_i64), _P(ctypes.c_float), _P(_i32)]),
        "ps_hot_layout": (_i32, [_P(Csr), _vp, _vp, _i32, _i32, _f64, _P(_i32), _vp, _vp, _P(_i32), _P(_i64),
                                 _vp]),
        "ps_coord_get_perm": (_i32, [_vp, _i64, _i32, _vp, _vp, _vp]),
        "ps_coord_set_perm": (_i32, [_vp, _i64, _i32, _vp, _vp, _vp]),
        "ps_coord_get": (_i32, [_vp, _i64, _i32, _vp, _vp]),
        "ps_coord_set": (_i32, [_vp, _i64, _i32, _vp, _vp]),
        "ps_atomic_gather": (_i32, [_vp, _i64, _vp, _i64, _vp, _vp]),
        "ps_atomic_scatter_add": (_i32, [_vp, _i64, _vp, _i64, _vp, _vp]),
        "ps_atomic_exchange": (_i32, [_vp, _i64, _vp, _i64, _vp, _vp, _vp]),
        "ps_atomic_fetch_add_i64": (_i32, [_vp, _i64, _i64, _i64, _vp, _vp]),
        "ps_atomic_add_repeat": (_i32, [_vp, _f64, _i64, _i32, _vp]),
        "ps_gen_zipf_csr": (_i32, [_i64, _i32, _i32, _vp, _i64, ctypes.c_uint64, _i32, _vp, _vp, _vp, _vp]),
        "ps_gen_labels": (_i32, [_i64, _i32, _vp, _vp, _vp, _f64, ctypes.c_uint64, _vp, _vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    if L.ps_abi_version() != ABI_VERSION:
        raise LibraryMissing(f"{LIB_PATH} has ABI {L.ps_abi_version()}, this package needs {ABI_VERSION}: rebuild it")
    _lib = L
    return L


def check(status):
    """Map a ps_status to the reference's exception conventions."""
    if status == PS_OK:
        return
    msg = load().ps_last_error().decode(errors="replace")
    if status == PS_EINVAL:
        raise ValueError(msg)
    if status == PS_ERANGE:
        raise IndexError(msg)
    if status == PS_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def require_device():
    """Fail loudly when no CUDA device is usable: the product has no CPU path."""
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_1707_06468_b200 needs a CUDA device (sm_100a); no CPU fallback exists")
    load()


def stream_ptr(stream=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)
