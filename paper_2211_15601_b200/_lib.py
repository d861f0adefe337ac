"""ctypes binding of the C-ABI in ``include/fsk.h`` (``libfsk_b200.so``).

This is the Python-side equivalent of the FFI stub a maintainer would add to bind
the reference's deformer API. There is no fallback: if the
library or an sm_100 device is missing, every call raises.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# FSK_LIB: load a tuning-variant build instead (scripts/build_variants.sh); default in-tree.
LIB_PATH = os.environ.get("FSK_LIB") or os.path.join(HERE, "libfsk_b200.so")

FSK_OK, FSK_EINVAL, FSK_ECUDA, FSK_ENODEV, FSK_EIO = 0, 1, 2, 3, 4
FSK_SEARCH_NO_SORT = 0x1
FSK_SEARCH_FP32_ONLY = 0x2
FSK_SEARCH_FP64 = 0x4
FSK_SEARCH_EXACT64 = 0x8
FSK_SEARCH_FAST_ESC = 0x10

# Every symbol include/fsk.h declares (checked by tests/test_lib_exports.py).
EXPORTS = [
    "fsk_ctx_create", "fsk_ctx_destroy", "fsk_last_error", "fsk_ctx_launch_count", "fsk_device_sm_count",
    "fsk_search_opts_defaults", "fsk_precompute_tgrid", "fsk_search_fwd", "fsk_compact_roots",
    "fsk_deform_host", "fsk_deform_host_frames", "fsk_eval_points", "fsk_init_states", "fsk_search_bwd", "fsk_grad_weights",
    "fsk_ctx_set_profiling", "fsk_ctx_prof_read", "fsk_measure_fp32_peak", "fsk_batch_search", "fsk_deform",
    "fsk_deform_frames",
    "fsk_search_bwd_roots", "fsk_ctx_search_stats", "fsk_measure_fp64_peak", "fsk_measure_l1_gather_peak",
    "fsk_distill", "fsk_posed_occupancy", "fsk_distill_bwd",
    "fsk_multi_create", "fsk_multi_destroy", "fsk_multi_device_count", "fsk_multi_deform_host",
    "fsk_multi_grad_weights_host", "fsk_search_fwd_mlp",
    "fsk_io_last_error", "fsk_sknv_read", "fsk_sknv_write", "fsk_points_bin_read", "fsk_points_bin_write",
    "fsk_write_correspondence_dump", "fsk_deform_files", "fsk_init_states64",
    "fsk_implicit_u_exact", "fsk_search_bwd_exact_roots", "fsk_search_bwd_roots_ordered", "fsk_ctx_query_order",
    "fsk_measure_red_peak", "fsk_search_bwd_max_term", "fsk_search_bwd_fixed", "fsk_fixed_to_float",
]


class GridDesc(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nz", ctypes.c_int32),
                ("n_bones", ctypes.c_int32), ("bbox_min", ctypes.c_double * 3), ("bbox_max", ctypes.c_double * 3)]


class SearchOpts(ctypes.Structure):
    _fields_ = [("max_iters", ctypes.c_int32), ("flags", ctypes.c_int32), ("conv_eps", ctypes.c_double),
                ("div_eps", ctypes.c_double), ("dedup_dist", ctypes.c_double)]


class SearchOut(ctypes.Structure):
    _fields_ = [("x_c", ctypes.c_void_p), ("jinv", ctypes.c_void_p), ("resid", ctypes.c_void_p),
                ("iters", ctypes.c_void_p), ("converged", ctypes.c_void_p), ("keep", ctypes.c_void_p),
                ("n_roots", ctypes.c_void_p), ("x_c64", ctypes.c_void_p)]


class BwdSrc(ctypes.Structure):
    _fields_ = [("x_c", ctypes.c_void_p), ("jinv", ctypes.c_void_p), ("root_sel", ctypes.c_void_p),
                ("n_init", ctypes.c_int32), ("roots", ctypes.c_void_p), ("root_index", ctypes.c_void_p)]


class Root(ctypes.Structure):
    _fields_ = [("x", ctypes.c_float * 3), ("residual", ctypes.c_float), ("inv_jacobian", ctypes.c_float * 9),
                ("source_bone", ctypes.c_int32), ("iterations", ctypes.c_int32), ("_pad", ctypes.c_int32)]


assert ctypes.sizeof(Root) == 64

_vp, _i32, _i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
_lib = None


class FskError(RuntimeError):
    pass


class FskInvalidArgument(FskError, ValueError):
    """std::invalid_argument of the reference, surfaced through FSK_EINVAL."""


def load():
    """Load the in-tree library (raises if it was not built — no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise FskError(f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(LIB_PATH)
    L.fsk_last_error.restype = ctypes.c_char_p
    L.fsk_ctx_create.argtypes = [ctypes.c_int, ctypes.POINTER(_vp)]
    L.fsk_ctx_destroy.argtypes = [_vp]
    L.fsk_ctx_launch_count.argtypes = [_vp]
    L.fsk_ctx_launch_count.restype = _i64
    L.fsk_device_sm_count.argtypes = [_vp]
    L.fsk_search_opts_defaults.argtypes = [ctypes.POINTER(GridDesc)]
    L.fsk_search_opts_defaults.restype = SearchOpts
    G, O, S = ctypes.POINTER(GridDesc), ctypes.POINTER(SearchOpts), ctypes.POINTER(SearchOut)
    L.fsk_precompute_tgrid.argtypes = [_vp, _vp, G, _vp, _i32, _vp, _vp, _vp]
    L.fsk_search_fwd.argtypes = [_vp, _vp, _vp, _vp, G, _vp, _i32, _vp, _i64, O, S, _vp]
    L.fsk_compact_roots.argtypes = [_vp, S, _i64, _i32, _vp, _vp, _i64, ctypes.POINTER(_i64), _vp]
    L.fsk_deform_host.argtypes = [_vp, _vp, G, _vp, _i32, _vp, _i64, O, _vp, _vp, _i64, ctypes.POINTER(_i64), _vp]
    L.fsk_deform_host_frames.argtypes = [_vp, _vp, G, _i32, _vp, _i32, _vp, _vp, O, _vp, _vp, _vp, _vp, _vp]
    L.fsk_eval_points.argtypes = [_vp, _vp, G, _vp, _i64, _vp, _vp, _vp, _vp]
    L.fsk_init_states.argtypes = [_vp, _vp, G, _vp, _i32, _vp, _i64, _vp, _vp, _vp]
    L.fsk_init_states64.argtypes = [_vp, _vp, G, _vp, _i32, _vp, _i64, _vp, _vp, _vp]
    L.fsk_search_bwd.argtypes = [_vp, G, _vp, _vp, _i32, _vp, _vp, _i64, _vp, ctypes.c_int, _vp]
    L.fsk_grad_weights.argtypes = [_vp, G, _vp, _vp, _i32, _vp, _vp]
    L.fsk_implicit_u_exact.argtypes = [_vp, _vp, G, _vp, _i32, _vp, _vp, _i64, _vp, _vp, _vp, _vp]
    L.fsk_search_bwd_exact_roots.argtypes = [_vp, _vp, G, _vp, _i32, _vp, _vp, _vp, _i64, _vp, _vp, ctypes.c_int, _vp]
    L.fsk_batch_search.argtypes = [_vp, _vp, _vp, _vp, G, _vp, _i32, _vp, _i64, O, _vp, _vp, _i64, _vp]
    L.fsk_deform.argtypes = [_vp, _vp, G, _vp, _i32, _vp, _i64, O, _vp, _vp, _vp, _i64, _vp]
    L.fsk_deform_frames.argtypes = [_vp, _vp, G, _i32, _vp, _i32, _vp, _vp, O, _vp, _vp, _vp, _vp, _vp]
    L.fsk_search_bwd_roots.argtypes = [_vp, G, _vp, _vp, _vp, _i64, _vp, ctypes.c_int, _vp]
    L.fsk_search_bwd_roots_ordered.argtypes = [_vp, G, _vp, _vp, _vp, _i64, _vp, _vp, ctypes.c_int, _vp]
    L.fsk_ctx_query_order.argtypes = [_vp, _i64, _vp, _vp]
    L.fsk_measure_red_peak.argtypes = [_vp, ctypes.POINTER(ctypes.c_double)]
    BS = ctypes.POINTER(BwdSrc)
    L.fsk_search_bwd_max_term.argtypes = [_vp, G, BS, _vp, _i64, _vp, _vp]
    L.fsk_search_bwd_fixed.argtypes = [_vp, G, BS, _vp, _i64, _i64, _vp, _vp, _vp]
    L.fsk_fixed_to_float.argtypes = [_vp, _vp, _i64, _i64, _vp, _vp, _vp]
    L.fsk_ctx_set_profiling.argtypes = [_vp, ctypes.c_int]
    L.fsk_ctx_prof_read.argtypes = [_vp, ctypes.c_char_p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_i64),
                                    ctypes.c_int]
    L.fsk_ctx_search_stats.argtypes = [_vp, ctypes.POINTER(ctypes.c_uint64), ctypes.c_int]
    L.fsk_measure_fp32_peak.argtypes = [_vp, ctypes.POINTER(ctypes.c_double)]
    L.fsk_measure_fp64_peak.argtypes = [_vp, ctypes.POINTER(ctypes.c_double)]
    L.fsk_measure_l1_gather_peak.argtypes = [_vp, ctypes.POINTER(ctypes.c_double)]
    L.fsk_distill.argtypes = [_vp, _vp, _vp, _i32, G, _vp, _vp]
    L.fsk_distill_bwd.argtypes = [_vp, _vp, _vp, _i32, G, _vp, _vp, _vp]
    L.fsk_search_fwd_mlp.argtypes = [_vp, _vp, _vp, _i32, _vp, _i32, _vp, _i64, O, S, _vp]
    _cp = ctypes.c_char_p
    L.fsk_io_last_error.restype = _cp
    L.fsk_sknv_read.argtypes = [_cp, G, _vp, _i64]
    L.fsk_sknv_write.argtypes = [_cp, G, _vp]
    L.fsk_points_bin_read.argtypes = [_cp, _vp, _i64, ctypes.POINTER(_i64)]
    L.fsk_points_bin_write.argtypes = [_cp, _vp, _i64]
    L.fsk_write_correspondence_dump.argtypes = [_cp, _vp, _i64, _vp, _vp, _i32]
    L.fsk_deform_files.argtypes = [_vp, _cp, _vp, _i32, _cp, O, _cp, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]
    L.fsk_multi_create.argtypes = [_i32, _vp, ctypes.POINTER(_vp)]
    L.fsk_multi_destroy.argtypes = [_vp]
    L.fsk_multi_device_count.argtypes = [_vp]
    L.fsk_multi_device_count.restype = _i32
    L.fsk_multi_deform_host.argtypes = [_vp, _vp, G, _vp, _i32, _vp, _i64, O, _vp, _vp, _i64, ctypes.POINTER(_i64)]
    L.fsk_multi_grad_weights_host.argtypes = [_vp, G, _vp, _i32, _vp, _vp, _vp, _i64, _vp, ctypes.c_int]
    L.fsk_posed_occupancy.argtypes = [_vp, _vp, _vp, _i32, _vp, _i32, _vp, _vp, _i64, _i64, _vp, _vp, _vp, _vp]
    _lib = L
    return L


def check(rc: int) -> None:
    if rc != FSK_OK:
        msg = load().fsk_last_error().decode()
        raise (FskInvalidArgument if rc == FSK_EINVAL else FskError)(msg)
