"""ctypes binding of libfieldmap.so (the C ABI declared in include/fieldmap.h).

The library is the only compute path: there is no CPU fallback.  Importing
this module on a machine without the built library raises immediately with
the build command; calling into it without a CUDA device raises from the
first CUDA launch (FM_ERR_CUDA).
"""

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FM_LIB_PATH") or os.path.join(_PKG, "_lib", "libfieldmap.so")

FM_OK = 0
FM_ERR_ARG = -1
FM_ERR_CUDA = -2
FM_ERR_UNSUPPORTED = -3
FM_ERR_WORKSPACE = -4
FM_MAX_DIM = 5
FM_NBUCKETS = 9
FM_BUCKET_EDGES = (8, 16, 24, 32, 48, 64, 96, 128, 2147483647)

c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_f64 = ctypes.c_double
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p
c_sz = ctypes.c_size_t


class FmGrid(ctypes.Structure):
    _fields_ = [("dim", c_i32), ("reserved", c_i32), ("n", c_i64 * FM_MAX_DIM),
                ("lo", c_dbl * FM_MAX_DIM), ("inv_d", c_dbl * FM_MAX_DIM), ("ncell", c_i64)]


class FmSelect(ctypes.Structure):
    _fields_ = [("adaptive", c_i32), ("min_pts", c_i32), ("r_c", c_dbl), ("r0", c_dbl),
                ("growth", c_dbl), ("r_max", c_dbl)]


class FmRbf(ctypes.Structure):
    _fields_ = [("kind", c_i32), ("reserved", c_i32), ("a", c_dbl)]


class FmFit(ctypes.Structure):
    _fields_ = [("dim", c_i32), ("degree", c_i32), ("lam", c_dbl), ("centering", c_i32),
                ("reserved", c_i32)]


class FmLists(ctypes.Structure):
    _fields_ = [("counts", c_vp), ("slot_id", c_vp), ("slot_pos", c_vp), ("slot_cap", c_i32),
                ("n_overflow", c_i32), ("overflow", c_vp), ("pos_info", c_vp),
                ("pos_targets", c_vp), ("bucket_list", c_vp), ("bucket_stride", c_i64),
                ("bucket_count", c_i32 * FM_NBUCKETS), ("bucket_count_dev", c_vp),
                ("bucket_mask", c_i32), ("skip_overflow", c_i32)]


P = ctypes.POINTER
# name -> (restype, argtypes); mirrors include/fieldmap.h and fieldmap_patch.h
SIGNATURES = {
    "fm_version": (c_i32, []),
    "fm_error_string": (ctypes.c_char_p, [c_i32]),
    "fm_n_monomials": (c_i32, [c_i32, c_i32]),
    "fm_grid_workspace": (c_sz, [c_i64, c_i64]),
    "fm_grid_build": (c_i32, [P(FmGrid), c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp]),
    "fm_bbox": (c_i32, [c_i32, c_vp, c_i64, c_vp, c_vp]),
    "fm_bbox_pair": (c_i32, [c_i32, c_vp, c_i64, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "fm_bbox_pair_async": (c_i32, [c_i32, c_vp, c_i64, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "fm_bbox_decode": (c_i32, [c_i32, c_vp, c_vp]),
    "fm_grid_geometry": (c_i32, [c_i32, c_vp, c_vp, c_i64, c_dbl, P(FmGrid), c_vp, c_vp]),
    "fm_order_workspace": (c_sz, [c_i64, P(FmGrid)]),
    "fm_target_order": (c_i32, [P(FmGrid), c_vp, c_i64, c_vp, c_vp, c_sz, c_vp]),
    "fm_order_workspace_blocked": (c_sz, [c_i64, P(FmGrid), c_i32]),
    "fm_target_order_blocked": (c_i32, [P(FmGrid), c_vp, c_i64, c_i32, c_vp, c_vp, c_sz, c_vp]),
    "fm_bucket_positions": (c_i32, [c_vp, c_vp, c_i64, c_i64, c_i32, c_vp, c_i64, c_vp, c_vp]),
    "fm_support_count": (c_i32, [P(FmGrid), c_vp, c_vp, c_vp, c_i64, c_vp, P(FmSelect), c_i32,
                                 c_vp, c_vp, c_vp, c_vp, c_vp]),
    "fm_scan_workspace": (c_sz, [c_i64]),
    "fm_offsets_from_counts": (c_i32, [c_vp, c_i64, c_vp, c_vp, c_sz, c_vp]),
    "fm_support_fill": (c_i32, [P(FmGrid), c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, P(FmSelect),
                                c_vp, c_vp, c_i32, c_vp, c_vp, P(FmRbf), c_vp, c_vp]),
    "fm_rbf_weights": (c_i32, [c_i32, c_dbl, c_dbl, c_vp, c_i64, c_vp, c_vp]),
    "fm_scale_points": (c_i32, [c_vp, c_i64, c_i32, c_vp, c_vp, c_vp]),
    "fm_fit_many": (c_i32, [P(FmFit), c_vp, c_i64, c_vp, c_vp, c_vp, c_i32, c_vp, c_vp, c_vp,
                            c_vp, c_vp, c_vp, c_vp]),
    "fm_select_supports": (c_i32, [P(FmGrid), c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, P(FmSelect),
                                   c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_vp, c_vp, c_vp,
                                   c_vp, c_vp]),
    "fm_select_supports_bucketed": (c_i32, [P(FmGrid), c_vp, c_vp, c_vp, c_vp, c_i64, c_vp,
                                            P(FmSelect), c_i32, c_vp, c_vp, c_vp, c_vp, c_vp,
                                            c_i32, c_vp, c_vp, c_vp, c_vp, c_i32, c_vp, c_vp,
                                            c_vp, c_vp]),
    "fm_offsets_ordered_workspace": (c_sz, [c_i64]),
    "fm_offsets_ordered_capped": (c_i32, [c_vp, c_vp, c_i64, c_i32, c_i32, c_vp, c_vp, c_vp,
                                          c_vp, c_sz, c_vp]),
    "fm_offsets_ordered": (c_i32, [c_vp, c_vp, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp, c_sz,
                                   c_vp]),
    "fm_build_operator": (c_i32, [P(FmGrid), c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, P(FmSelect),
                                  c_vp, P(FmLists), c_vp, c_i32, P(FmRbf), P(FmFit), c_vp, c_vp,
                                  c_vp, c_vp, c_vp]),
    "fm_transfer_values": (c_i32, [P(FmGrid), c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, P(FmSelect),
                                   c_vp, P(FmLists), c_i32, P(FmRbf), P(FmFit), c_vp, c_vp, c_vp,
                                   c_vp, c_vp]),
    "fm_apply": (c_i32, [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_vp, c_vp]),
    "fm_fp64_probe": (c_i32, [c_i32, c_i32, c_i32, c_vp, c_vp]),
    # include/fieldmap_dist.h
    "fm_ipc_handle_size": (c_i32, []),
    "fm_device_alloc": (c_i32, [c_sz, P(c_vp)]),
    "fm_device_free": (c_i32, [c_vp]),
    "fm_ipc_export": (c_i32, [c_vp, c_vp]),
    "fm_ipc_open": (c_i32, [c_vp, P(c_vp)]),
    "fm_ipc_close": (c_i32, [c_vp]),
    "fm_push_rows": (c_i32, [c_vp, c_sz, c_sz, c_i32, c_vp, c_vp, c_vp]),
    "fm_build_apply_blocks": (c_i32, [P(FmGrid), c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, P(FmSelect),
                                      c_vp, P(FmLists), c_vp, c_i32, P(FmRbf), P(FmFit), c_vp,
                                      c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_vp, c_i32, c_vp,
                                      c_i32, c_vp, c_vp, c_vp]),
    # include/fieldmap_patch.h
    "fm_patch_count": (c_i32, [c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_i64, c_i32, c_i32, c_vp,
                               c_vp]),
    "fm_patch_fill": (c_i32, [c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_i64, c_i32, c_i32, c_vp,
                              c_vp, c_vp]),
    "fm_patch_big_workspace": (c_sz, [c_i64, c_i32, c_i32]),
    "fm_patch_count_big": (c_i32, [c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_i64, c_i32, c_i32, c_i32,
                                   c_i32, c_vp, c_sz, c_vp, c_vp]),
    "fm_patch_fill_big": (c_i32, [c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_i64, c_i32, c_i32, c_i32,
                                  c_i32, c_vp, c_sz, c_vp, c_vp, c_vp]),
    "fm_locate_batch": (c_i32, [c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_f64,
                                c_f64, c_f64, c_f64, c_i64, c_i64, c_vp, c_vp, c_f64, c_vp, c_vp,
                                c_vp, c_vp, c_vp, c_vp]),
}

_lib = None


class FieldmapError(RuntimeError):
    pass


def lib():
    """The loaded library (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the CUDA extension with "
                "`python -m paper_2510_18838_b200._build` (or __graft_entry__.build()); "
                "there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc, what):
    if rc != FM_OK:
        msg = lib().fm_error_string(rc).decode()
        raise FieldmapError(f"{what} failed: {msg} (code {rc})")


def ptr(t):
    """Device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else ctypes.c_void_p(t.data_ptr())
