"""ctypes binding of the C ABI in ``include/vpb200.h`` (``_lib/libvpb200.so``).

The product path has no CPU fallback: if the library is missing or no CUDA
device is visible, every entry point raises.  Device memory and streams come
from torch (plumbing only); the library receives raw device pointers and the
current stream handle.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

PKG = Path(__file__).resolve().parent
# VPB_LIB_PATH: load another build of the library (A/B timing, tools/ab_time.py)
LIB_PATH = Path(os.environ["VPB_LIB_PATH"]) if os.environ.get("VPB_LIB_PATH") else PKG / "_lib" / "libvpb200.so"

MAX_JOINTS = 16
MAX_SPHERES = 64
MAX_PAIRS = 256
MAX_MASK_SPHERES = 64

PREC_F32 = 0
PREC_F64 = 1
DTYPE_F32 = 0
DTYPE_F64 = 1

_d = ctypes.c_double
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_p = ctypes.c_void_p
_sz = ctypes.c_size_t


class VpbCamera(ctypes.Structure):
    _fields_ = [
        ("fx", _d), ("fy", _d), ("cx", _d), ("cy", _d), ("d_min", _d), ("d_max", _d),
        ("width", _i64), ("height", _i64),
        ("pose_r", _d * 9), ("pose_t", _d * 3), ("w2c_r", _d * 9), ("w2c_t", _d * 3),
    ]


class VpbMapParams(ctypes.Structure):
    _fields_ = [("l_hit", _d), ("l_miss", _d), ("l_min", _d), ("l_max", _d),
                ("l_occ_threshold", _d), ("tau", _d)]


class VpbGrid(ctypes.Structure):
    _fields_ = [("log_odds", _p), ("observed", _p), ("occ_bits", _p), ("dims", _i64 * 3),
                ("origin", _d * 3), ("voxel", _d)]


class VpbJournal(ctypes.Structure):
    _fields_ = [("idx", _p), ("lo", _p), ("ob", _p), ("occ", _p), ("count", _p), ("overflow", _p),
                ("capacity", ctypes.c_uint64), ("starts", _p), ("seg", _i32), ("reset", _i32)]


class VpbField(ctypes.Structure):
    _fields_ = [("sq", _p), ("n", _i64 * 3), ("lo", _i64 * 3), ("origin", _d * 3), ("voxel", _d),
                ("outside_default", _d)]


class VpbProblem(ctypes.Structure):
    _fields_ = [
        ("n_joints", _i32), ("n_spheres", _i32), ("n_pairs", _i32), ("horizon", _i32),
        ("dt", _d),
        ("base_r", _d * 9), ("base_t", _d * 3),
        ("off_r", _d * (MAX_JOINTS * 9)), ("off_t", _d * (MAX_JOINTS * 3)),
        ("axes", _d * (MAX_JOINTS * 3)),
        ("sph_link", _i32 * MAX_SPHERES), ("sph_orig", _i32 * MAX_SPHERES),
        ("sph_loc", _d * (MAX_SPHERES * 3)), ("sph_r", _d * MAX_SPHERES),
        ("pairs", _i32 * (MAX_PAIRS * 2)),
        ("goal_r", _d * 9), ("goal_t", _d * 3),
        ("pose_weight", _d * 36), ("terminal_weight", _d * 36),
        ("pos_lo", _d * MAX_JOINTS), ("pos_hi", _d * MAX_JOINTS),
        ("vel_lo", _d * MAX_JOINTS), ("vel_hi", _d * MAX_JOINTS),
        ("acc_lo", _d * MAX_JOINTS), ("acc_hi", _d * MAX_JOINTS),
        ("acc_limit", _d * MAX_JOINTS), ("q_ref", _d * MAX_JOINTS),
        ("q0", _d * MAX_JOINTS), ("qd0", _d * MAX_JOINTS),
        ("w_env", _d), ("w_self", _d), ("w_q", _d), ("w_qd", _d), ("w_qdd", _d),
        ("w_s", _d), ("w_ns", _d), ("d_act", _d), ("lam", _d), ("dyn_state", _p),
        ("field_sq_dev", _p),
    ]


_P = ctypes.POINTER
SIGNATURES = {
    "vpb_version": (ctypes.c_int, []),
    "vpb_last_error": (ctypes.c_char_p, []),
    "vpb_launch_count": (ctypes.c_uint64, []),
    "vpb_stage_h2d": (ctypes.c_int, [_p, _p, _p, _i64, _p]),
    "vpb_occ_words": (_i64, [_P(_i64)]),
    "vpb_occ_bits_from_log_odds": (ctypes.c_int, [_P(VpbGrid), _d, _p]),
    "vpb_masked_pixels": (ctypes.c_int, [_p, _P(VpbCamera), _p, _p, _i64, _d, _p, _p]),
    "vpb_fuse_voxels": (ctypes.c_int, [_P(VpbGrid), _P(_i64), _P(_i64), _P(VpbCamera), _p, _p, _p, _p,
                                       _i64, _P(VpbMapParams), _p]),
    "vpb_update_occupancy": (ctypes.c_int, [_P(VpbGrid), _P(_i64), _P(_i64), _P(VpbCamera), _p, _p, _p,
                                            _i64, _d, _P(VpbMapParams), _p, _p]),
    "vpb_update_occupancy_journaled": (ctypes.c_int, [_P(VpbGrid), _P(_i64), _P(_i64), _P(VpbCamera), _p, _p,
                                                      _p, _i64, _d, _P(VpbMapParams), _p, _P(VpbJournal), _p]),
    "vpb_journal_restore": (ctypes.c_int, [_P(VpbGrid), _P(VpbJournal), _i64, _i64, _p]),
    "vpb_edt3d_workspace_bytes": (_sz, [_P(_i64)]),
    "vpb_edt3d": (ctypes.c_int, [_P(VpbGrid), _P(_i64), _P(_i64), _d, ctypes.c_int, _p, _p, _sz, _p]),
    "vpb_query_distance": (ctypes.c_int, [_P(VpbField), _p, _i64, _p, _p]),
    "vpb_evaluate_batch": (ctypes.c_int, [_P(VpbProblem), _P(VpbField), _p, _p, ctypes.c_int, _i64,
                                          ctypes.c_int, _p, _p, _p, _p, _p, _p, _p]),
    "vpb_soft_weights_workspace_bytes": (_sz, [_i64]),
    "vpb_soft_weights": (ctypes.c_int, [_p, _i64, _d, _p, _p, _p, _sz, _p]),
    "vpb_update_controls_workspace_bytes": (_sz, [_i64, _i64]),
    "vpb_update_controls": (ctypes.c_int, [_p, _p, ctypes.c_int, _p, _i64, _i64, _p, _p, _sz, _p]),
    "vpb_smpc_workspace_bytes": (_sz, [_i64, _i64, _i64]),
    "vpb_smpc_partial_len": (_i64, [_i64, _i64]),
    "vpb_smpc_partial": (ctypes.c_int, [_P(VpbProblem), _P(VpbField), _p, ctypes.c_int, _p, _i64, _i64,
                                        ctypes.c_int, _p, _p, _p, _p, _sz, _p]),
    "vpb_smpc_out_len": (_i64, [_i64, _i64]),
    "vpb_smpc_step": (ctypes.c_int, [_P(VpbProblem), _P(VpbField), _p, ctypes.c_int, _p, _i64, ctypes.c_int, _p,
                                     _p, _p, _p, _sz, _p]),
    "vpb_smpc_generate": (ctypes.c_int, [_P(VpbProblem), _P(VpbField), ctypes.c_uint64, _p, _i64, _i64, _p, _p, _i64,
                                         ctypes.c_int, _p, _p, _p, _p, _p, _p, _sz, _p]),
    "vpb_smpc_finish_workspace_bytes": (_sz, [_i64, _i64, _i64]),
    "vpb_smpc_finish": (ctypes.c_int, [_P(VpbProblem), _P(VpbField), _p, _i64, _p, ctypes.c_int, _p, _p,
                                       _sz, _p]),
    "vpb_sample_perturbations": (ctypes.c_int, [ctypes.c_uint64, _p, _i64, _i64, _i64, _i64, _i64, _p,
                                                ctypes.c_int, _p, _p]),
    "vpb_debug_smpc_trace": (None, [_p]),
    "vpb_smpc_debug_weights": (ctypes.c_int, [_P(VpbProblem), _i64, _p, _sz, _p, _p]),
    "vpb_pixel_scratch_bytes": (_i64, [_i64, _i64]),
    "vpb_smpc_session_out_len": (_i64, [_i64, _i64]),
    "vpb_smpc_session_create": (ctypes.c_int, [_P(VpbProblem), _P(VpbField), _i64, _i64, _p, ctypes.c_int,
                                               _P(_p)]),
    "vpb_smpc_session_step": (ctypes.c_int, [_p, _p, _p, _p, _p, _p, ctypes.c_uint64, _p, _p, _p]),
    "vpb_smpc_session_launch": (ctypes.c_int, [_p, _p]),
    "vpb_smpc_session_destroy": (ctypes.c_int, [_p]),
    "vpb_ee_errors": (ctypes.c_int, [_P(VpbProblem), _p, _p, _p, _p, _p]),
}

_lib: ctypes.CDLL | None = None


class NativeError(RuntimeError):
    """A CUDA or argument error reported by libvpb200."""


def load() -> ctypes.CDLL:
    """Load the in-tree library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise NativeError(
                f"{LIB_PATH} is missing; build it with `python -m paper_2512_22575_b200.build` "
                "(there is no CPU fallback)"
            )
        lib = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def exported_symbols() -> list[str]:
    return list(SIGNATURES)


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().vpb_last_error().decode(errors="replace")
        if rc == 1:
            raise ValueError(f"{what}: {msg}")
        raise NativeError(f"{what}: {msg}")


def i64x3(v) -> ctypes.Array:
    return (_i64 * 3)(*[int(x) for x in v])


def fill(arr, values) -> None:
    vals = np.asarray(values, dtype=np.float64).reshape(-1)
    for i, v in enumerate(vals):
        arr[i] = float(v)
