"""ctypes binding of libsgad.so (the C ABI in include/sgad.h).

There is no CPU fallback: if the library is missing or no CUDA device is
visible, every hot-path entry point raises.  PyTorch supplies device memory
and the current stream; only raw pointers cross the boundary.
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# SGAD_LIB overrides the library path (A/B experiments with alternative builds)
LIB_PATH = os.environ.get("SGAD_LIB") or os.path.join(_HERE, "libsgad.so")

SGAD_OK = 0
_ERRORS = {-1: ValueError, -2: RuntimeError, -3: MemoryError, -4: RuntimeError}

_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_f64 = ctypes.c_double


class Frame(ctypes.Structure):
    _fields_ = [("planes", _vp), ("mask", _vp), ("gauss_offset", _i64), ("frame_index", _i64),
                ("height", _i32), ("width", _i32), ("learnable", _i32), ("planes_f64", _i32),
                ("fx", _f64), ("fy", _f64), ("cx", _f64), ("cy", _f64),
                ("rot", _f64 * 9), ("trans", _f64 * 3)]


class Camera(ctypes.Structure):
    _fields_ = [("fx", _f64), ("fy", _f64), ("cx", _f64), ("cy", _f64),
                ("width", _i32), ("height", _i32)]


class LossTarget(ctypes.Structure):
    _fields_ = [("color", _vp), ("depth", _vp), ("mask", _vp), ("rho", _f64), ("sigma", _f64),
                ("n_depth", _i64), ("loss_accum", _vp)]


assert ctypes.sizeof(Frame) == 176

_SIGNATURES = {
    "sgad_last_error": (ctypes.c_char_p, []),
    "sgad_version": (_i32, []),
    "sgad_launch_count": (_i32, [ctypes.POINTER(_i64)]),
    "sgad_voxels_create": (_i32, [ctypes.POINTER(_vp)]),
    "sgad_voxels_destroy": (_i32, [_vp]),
    "sgad_voxels_gate": (_i32, [_vp, _vp, _i64, _f64, _vp, ctypes.POINTER(_i64), _vp]),
    "sgad_irls_normal_eqs": (_i32, [_vp, _vp, _i64, ctypes.POINTER(_f64), _f64, _vp, _vp, _vp]),
    "sgad_inpaint_jacobi": (_i32, [_vp, _vp, _i32, _i32, _i32, _f64, _vp, ctypes.POINTER(_i32),
                                   _vp]),
    "sgad_ssim_workspace_size": (_i32, [_i32, _i32, _i32, ctypes.POINTER(_i64)]),
    "sgad_ssim": (_i32, [_vp, _vp, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _f64, _f64, _i32, _vp]),
    "sgad_raster_create": (_i32, [ctypes.POINTER(_vp)]),
    "sgad_raster_destroy": (_i32, [_vp]),
    "sgad_raster_prepare": (_i32, [_vp, ctypes.POINTER(Frame), _i32, ctypes.POINTER(Camera), _i32,
                                   _vp, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
    "sgad_raster_prepare_async": (_i32, [_vp, ctypes.POINTER(Frame), _i32, ctypes.POINTER(Camera),
                                         _i32, _vp, _vp, _vp, _vp]),
    "sgad_raster_reserve": (_i32, [_vp, _i64]),
    "sgad_raster_forward": (_i32, [_vp, _vp, _vp, _vp, _vp, _i32, ctypes.POINTER(LossTarget), _vp]),
    "sgad_raster_backward": (_i32, [_vp, _i32, _vp, _vp, _vp, ctypes.POINTER(_vp), _vp, _vp]),
    "sgad_raster_forward_backward": (_i32, [_vp, ctypes.POINTER(LossTarget), _vp, _vp]),
    "sgad_raster_get_survivors": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "sgad_raster_get_tiles": (_i32, [_vp, _vp, _vp, _vp]),
    "sgad_raster_tile_count": (_i32, [_vp, ctypes.POINTER(_i64)]),
    "sgad_adam_step": (_i32, [_vp, _vp, _vp, _vp, _i64, _i64, ctypes.POINTER(_f64), _f64, _f64,
                              _f64, _f64, _f64, _i32, _i32, _vp, _vp, _vp]),
    "sgad_sym_eigh3": (_i32, [_vp, _i64, _vp, _vp, _vp]),
    "sgad_track_fit": (_i32, [_vp, _vp, _i32, _i32, _f64, _f64, _f64, _f64, _i32, _i32, _i32, _i32,
                              _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "sgad_geomset_create": (_i32, [ctypes.POINTER(_vp)]),
    "sgad_geomset_destroy": (_i32, [_vp]),
    "sgad_geomset_set": (_i32, [_vp, _vp, _vp, _vp, _i64, _vp]),
    "sgad_geomset_nearest": (_i32, [_vp, _vp, _i64, _vp, _vp, _vp]),
    "sgad_track_normal_eqs": (_i32, [_vp, _vp, _vp, _i64, ctypes.POINTER(_f64),
                                     ctypes.POINTER(_f64), _i32, _f64, _i32, _vp, _vp]),
    "sgad_track_accepted": (_i32, [_vp, _vp, _i64, _vp]),
    "sgad_track_correspondences": (_i32, [_vp, _vp, _i64, _vp]),
    "sgad_track_cost": (_i32, [_vp, _vp, _i64, ctypes.POINTER(_f64), _i32, _vp, _vp]),
    "sgad_track_to_world": (_i32, [_vp, _vp, _vp, _vp, _i64, ctypes.POINTER(_f64),
                                   ctypes.POINTER(_f64), _vp, _vp, _vp, _vp, _vp]),
    "sgad_track_gicp": (_i32, [_vp, _vp, _vp, _i64, ctypes.POINTER(_f64), _i32, _f64, _i32, _f64,
                               _i32, _i32, _vp, _vp, _vp, _vp, _vp]),
}

EXPORTS = tuple(_SIGNATURES)

_lib = None
_lock = threading.Lock()


def load(require_cuda: bool = True):
    """Load libsgad.so; raise loudly when it (or a CUDA device) is missing."""
    global _lib
    if require_cuda and not torch.cuda.is_available():
        raise RuntimeError("paper_2603_21055_b200 needs a CUDA device (B200); no CPU fallback")
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                                       "or python -m paper_2603_21055_b200.build")
                lib = ctypes.CDLL(LIB_PATH)
                for name, (res, args) in _SIGNATURES.items():
                    fn = getattr(lib, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = lib
    return _lib


def check(rc: int):
    if rc != SGAD_OK:
        msg = _lib.sgad_last_error().decode(errors="replace") if _lib is not None else "?"
        raise _ERRORS.get(rc, RuntimeError)(f"libsgad error {rc}: {msg}")


def call(name, *args):
    check(getattr(load(), name)(*args))


def ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def launch_count() -> int:
    """Kernels of libsgad launched so far in this process."""
    n = _i64()
    check(load().sgad_launch_count(ctypes.byref(n)))
    return n.value
