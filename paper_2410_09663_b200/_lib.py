"""ctypes binding of the sm_100a C-ABI library (include/enks_b200.h).

There is no CPU fallback: if ``libenks_b200.so`` is missing, fails to load,
or the current device is not a B200 (sm_100), every entry point raises
:class:`NativeUnavailable`.  Build it with ``python -m paper_2410_09663_b200.build``.
"""
from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libenks_b200.so")

ENKS_OK = 0


class NativeUnavailable(RuntimeError):
    """The CUDA library could not be loaded or the device is unsupported."""


class NativeError(RuntimeError):
    """A C-ABI call returned a non-zero status."""


_c_i64 = ctypes.c_int64
_c_int = ctypes.c_int
_c_f = ctypes.c_float
_c_d = ctypes.c_double
_vp = ctypes.c_void_p
_u32p = ctypes.POINTER(ctypes.c_uint32)
_ip = ctypes.POINTER(ctypes.c_int)

# name -> (restype, argtypes)
_SIGS = {
    "enks_version": (_c_int, []),
    "enks_last_error": (ctypes.c_char_p, []),
    "enks_device_check": (_c_int, []),
    "enks_noise_fill": (_c_int, [_u32p, _c_int, ctypes.c_uint32, ctypes.c_uint32, _c_i64, _c_i64,
                                 _c_int, _c_int, _vp, _vp, _c_i64, _vp, _c_i64, _vp, _c_i64, _vp]),
    "enks_noise_fill_multi": (_c_int, [_u32p, _c_int, _c_i64, _c_i64, _c_int, _c_int, _u32p, _u32p,
                                       _ip, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _c_i64, _vp]),
    "enks_noise_fill_multi_dev": (_c_int, [_vp, _c_int, _c_i64, _c_i64, _c_int, _c_int, _u32p,
                                           _u32p, _ip, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                           _c_i64, _vp]),
    "enks_noise_ws_bytes": (_c_i64, [_c_i64, _c_int, _c_int, _c_int]),
    "enks_member_sum_ws_bytes": (_c_i64, [_c_int, _c_i64, _c_int]),
    "enks_member_sum2_ws_bytes": (_c_i64, [_c_int, _c_int, _c_i64, _c_int]),
    "enks_member_sum2": (_c_int, [_vp, _c_i64, _c_int, _vp, _c_i64, _c_int, _c_i64, _c_int, _vp, _vp,
                                  _vp, _vp, _vp, _vp]),
    "enks_cnn_noise_fusable": (_c_int, [_c_int, _ip, _c_int, _c_int]),
    "enks_cnn_forward_noise": (_c_int, [_c_int, _ip, _vp, _vp, _c_f, _vp, _c_i64, _vp, _c_i64, _vp,
                                        _c_i64, _c_int, _c_int, _c_i64, _u32p, _vp, _c_int, _c_i64,
                                        _c_int, _u32p, _u32p, _ip, _vp, _vp, _vp, _vp, _vp, _vp,
                                        _vp, _vp]),
    "enks_member_sum": (_c_int, [_vp, _c_i64, _vp, _c_i64, _c_int, _c_i64, _c_int, _vp, _vp, _vp,
                                 _vp, _vp]),
    "enks_member_sum_rebase": (_c_int, [_vp, _c_i64, _vp, _c_i64, _c_int, _c_int, _vp, _c_d, _vp]),
    "enks_member_center_f16pair_t": (_c_int, [_vp, _c_i64, _vp, _c_i64, _c_int, _c_i64, _c_int,
                                              _vp, _vp, _vp, _c_i64, _vp, _vp, _vp, _c_i64, _vp,
                                              _vp, _vp, _vp, _c_i64, _vp, _vp]),
    "enks_member_center_f16pair": (_c_int, [_vp, _c_i64, _c_int, _c_i64, _c_int, _vp, _vp, _vp,
                                            _c_i64, _vp, _vp, _vp, _c_i64, _vp, _vp, _vp, _c_i64,
                                            _c_int, _c_int, _c_int, _vp]),
    "enks_uchain_apply": (_c_int, [_vp, _c_i64, _vp, _c_i64, _vp, _c_i64, _vp, _c_i64, _c_int,
                                   _c_int, _c_int, _c_int, _c_int, _vp]),
    "enks_member_center": (_c_int, [_vp, _c_i64, _c_int, _c_i64, _c_int, _vp, _vp, _c_i64, _vp,
                                    _vp, _c_i64, _vp]),
    "enks_gemm_ws_bytes": (_c_i64, [_c_i64, _c_i64, _c_int]),
    "enks_gemm": (_c_int, [_c_int, _c_int, _c_i64, _c_i64, _c_i64, _c_f, _vp, _c_i64, _vp, _c_i64,
                           _c_f, _vp, _c_i64, _vp, _c_i64, _c_int, _vp, _c_i64, _c_i64, _c_i64,
                           _c_int, _vp, _c_int, _vp]),
    "enks_tc_gemm_ws_bytes": (_c_i64, [_c_i64, _c_i64, _c_i64, _c_int]),
    "enks_tf32_split": (_c_int, [_vp, _c_i64, _c_i64, _c_i64, _vp, _vp, _c_int, _vp]),
    "enks_gemm_nt_tc": (_c_int, [_c_i64, _c_i64, _c_i64, _c_f, _vp, _c_i64, _vp, _vp, _c_i64, _vp,
                                 _c_i64, _c_int, _vp, _vp]),
    "enks_gemm_tc": (_c_int, [_c_i64, _c_i64, _c_i64, _c_f, _vp, _c_i64, _vp, _vp, _c_i64, _c_int,
                              _c_f, _vp, _c_i64, _vp, _c_i64, _c_int, _vp, _c_i64, _c_i64, _c_i64,
                              _c_int, _vp, _vp]),
    "enks_f16pair_split": (_c_int, [_vp, _c_i64, _c_i64, _c_i64, _vp, _vp, _c_i64, _vp, _vp]),
    "enks_f16pair_recon": (_c_int, [_vp, _vp, _c_i64, _vp, _c_i64, _c_i64, _vp, _c_i64, _vp]),
    "enks_gemm_f16pair_ws_bytes": (_c_i64, [_c_i64, _c_i64, _c_i64]),
    "enks_set_sm_reserve": (_c_int, [_c_int]),
    "enks_gemm_f16pair": (_c_int, [_c_i64, _c_i64, _c_i64, _c_f, _vp, _vp, _c_i64, _vp, _vp, _vp,
                                   _c_i64, _vp, _vp, _c_i64, _vp, _vp]),
    "enks_gemm_f16pair_ex": (_c_int, [_c_i64, _c_i64, _c_i64, _c_f, _vp, _vp, _c_i64, _vp, _vp, _vp,
                                      _c_i64, _vp, _c_f, _vp, _c_i64, _vp, _c_i64, _c_int, _vp,
                                      _c_i64, _vp]),
    "enks_gemm_f16pair_ex_mn": (_c_int, [_c_i64, _c_i64, _c_i64, _c_f, _vp, _vp, _c_i64, _vp, _vp,
                                         _vp, _c_i64, _vp, _c_f, _vp, _c_i64, _vp, _c_i64, _c_int,
                                         _vp, _c_i64, _vp]),
    "enks_f16pair_split_cs": (_c_int, [_vp, _c_i64, _c_i64, _c_i64, _vp, _vp, _vp, _c_i64, _vp,
                                       _vp]),
    "enks_f16pair_transpose": (_c_int, [_vp, _vp, _c_i64, _vp, _c_int, _c_i64, _vp, _vp, _c_i64,
                                        _vp, _vp]),
    "enks_spd_max_p": (_c_int, []),
    "enks_spd_ws_bytes": (_c_i64, [_c_int]),
    "enks_spd_inverse": (_c_int, [_vp, _c_i64, _c_int, _c_f, _vp, _vp, _vp, _vp, _vp]),
    "enks_cnn_max_width": (_c_int, []),
    "enks_cnn_forward": (_c_int, [_c_int, _ip, _vp, _vp, _c_f, _vp, _c_i64, _vp, _c_i64, _vp,
                                  _c_i64, _c_int, _c_int, _c_i64, _vp]),
    "enks_cnn_ws_bytes": (_c_i64, [_c_int, _ip, _c_int, _c_int, _c_i64]),
    "enks_cnn_forward_ws": (_c_int, [_c_int, _ip, _vp, _vp, _c_f, _vp, _c_i64, _vp, _c_i64, _vp,
                                     _c_i64, _c_int, _c_int, _c_i64, _vp, _c_i64, _vp]),
    "enks_burgers_ws_bytes": (_c_i64, [_c_int, _c_int, _c_int]),
    "enks_burgers_forward": (_c_int, [_vp, _c_i64, _vp, _c_i64, _c_int, _vp, _c_i64, _c_int,
                                      _c_int, _c_int, _c_d, _c_d, _c_d, _vp, _vp, _vp, _vp]),
    "enks_barrier_row": (_c_int, [_vp, _c_i64, _c_int, _c_int, _c_i64, _c_int, _vp, _c_i64, _c_d,
                                  _c_int, _c_int, _c_d, _c_d, _c_d, _vp, _vp, _vp]),
    "enks_quad_form": (_c_int, [_vp, _c_i64, _vp, _c_i64, _c_i64, _c_i64, _c_d, _vp, _c_int, _vp]),
    "enks_add": (_c_int, [_vp, _c_i64, _vp, _c_i64, _vp, _c_i64, _c_i64, _c_i64, _vp]),
    "enks_sub": (_c_int, [_vp, _c_i64, _vp, _c_i64, _vp, _c_i64, _c_i64, _c_i64, _vp]),
}

EXPORTED = tuple(_SIGS)

_lock = threading.Lock()
_lib = None
_checked_device = False


def load_library(check_device: bool = True) -> ctypes.CDLL:
    """Load libenks_b200.so (once).  With check_device, also verify an sm_100 GPU."""
    global _lib, _checked_device
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeUnavailable(
                    f"{LIB_PATH} not built; run `python -m paper_2410_09663_b200.build`")
            try:
                lib = ctypes.CDLL(LIB_PATH)
            except OSError as exc:  # pragma: no cover - environment specific
                raise NativeUnavailable(f"cannot load {LIB_PATH}: {exc}") from exc
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
        if check_device and not _checked_device:
            import torch

            if not torch.cuda.is_available():
                raise NativeUnavailable("no CUDA device: the B200 path has no CPU fallback")
            torch.cuda.init()
            if not _lib.enks_device_check():
                raise NativeUnavailable("device check failed: "
                                        + _lib.enks_last_error().decode(errors="replace"))
            _checked_device = True
        return _lib


def call(name: str, *args) -> int:
    lib = load_library()
    rc = getattr(lib, name)(*args)
    if getattr(lib, name).restype is _c_int and name not in ("enks_version", "enks_device_check",
                                                              "enks_spd_max_p",
                                                              "enks_cnn_max_width"):
        if rc != ENKS_OK:
            raise NativeError(f"{name} failed ({rc}): "
                              + lib.enks_last_error().decode(errors="replace"))
    return rc
