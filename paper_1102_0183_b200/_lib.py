"""ctypes binding of ``libckb200.so`` (the C ABI in ``include/ckb200.h``).

The library is built in-tree by ``build.py`` (nvcc, sm_100a).  There is no
fallback: if the shared object is missing or fails to load, every entry
point raises, so a silent CPU path can never stand in for the CUDA one.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import CK_OK, StateError, error_for_status

LIB_NAME = "libckb200.so"
LIB_PATH = os.environ.get("CKB200_LIB") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), LIB_NAME)   # override: experiments only

_i32 = C.c_int
_i64 = C.c_int64
_f64 = C.c_double
_vp = C.c_void_p
_pf = C.c_void_p      # device or host float* (passed as integers/addresses)
_pi64 = C.c_void_p


class LayerDesc(C.Structure):
    """Mirror of ``ck_layer_desc``."""

    _fields_ = [
        ("kind", C.c_int32),
        ("maps", C.c_int32), ("width", C.c_int32), ("height", C.c_int32),
        ("kx", C.c_int32), ("ky", C.c_int32), ("sx", C.c_int32), ("sy", C.c_int32),
        ("px", C.c_int32), ("py", C.c_int32),
        ("n_pairs", C.c_int32),
        ("arena_size", C.c_int32),
        ("fwd_offsets", _vp), ("fwd_srcs", _vp), ("fwd_widx", _vp), ("bias_offset", _vp),
        ("n_filters", C.c_int32),
        ("filter_h", C.c_int32), ("filter_w", C.c_int32),
        ("filter_coeffs", _vp),
    ]


# name -> (restype, argtypes)
_SIGNATURES = {
    "ck_last_error": (C.c_char_p, []),
    "ck_abi_version": (_i32, []),
    "ck_kernel_launches": (_i32, [C.POINTER(_i64)]),
    "ck_conv_fwd": (_i32, [_pf, _i32, _i32, _i32, _pf, _pi64, _pi64, _pi64, _pi64,
                           _i32, _i32, _i32, _i32, _pf, _pf, _i32, _i32, _i32, _i32,
                           _i32, _vp]),
    "ck_pull_bwd": (_i32, [_pf, _i32, _i32, _i32, _i32, _i32, _pf, _pi64, _pi64, _pi64,
                           _i32, _i32, _i32, _i32, _pf, _i32, _i32, _i32, _i32, _i32,
                           _vp]),
    "ck_weight_grad": (_i32, [_pf, _i32, _i32, _i32, _i32, _i32, _pf, _i32, _i32, _i32,
                              _pi64, _pi64, _pi64, _i32, _i32, _i32, _i32, _i32, _pf,
                              _vp]),
    "ck_bias_grad": (_i32, [_pf, _i32, _i32, _i32, _i32, _i32, _pi64, _pf, _vp]),
    "ck_maxpool_fwd": (_i32, [_pf, _i32, _i32, _i32, _i32, _i32, _pf, _i32, _i32, _i32,
                              _i32, _pi64, _pi64, _vp]),
    "ck_maxpool_bwd": (_i32, [_pf, _i32, _i32, _i32, _i32, _i32, _pi64, _pi64, _pf,
                              _i32, _i32, _vp]),
    "ck_contrast": (_i32, [_pf, _i32, _i32, _i32, _i32, _i32, _vp, _i32, _i32, _i32,
                           _pf, _i32, _i32, _vp]),
    "ck_fc_fwd": (_i32, [_pf, _i32, _pf, _pf, _i32, _pf, _pf, _vp]),
    "ck_fc_bwd_update": (_i32, [_pf, _i32, _pf, _pf, _i32, _pf, _pf, _pf, _pf, _f64, _vp]),
    "ck_act_deriv_mul": (_i32, [_pf, _pf, _i32, _i32, _i32, _i32, _i32, _vp]),
    "ck_sgd_update": (_i32, [_pf, _pf, _i64, _f64, _vp]),
    "ck_output_deltas": (_i32, [_pf, _pf, _vp, _i32, _pf, _vp, _vp, _vp]),
    "ck_net_create": (_i32, [C.POINTER(LayerDesc), _i32, _i32, C.POINTER(_vp)]),
    "ck_net_destroy": (_i32, [_vp]),
    "ck_net_set_team": (_i32, [_vp, _i32, _i32, _i32]),
    "ck_net_get_team": (_i32, [_vp, C.POINTER(_i32), C.POINTER(_i32), C.POINTER(_i32)]),
    "ck_net_num_params": (_i32, [_vp, C.POINTER(_i64)]),
    "ck_net_set_params": (_i32, [_vp, _vp, _i64]),
    "ck_net_get_params": (_i32, [_vp, _vp, _i64]),
    "ck_net_forward": (_i32, [_vp, _vp, _vp]),
    "ck_net_backward": (_i32, [_vp, _vp]),
    "ck_net_apply_gradients": (_i32, [_vp, _f64]),
    "ck_net_train_step": (_i32, [_vp, _vp, _vp, _f64, C.POINTER(_f64)]),
    "ck_net_buffer_size": (_i32, [_vp, _i32, _i32, C.POINTER(_i64)]),
    "ck_net_read_buffer": (_i32, [_vp, _i32, _i32, _vp, _i64]),
    "ck_net_train_epoch": (_i32, [_vp, _vp, _vp, _vp, _vp, _i64, _f64, _vp,
                                  C.POINTER(_f64), _vp]),
    "ck_committee_train_epoch": (_i32, [C.POINTER(_vp), _i32, _vp, _vp, _vp, _vp, _i64,
                                        _f64, C.POINTER(_f64), _vp]),
    "ck_net_eval": (_i32, [_vp, _vp, _vp, _i64, _i64, _vp, _vp, _vp]),
    "ck_net_profile_epoch": (_i32, [_vp, _vp, _vp, _vp, _vp, _i64, _f64, _vp, _i32,
                                    C.POINTER(_i32)]),
    "ck_net_describe_program": (_i32, [_vp, _i32, C.c_char_p, _i32]),
    "ck_debug_subprof": (_i32, [_vp, _i32]),
    "ck_net_spec_source": (_i32, [C.POINTER(LayerDesc), _i32, C.c_char_p, C.c_char_p, _i64,
                                  C.POINTER(_i64)]),
    "ck_net_set_specialized": (_i32, [_vp, _i32]),
    "ck_net_kernel_info": (_i32, [_vp, C.c_char_p, _i32]),
    "ck_deform_epoch": (_i32, [_vp, _vp, _i32, _i32, _i32, _i64, _vp, _vp, _i32,
                               C.c_uint64, C.c_uint64, _vp, _vp, _vp]),
    "ck_tc_create": (_i32, [C.POINTER(LayerDesc), _i32, _i32, _i64, _i32, C.POINTER(_vp)]),
    "ck_tc_destroy": (_i32, [_vp]),
    "ck_tc_set_params": (_i32, [_vp, _vp, _vp]),
    "ck_tc_eval_run": (_i32, [_vp, _vp, _vp, _i64, _i64, _vp, _vp, _vp]),
    "ck_net_device_params": (_i32, [_vp, C.POINTER(_vp)]),
    "ck_tct_create": (_i32, [C.POINTER(LayerDesc), _i32, _i32, _vp, C.POINTER(_vp)]),
    "ck_tct_destroy": (_i32, [_vp]),
    "ck_tct_train_epoch": (_i32, [_vp, _vp, _vp, _vp, _vp, _i64, _f64, C.POINTER(_f64), _vp]),
    "ck_deform_apply": (_i32, [_vp, _vp, _i32, _i32, _i32, _i64, _vp, _vp, _i32, _vp, _vp]),
}

EXPORTED_SYMBOLS = tuple(_SIGNATURES)

_lock = threading.Lock()
_lib = None


def load():
    """The loaded library (raises StateError if it is absent or broken)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise StateError(
                    f"{LIB_PATH} is missing: build it with `python build.py` "
                    "(there is no CPU fallback)")
            lib = C.CDLL(LIB_PATH)
            for name, (res, args) in _SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def call(name: str, *args) -> None:
    """Invoke a status-returning entry point; non-zero status raises the
    mapped reference exception type."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != CK_OK:
        msg = lib.ck_last_error()
        raise error_for_status(rc, msg.decode() if msg else "")


def kernel_launches() -> int:
    n = _i64(0)
    call("ck_kernel_launches", C.byref(n))
    return int(n.value)
