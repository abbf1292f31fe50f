"""ctypes binding of libevoformer_sm100.so (declared in include/evoformer_sm100.h).

The product path has exactly one implementation: these sm_100a kernels.
There is no CPU or eager-PyTorch fallback -- if the library is missing, or
the device is not a B200, every op raises ``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes
import os

from .errors import ContractError, DimensionError, NativeUnavailable

_HERE = os.path.dirname(os.path.abspath(__file__))
# EVO_LIB_PATH: load another build of the same library (A/B timing of kernel variants)
LIB_PATH = os.environ.get("EVO_LIB_PATH") or os.path.join(_HERE, "libevoformer_sm100.so")

F32, BF16 = 0, 1
PARTIAL_BLOCKS = 256

_i, _i64, _f, _d, _p, _sz = (ctypes.c_int, ctypes.c_int64, ctypes.c_float, ctypes.c_double,
                             ctypes.c_void_p, ctypes.c_size_t)

# name -> (restype, argtypes); the single source of truth for the ABI binding
SIGNATURES = {
    "evo_last_error": (ctypes.c_char_p, []),
    "evo_version": (_i, []),
    "evo_device_check": (_i, [ctypes.POINTER(_i), ctypes.POINTER(_i), ctypes.POINTER(_i)]),
    "evo_launch_count": (_i64, []),
    "evo_defer_begin": (_i, [_p, _sz]),
    "evo_defer_end": (_i, [_p]),
    "evo_defer_used": (_sz, []),
    "evo_gemm": (_i, [_i64, _i64, _i64, _p, _i64, _i, _i64, _p, _i64, _i, _i64, _p, _i64, _i64,
                      _i, _f, _f, _i, _i, _p]),
    "evo_gemm_tc_launches": (_i64, []),
    "evo_gemm_relu_mask": (_i, [_i64, _i64, _i64, _p, _i64, _i, _p, _i64, _i, _p, _p, _i, _p, _i, _p, _p]),
    "evo_gemm_relu_mask_workspace": (_i64, [_i64, _i64]),
    "evo_gemm_bias": (_i, [_i64, _i64, _i64, _p, _i64, _i, _p, _i64, _i, _p, _i, _p, _p, _i, _p, _i64, _i,
                           _i, _p]),
    "evo_layernorm_fwd": (_i, [_p, _i, _p, _p, _p, _i, _p, _p, _i64, _i64, _f, _p]),
    "evo_layernorm_bwd_workspace": (_i64, [_i64, _i64]),
    "evo_layernorm_bwd": (_i, [_p, _i, _p, _i, _p, _p, _p, _p, _p, _p, _p, _i, _p, _i64, _i64, _p]),
    "evo_layernorm_bwd_ex": (_i, [_p, _i, _p, _i, _p, _p, _p, _p, _p, _p, _p, _p, _p, _i, _p, _i64,
                                  _i64, _p]),
    "evo_bias_residual": (_i, [_p, _i, _p, _i, _p, _p, _i, _i64, _i64, _p]),
    "evo_bias_relu": (_i, [_p, _i, _p, _i64, _i64, _p]),
    "evo_relu_bwd_colsum": (_i, [_p, _p, _i, _p, _i, _p, _i64, _i64, _p]),
    "evo_colsum_workspace": (_i64, [_i64]),
    "evo_colsum_cast": (_i, [_p, _i, _p, _i, _p, _i, _p, _i64, _i64, _p]),
    "evo_colsum_strided": (_i, [_p, _i, _i64, _p, _i, _p, _i64, _i64, _p]),
    "evo_cast": (_i, [_p, _i, _p, _i, _i64, _p]),
    "evo_pack_cols": (_i, [ctypes.POINTER(_p), ctypes.POINTER(_p), ctypes.POINTER(_i64),
                           ctypes.POINTER(_i64), _i, _i, _i, _i, _p]),
    "evo_pack_cols_ns": (_i, [ctypes.POINTER(_p), ctypes.POINTER(_p), ctypes.POINTER(_i64),
                           ctypes.POINTER(_i64), _i, _i, _i, _i, _i, _p]),
    "evo_scale_inplace": (_i, [_p, _f, _i64, _p]),
    "evo_attn_fwd": (_i, [_p, _i64, _p, _i64, _i64, _p, _p, _p, _p, _p, _p,
                          _i64, _i64, _i64, _i64, _i64, _i64, _i, _p]),
    "evo_attn_bwd_workspace": (_i64, [_i64, _i64, _i64, _i64, _i]),
    "evo_softmax_masked_rows": (_i, [_p, _p, _i64, _i64, _p, _i64, _i64, _i64, _p]),
    "evo_softmax_rows_bwd": (_i, [_p, _p, _i64, _i64, _p]),
    "evo_gate_fwd": (_i, [_p, _p, _p, _p, _i64, _p]),
    "evo_gate_bwd": (_i, [_p, _p, _p, _p, _p, _i64, _p]),
    "evo_sum_rows": (_i, [_p, _i64, _i64, _p, _i, _p]),
    "evo_attn_bwd": (_i, [_p, _i64, _p, _i64, _i64, _p, _p, _p, _p, _p, _p, _p, _p, _i, _p, _sz,
                          _i64, _i64, _i64, _i64, _i64, _i64, _i, _p]),
    "evo_pair_bias_fwd": (_i, [_p, _i, _p, _p, _p, _p, _p, _p, _i64, _i64, _i64, _i, _p]),
    "evo_pair_bias_fwd_rect": (_i, [_p, _i, _p, _p, _p, _p, _p, _p, _i64, _i64, _i64, _i64, _i, _p]),
    "evo_ln_pair_bias_fwd": (_i, [_p, _i, _p, _p, _p, _p, _p, _p, _p, _p, _p, _i64, _i64, _i64, _i64, _i, _p]),
    "evo_pair_bias_bwd_rect": (_i, [_p, _i, _p, _p, _p, _p, _p, _p, _i, _p, _p, _p, _p, _i, _p,
                                    _i64, _i64, _i64, _i64, _p]),
    "evo_pair_bias_bwd_ex": (_i, [_p, _i, _p, _p, _p, _p, _p, _p, _i, _p, _p, _p, _p, _i, _p,
                                  _i64, _i64, _i64, _i64, _p, _p, _p]),
    "evo_opm_norm_fwd_rows": (_i, [_p, _i, _p, _p, _p, _i, _i64, _i64, _i64, _i64, _i64, _p]),
    "evo_opm_norm_bwd_rows": (_i, [_p, _i, _p, _p, _i, _i64, _i64, _i64, _p]),
    "evo_swap01": (_i, [_p, _p, _i64, _i64, _i64, _p]),
    "evo_opm_dnum": (_i, [_p, _p, _p, _p, _i64, _i64, _i64, _i64, _i, _p]),
    "evo_opm_outn": (_i, [_p, _p, _p, _p, _i64, _i64, _i64, _i64, _i, _p]),
    "evo_opm_rec": (_i, [_p, _p, _i64, _i64, _i64, _i64, _p]),
    "evo_opm_norm_apply_rows": (_i, [_p, _i, _p, _p, _i, _i64, _i64, _i64, _p]),
    "evo_pair_bias_bwd_workspace": (_i64, [_i64, _i64]),
    "evo_pair_bias_bwd": (_i, [_p, _i, _p, _p, _p, _p, _p, _p, _i, _p, _p, _p, _p, _i, _p,
                               _i64, _i64, _i64, _p]),
    "evo_opm_proj": (_i, [_p, _p, _p, _p, _p, _p, _i64, _i64, _i, _p]),
    "evo_opm_proj_bwd": (_i, [_p, _p, _p, _p, _p, _p, _i, _p, _i64, _i64, _i, _p]),
    "evo_opm_norm_fwd": (_i, [_p, _i, _p, _p, _p, _i, _i64, _i64, _i64, _p]),
    "evo_opm_norm_bwd": (_i, [_p, _i, _p, _p, _i, _i64, _i64, _p]),
    "evo_sq_loss_workspace": (_i64, []),
    "evo_sq_loss": (_i, [_p, _i64, _p, _i64, _i, _f, _f, _p, _p, _p, _p, _p]),
    "evo_trimul_gate_fwd": (_i, [_p, _i64, _p, _p, _p, _p, _p, _p, _p, _i64, _i64, _i, _p]),
    "evo_trimul_gate_bwd": (_i, [_p, _i64, _p, _p, _p, _p, _p, _p, _p, _p, _i64, _i64, _i, _p]),
    "evo_transpose2d": (_i, [_p, _i, _p, _i, _i64, _i64, _p]),
    "evo_gated_residual": (_i, [_p, _p, _i64, _p, _p, _p, _p, _p, _i64, _i64, _i, _p]),
    "evo_gated_residual_bwd": (_i, [_p, _p, _p, _p, _p, _p, _i64, _i64, _i, _p]),
    "evo_sumsq_workspace": (_i64, []),
    "evo_sumsq_f64": (_i, [_p, _i64, _p, _p, _p]),
    "evo_sumsq_f64_step": (_i, [_p, _i64, _p, _p, _p, _p, _i64, _p, _p]),
    "evo_adam_clip_ema_dev": (_i, [_p, _p, _p, _p, _p, _p, _i64, _p, _d, _f, _f, _f, _f, _f, _f, _p,
                                   _f, _f, _p]),
    "evo_adam_clip_ema": (_i, [_p, _p, _p, _p, _p, _p, _i64, _p, _d, _f, _f, _f, _f, _f, _f,
                               _f, _f, _f, _f, _p]),
}

_lib = None


def load(path: str = LIB_PATH):
    """Load and bind the library (no device needed)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeUnavailable(
            f"{path} is missing: build it with `python -m paper_2207_05477_b200.build` "
            "(there is no fallback implementation)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


_device_ok = None


def lib():
    """The bound library, after checking that the current device is sm_100."""
    global _device_ok
    L = load()
    if _device_ok is None:
        ma, mi, n = _i(), _i(), _i()
        rc = L.evo_device_check(ctypes.byref(ma), ctypes.byref(mi), ctypes.byref(n))
        if rc != 0:
            raise NativeUnavailable(L.evo_last_error().decode())
        _device_ok = (ma.value, mi.value, n.value)
    return L


def check(rc: int):
    if rc == 0:
        return
    msg = _lib.evo_last_error().decode() if _lib is not None else "unknown"
    if rc == 1:
        raise ContractError(msg)
    if rc == 3:
        raise DimensionError(msg)
    raise RuntimeError(f"libevoformer_sm100 error {rc}: {msg}")


def call(name: str, *args):
    check(getattr(lib(), name)(*args))


def launch_count() -> int:
    return int(load().evo_launch_count())
