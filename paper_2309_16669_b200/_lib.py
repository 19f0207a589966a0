"""ctypes binding of libavion_b200.so -- the ONLY route to compute in this package.

There is no CPU or eager-PyTorch fallback: if the library is missing or a
call fails, the wrapper raises.  Signatures mirror include/avion_b200.h;
`EXPORTS` lists every symbol the header declares (checked by
tests/test_capi.py without a GPU).
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import ConfigurationError, InputError, KernelError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("AVB_LIB", os.path.join(_HERE, "libavion_b200.so"))

AVB_OK, AVB_E_ARG, AVB_E_BOX, AVB_E_UNSUPPORTED, AVB_E_CUDA = 0, 1, 2, 3, 4
AVB_DTYPE_BF16, AVB_DTYPE_F32 = 0, 1
AVB_LAYOUT_CTHW, AVB_LAYOUT_TCHW, AVB_LAYOUT_TUBELET = 0, 1, 2
AVB_K1_PATH_AUTO, AVB_K1_PATH_GENERIC, AVB_K1_PATH_STRIP = 0, 1, 2

_vp, _i32, _i64, _f32p = C.c_void_p, C.c_int, C.c_int64, C.POINTER(C.c_float)

# name -> (restype, argtypes); must match include/avion_b200.h exactly
EXPORTS: dict[str, tuple] = {
    "avb_last_error": (C.c_char_p, []),
    "avb_version": (_i32, []),
    "avb_device_sm_count": (_i32, []),
    "avb_rrc_normalize": (_i32, [_vp, _i64, _i32, _i32, _i32, _i64, _i64, _i64, _i64, _i64,
                                 _vp, _vp, _vp, _i32, _i32, _f32p, _f32p, _i32, _i32, _vp, _vp]),
    "avb_rrc_taps": (_i32, [_i32, _i32, _vp, _vp, _vp, _i32, _vp]),
    "avb_k1_force_path": (_i32, [_i32]),
    "avb_rrc_normalize_tubelet": (_i32, [_vp, _i64, _i32, _i32, _i32, _i64, _i64, _i64, _i64, _i64, _vp, _vp, _vp,
                                         _i32, _i32, _f32p, _f32p, _i32, _i32, _i32, _i32, _vp, _vp]),
    "avb_layernorm_fwd": (_i32, [_vp, _i64, _vp, _vp, _vp, _i64, _vp, _vp, _i32, _i32, C.c_float, _vp]),
    "avb_layernorm_bwd": (_i32, [_vp, _i64, _vp, _i64, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _i32, _i32,
                                 _i32, _vp]),
    "avb_layernorm_bwd_workspace": (_i32, [_i32]),
    "avb_colsum_accum": (_i32, [_vp, _i64, _i32, _i32, _vp, _vp]),
    "avb_tokens_fwd": (_i32, [_vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _vp]),
    "avb_tokens_bwd": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _vp]),
    "avb_patchify": (_i32, [_vp, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _vp, _vp]),
    "avb_xent": (_i32, [_vp, _i64, _vp, _i32, _i32, C.c_float, _vp, _vp, _i64, _vp]),
    "avb_adamw": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _i64, C.c_float, C.c_float, C.c_float, C.c_float, C.c_float, _i32,
                         C.c_float, _vp]),
    "avb_adamw_dev": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _i64, C.c_float, C.c_float, C.c_float, C.c_float, C.c_float,
                             _vp, C.c_float, _vp]),
    "avb_cast_bf16": (_i32, [_vp, _vp, _i64, _vp]),
    "avb_infonce_fwd": (_i32, [_vp, _vp, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "avb_infonce_bwd": (_i32, [_vp, _vp, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _i32, _i32, C.c_float, _vp, _vp,
                               _vp]),
    "avb_embed_fwd": (_i32, [_vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _vp]),
    "avb_embed_bwd": (_i32, [_vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _vp]),
    "avb_rows_copy": (_i32, [_vp, _i64, _vp, _vp, _i64, _vp, _i32, _i32, _vp]),
    "avb_gemm": (_i32, [_vp, _i64, _i32, _vp, _i64, _i32, _vp, _i64, _i32, _i32, _i32, _i32, _vp, _vp, _i64, _vp,
                        C.c_float, _i32, _vp, _vp]),
    "avb_attn_fwd": (_i32, [_vp, _vp, _vp, _i64, _i64, _vp, _i64, _i64, _vp, _i32, _i32, _i32, _i32, C.c_float,
                            _i32, _vp]),
    "avb_attn_bwd": (_i32, [_vp, _vp, _vp, _i64, _i64, _vp, _vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _i64,
                            _i64, _i32, _i32, _i32, _i32, C.c_float, _i32, _vp]),
    "avb_attn_bwd_deterministic": (_i32, [_vp, _vp, _vp, _i64, _i64, _vp, _vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp,
                                          _vp, _i64, _i64, _i32, _i32, _i32, _i32, C.c_float, _i32, _vp]),
}

_lock = threading.Lock()
_lib = None


def load() -> C.CDLL:
    """Load (once) and type the native library; raise if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise KernelError(f"{LIB_PATH} is not built; run `python -m paper_2309_16669_b200.build` "
                              "(there is no CPU fallback)")
        lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        for name, (res, args) in EXPORTS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(status: int, what: str) -> None:
    """Map AVB_E_* to the reference's exception classes (errors.py:18-40)."""
    if status == AVB_OK:
        return
    msg = load().avb_last_error().decode(errors="replace")
    if status == AVB_E_BOX:
        raise InputError(f"{what}: {msg}")
    if status == AVB_E_ARG:
        raise InputError(f"{what}: {msg}")
    if status == AVB_E_UNSUPPORTED:
        raise ConfigurationError(f"{what}: {msg}")
    raise KernelError(f"{what}: {msg} (status {status})")


def f32x3(vals) -> C.Array:
    return (C.c_float * 3)(*[float(v) for v in vals])


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)
