"""ctypes binding of include/ensemble_b200.h.

The library is the product path: there is no CPU fallback.  If the shared
object is missing or cannot be loaded, every entry point raises at import of
the consumer (``load()``), loudly.
"""

from __future__ import annotations

import ctypes
import os
import threading
from ctypes import POINTER, c_char_p, c_double, c_float, c_int, c_int32, c_int64, c_uint64, c_void_p
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libensemble_b200.so"

EB_OK = 0
EB_E_INVALID = 1
EB_E_CUDA = 2
EB_E_SHAPE = 3
EB_E_EMPTY = 4
EB_E_TOO_LARGE = 5
EB_E_POLICY = 6
EB_E_BAD_K = 7
EB_E_NOMEM = 8
EB_E_STATE = 9

EB_IN_F32_CHW = 0
EB_IN_U8_HWC = 1

EB_BF16, EB_F32, EB_F64 = 0, 1, 2
EB_T_IMAGE_NHWC8 = 0
EB_T_IMAGE_F32 = 1

EB_OP_CONV, EB_OP_POOL, EB_OP_BNRELU, EB_OP_GAP, EB_OP_LIN1, EB_OP_RESIZE = 0, 1, 2, 3, 4, 5
EB_POOL_MAX, EB_POOL_AVG, EB_POOL_AVG_EXCL_PAD = 0, 1, 2
EB_POLICY_NONE, EB_POLICY_ANY, EB_POLICY_ALL, EB_POLICY_AT_LEAST = 0, 1, 2, 3
EB_MEMBER_CNN, EB_MEMBER_LIN1 = 0, 1
EB_PREC_BF16, EB_PREC_F32 = 0, 1
EB_NO_OFFSET = (1 << 64) - 1


class OpDesc(ctypes.Structure):
    _fields_ = [
        ("kind", c_int32),
        ("src", c_int32), ("dst", c_int32), ("res", c_int32),
        ("src_c_off", c_int32), ("src_c", c_int32),
        ("dst_c_off", c_int32), ("cout", c_int32),
        ("kh", c_int32), ("kw", c_int32), ("sh", c_int32), ("sw", c_int32),
        ("ph", c_int32), ("pw", c_int32),
        ("relu", c_int32),
        ("pool_mode", c_int32),
        ("flatten", c_int32),
        ("stream", c_int32),
        ("groups", c_int32),
        ("prefork", c_int32),
        ("dst2", c_int32), ("dst2_c_off", c_int32), ("n_split", c_int32),
        ("w_off", c_uint64), ("b_off", c_uint64), ("scale_off", c_uint64), ("shift_off", c_uint64),
    ]


class EbError(RuntimeError):
    """A native call failed; ``status`` is the eb_status code."""

    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status


_SIGS = {
    "eb_last_error": (c_char_p, []),
    "eb_abi_version": (c_int, []),
    "eb_engine_create": (c_int, [c_int, c_int, c_int, c_int, c_int, POINTER(c_void_p)]),
    "eb_engine_destroy": (c_int, [c_void_p]),
    "eb_engine_set_precision": (c_int, [c_void_p, c_int]),
    "eb_engine_clone": (c_int, [c_void_p, POINTER(c_void_p)]),
    "eb_engine_warmup": (c_int, [c_void_p, c_int, c_int]),
    "eb_set_preprocess": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_void_p]),
    "eb_pool_reserve": (c_int, [c_void_p, c_uint64]),
    "eb_pool_write": (c_int, [c_void_p, c_uint64, c_void_p, c_uint64]),
    "eb_pool_bytes": (c_int, [c_void_p, POINTER(c_uint64)]),
    "eb_tensor": (c_int, [c_void_p, c_int, c_int, c_int, c_int, POINTER(c_int)]),
    "eb_add_op": (c_int, [c_void_p, POINTER(OpDesc)]),
    "eb_add_member": (c_int, [c_void_p, c_int, c_int, c_int, c_int]),
    "eb_finalize": (c_int, [c_void_p]),
    "eb_forward": (c_int, [c_void_p, c_void_p, c_int, c_int, c_void_p, c_void_p, c_int,
                           c_void_p, c_void_p, c_int, c_int, c_void_p]),
    "eb_forward_device": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_int]),
    "eb_forward_batches": (c_int, [c_void_p, POINTER(c_void_p), c_int, c_int, c_int,
                                   POINTER(c_void_p)]),
    "eb_input_buffer": (c_int, [c_void_p, c_int, POINTER(c_void_p)]),
    "eb_output_labels": (c_int, [c_void_p, POINTER(c_void_p)]),
    "eb_tensor_ptr": (c_int, [c_void_p, c_int, POINTER(c_void_p), POINTER(c_int), POINTER(c_int),
                              POINTER(c_int), POINTER(c_int)]),
    "eb_engine_stream": (c_int, [c_void_p, POINTER(c_void_p)]),
    "eb_launch_count": (c_int, [c_void_p, c_int, c_int, POINTER(c_int)]),
    "eb_profile_ops": (c_int, [c_void_p, c_int, c_int, c_void_p, c_int]),
    "eb_profile_ops_repeat": (c_int, [c_void_p, c_int, c_int, c_void_p, c_int, c_int]),
    "eb_decode_request2": (c_int, [c_char_p, c_uint64, c_void_p, c_int, c_float, c_void_p, c_int,
                                   POINTER(c_int), POINTER(c_uint64), POINTER(c_uint64)]),
    "eb_render_prediction": (c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p, c_int,
                                     c_void_p, c_void_p, c_void_p, c_void_p, c_uint64,
                                     POINTER(c_uint64)]),
    "eb_decode_request": (c_int, [c_char_p, c_uint64, c_void_p, c_int, c_void_p, c_int,
                                  POINTER(c_int), POINTER(c_uint64), POINTER(c_uint64)]),
    "eb_k_preprocess_f32": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int64, c_void_p, c_void_p,
                                    c_int, c_void_p]),
    "eb_k_preprocess_u8_nhwc8": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int64, c_void_p,
                                         c_void_p]),
    "eb_k_conv": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_int, c_void_p, c_void_p,
                          c_void_p, c_int, c_void_p, c_int, c_int, c_int, c_int, c_int, c_int,
                          c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int,
                          c_void_p, c_void_p, c_void_p, c_void_p]),
    "eb_k_conv_maxpool2": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_int, c_void_p,
                                   c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_int, c_int,
                                   c_int, c_int, c_void_p]),
    "eb_k_preprocess_u8_layout": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_void_p, c_int,
                                          c_int, c_int, c_int, c_int, c_int, c_void_p, c_void_p]),
    "eb_k_stem_layout": (c_int, [c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int,
                                 POINTER(c_uint64)]),
    "eb_k_stem_relayout": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_int, c_int, c_int,
                                   c_int, c_int, c_void_p, c_void_p]),
    "eb_k_resize": (c_int, [c_void_p, c_int, c_void_p, c_int, c_int, c_int, c_int, c_int, c_int,
                            c_int, c_void_p]),
    "eb_k_pool": (c_int, [c_void_p, c_int, c_void_p, c_int, c_int, c_int, c_int, c_int, c_int,
                          c_int, c_int, c_int, c_int, c_void_p, c_void_p, c_void_p]),
    "eb_k_gap": (c_int, [c_void_p, c_int, c_void_p, c_int, c_int, c_int, c_void_p, c_void_p,
                         c_void_p]),
    "eb_k_lin1": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_int64,
                          c_int, c_void_p]),
    "eb_k_combine": (c_int, [c_void_p, c_int, c_void_p, c_int, c_void_p, c_void_p, c_void_p,
                             c_int, c_int, c_void_p, c_int, c_void_p, c_void_p, c_int, c_int,
                             c_void_p, c_void_p]),
}

EXPORTED = tuple(_SIGS)

_lock = threading.Lock()
_lib = None


def load(path: str | os.PathLike | None = None):
    """Load (once) and return the native library.  Raises if it is absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        # EB_LIB_PATH: load another build of the library (A/B timing experiments only)
        override = os.environ.get("EB_LIB_PATH")
        p = Path(path) if path else Path(override) if override else LIB_PATH
        if not p.exists():
            raise ImportError(
                f"native library {p} is missing: run `python -m paper_2003_01538_b200.build` "
                "(there is no CPU fallback)"
            )
        lib = ctypes.CDLL(str(p))
        for name, (res, args) in _SIGS.items():
            if override and not hasattr(lib, name):
                continue
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def last_error() -> str:
    msg = load().eb_last_error()
    return msg.decode("utf-8", "replace") if msg else ""


def check(status: int) -> None:
    if status != EB_OK:
        raise EbError(status, last_error())
