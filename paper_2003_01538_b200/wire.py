"""F1: native fast path for ``/v1/predict`` request bodies (eg/wire.py:76-109).

``fast_decode`` hands the body to ``eb_decode_request`` (csrc/wire_decode.cpp), which
base64-decodes every f32le sample in parallel straight into a (pinned, per-thread)
host buffer that ``eb_forward`` then copies to the device.  It returns ``None`` for
anything outside the well-formed f32le case; callers then run the reference's own
``decode_request``, so every error keeps the reference's exact type and message.
"""

from __future__ import annotations

import ctypes
import threading
from ctypes import byref, c_int, c_uint64

import numpy as np

from . import _lib

_tls = threading.local()


def _buffer(n_floats: int, pinned: bool) -> np.ndarray:
    buf = getattr(_tls, "buf", None)
    if buf is None or buf.size < n_floats or getattr(_tls, "pinned", None) != pinned:
        if pinned:
            import torch

            t = torch.empty(n_floats, dtype=torch.float32, pin_memory=True)
            _tls.tensor = t  # keep the pinned allocation alive
            buf = t.numpy()
        else:
            buf = np.empty(n_floats, dtype=np.float32)
        _tls.buf, _tls.pinned = buf, pinned
    return buf


def fast_decode(body: bytes, dims, max_batch: int, pinned: bool = True, pixel_scale: float = 0.0):
    """(data (B, D) float32 view, policy bytes or None), or None when not accepted.
    pixel_scale > 0 also accepts "pgm" samples for a [1, H, W] shape."""
    lib = _lib.load()
    dims = tuple(int(d) for d in dims)
    d = int(np.prod(dims))
    out = _buffer(max_batch * d, pinned)
    dims_arr = (ctypes.c_int32 * len(dims))(*dims)
    n = c_int(0)
    poff, plen = c_uint64(0), c_uint64(0)
    rc = lib.eb_decode_request2(body, len(body), dims_arr, len(dims), float(pixel_scale),
                                out.ctypes.data, max_batch, byref(n), byref(poff), byref(plen))
    if rc != _lib.EB_OK:
        return None
    data = out[: n.value * d].reshape(n.value, d)
    policy = body[poff.value: poff.value + plen.value] if plen.value else None
    return data, policy
