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


class Renderer:
    """F4: native response bodies (eb_render_prediction) for one ensemble -- the keys'
    sorted order and every label's JSON encoding are prepared once, with the reference's
    own json.dumps(ensure_ascii=True), so the bytes equal
    dumps_canonical(render_prediction(ensemble, output, combined)) (eg/wire.py:136-143)."""

    def __init__(self, ensemble):
        import json

        self.lib = _lib.load()
        models = list(ensemble.models)
        self.n = len(models)
        self._label_bufs, offs = [], []
        for m in models:
            enc = [json.dumps(lab, ensure_ascii=True).encode() for lab in m.labels]
            self._label_bufs.append(ctypes.create_string_buffer(b"".join(enc), sum(map(len, enc)) + 1))
            offs.append(np.concatenate([[0], np.cumsum([len(e) for e in enc])]).astype(np.int64))
        self._offs = offs
        self._label_ptrs = (ctypes.c_char_p * self.n)(*[ctypes.cast(b, ctypes.c_char_p) for b in self._label_bufs])
        self._off_ptrs = (ctypes.c_void_p * self.n)(*[o.ctypes.data for o in offs])
        self._nlab = (ctypes.c_int32 * self.n)(*[len(m.labels) for m in models])
        self._keys = {}
        for with_comb in (False, True):
            entries = [("_batch_size", -1)] + [(m.id, i) for i, m in enumerate(models)]
            if with_comb:
                entries.append(("_combined", -2))
            entries.sort(key=lambda e: e[0])
            kj = [json.dumps(k, ensure_ascii=True).encode() for k, _ in entries]
            self._keys[with_comb] = ((ctypes.c_char_p * len(kj))(*kj),
                                     (ctypes.c_int32 * len(kj))(*[k for _, k in entries]), len(kj), kj)

    def render(self, labels: np.ndarray, combined=None) -> bytes:
        labels = np.ascontiguousarray(labels, dtype=np.int32)
        b = int(labels.shape[1]) if labels.ndim == 2 else 0
        keys, kinds, nk, _ = self._keys[combined is not None]
        comb = None if combined is None else np.ascontiguousarray(np.asarray(combined, dtype=np.int32))
        cap = 64 + b * (self.n + 1) * 32
        for _ in range(2):
            out = ctypes.create_string_buffer(cap)
            n = c_uint64(0)
            rc = self.lib.eb_render_prediction(labels.ctypes.data, self.n, b,
                                               comb.ctypes.data if comb is not None else None,
                                               keys, kinds, nk, self._label_ptrs, self._off_ptrs,
                                               self._nlab, out, cap, byref(n))
            if rc == _lib.EB_OK:
                return out.raw[: n.value]
            if rc != _lib.EB_E_TOO_LARGE:
                _lib.check(rc)
            cap = n.value
        raise RuntimeError("render buffer sizing failed")
