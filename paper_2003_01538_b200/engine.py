"""Python owner of one native engine (include/ensemble_b200.h).

An Engine is built once per loaded ensemble: tensors and ops are declared by the
member lowerings (zoo.py for CNN members, ensemble.py for LIN1 members), weights
are collected into one host staging area and written into the single device
pool at finalize(), and forward() is one native call with host buffers.
"""

from __future__ import annotations

import ctypes
from ctypes import byref, c_int, c_uint64, c_void_p

import numpy as np
import torch

from . import _lib
from ._lib import OpDesc, check

_ALIGN = 256


def _host_bytes(arr) -> np.ndarray:
    if isinstance(arr, torch.Tensor):
        t = arr.detach().cpu().contiguous()
        if t.dtype == torch.bfloat16:
            return t.view(torch.int16).numpy().view(np.uint8).reshape(-1)
        return t.numpy().view(np.uint8).reshape(-1)
    a = np.ascontiguousarray(arr)
    return a.view(np.uint8).reshape(-1)


class TRef:
    """A channel slice of an engine tensor: (id, channel offset, channels, h, w)."""

    __slots__ = ("id", "c_off", "c", "h", "w", "ctot")

    def __init__(self, tid, c_off, c, h, w, ctot):
        self.id, self.c_off, self.c, self.h, self.w, self.ctot = tid, c_off, c, h, w, ctot

    def slice(self, c_off, c):
        return TRef(self.id, self.c_off + c_off, c, self.h, self.w, self.ctot)

    def __repr__(self):
        return f"TRef(id={self.id}, c=[{self.c_off},{self.c_off + self.c}) of {self.ctot}, {self.h}x{self.w})"


class Engine:
    def __init__(self, in_shape, max_batch: int, device: int = 0, precision: str = "bf16"):
        self.lib = _lib.load()
        c, h, w = in_shape
        self.C, self.H, self.W = c, h, w
        self.max_batch = max_batch
        self.device = device
        if precision not in ("bf16", "fp32"):
            raise ValueError(f"precision must be 'bf16' or 'fp32', got {precision!r}")
        self.precision = precision
        self.f32 = precision == "fp32"
        self._h = c_void_p()
        check(self.lib.eb_engine_create(device, max_batch, c, h, w, byref(self._h)))
        if self.f32:  # the fp32-faithful parity mode (csrc/ref32.cu)
            check(self.lib.eb_engine_set_precision(self._h, _lib.EB_PREC_F32))
        self._blobs: list[tuple[int, np.ndarray]] = []
        self._pool_size = 0
        self.members: list[tuple[int, int, int, int]] = []
        self.n_ops = 0
        self.op_meta: list[dict] = []
        self.finalized = False
        self.image = TRef(_lib.EB_T_IMAGE_NHWC8, 0, 8, h, w, 8)
        self.image_f32 = TRef(_lib.EB_T_IMAGE_F32, 0, c, h, w, c)

    # ------------------------------------------------------------ declaration
    def set_preprocess(self, mean, std, lut: np.ndarray):
        m = np.ascontiguousarray(np.asarray(mean, dtype=np.float32))
        s = np.ascontiguousarray(np.asarray(std, dtype=np.float32))
        lut = np.ascontiguousarray(lut, dtype=np.float32)
        check(self.lib.eb_set_preprocess(self._h, m.ctypes.data, s.ctypes.data, m.size,
                                         lut.ctypes.data))

    def weight(self, arr) -> int:
        """Stage a weight blob for the pool; returns its byte offset."""
        b = _host_bytes(arr)
        off = self._pool_size
        self._blobs.append((off, b))
        self._pool_size = (off + b.size + _ALIGN - 1) // _ALIGN * _ALIGN
        return off

    def tensor(self, h, w, c, dtype=None) -> TRef:
        """An activation tensor (bf16, or fp32 in the fp32 mode) unless dtype is given."""
        if dtype is None:
            dtype = _lib.EB_F32 if self.f32 else _lib.EB_BF16
        self._arena_bytes = getattr(self, "_arena_bytes", 0) + self.max_batch * h * w * c * (2, 4, 8)[dtype]
        tid = c_int()
        check(self.lib.eb_tensor(self._h, h, w, c, dtype, byref(tid)))
        return TRef(tid.value, 0, c, h, w, c)

    def op(self, kind, src: TRef, dst: TRef, *, cout=0, res: TRef | None = None, kh=1, kw=1,
           sh=1, sw=1, ph=0, pw=0, relu=0, pool_mode=0, flatten=0, lane=0, w_off=None,
           b_off=None, scale_off=None, shift_off=None, meta: dict | None = None, groups=1,
           prefork=False, dst2: TRef | None = None, n_split=0):
        d = OpDesc()
        d.kind = kind
        d.src, d.dst = src.id, dst.id
        d.res = res.id if res is not None else -1
        d.src_c_off, d.src_c = src.c_off, src.c
        d.dst_c_off, d.cout = dst.c_off, cout
        d.kh, d.kw, d.sh, d.sw, d.ph, d.pw = kh, kw, sh, sw, ph, pw
        d.relu, d.pool_mode, d.flatten, d.stream = int(relu), pool_mode, int(flatten), lane
        d.groups = int(groups)
        d.prefork = int(prefork)
        d.dst2 = dst2.id if dst2 is not None else -1
        d.dst2_c_off = dst2.c_off if dst2 is not None else 0
        d.n_split = int(n_split)
        none = _lib.EB_NO_OFFSET
        d.w_off = none if w_off is None else w_off
        d.b_off = none if b_off is None else b_off
        d.scale_off = none if scale_off is None else scale_off
        d.shift_off = none if shift_off is None else shift_off
        check(self.lib.eb_add_op(self._h, byref(d)))
        self.n_ops += 1
        self.op_meta.append(dict(meta or {}, kind=kind, lane=lane, src=src.id, dst=dst.id,
                                 res=res.id if res is not None else -1))

    def member(self, kind, logits: TRef, k_off: int, k: int):
        check(self.lib.eb_add_member(self._h, kind, logits.id, k_off, k))
        self.members.append((kind, logits.id, k_off, k))

    def finalize(self):
        check(self.lib.eb_pool_reserve(self._h, max(self._pool_size, _ALIGN)))
        for off, b in self._blobs:
            check(self.lib.eb_pool_write(self._h, off, b.ctypes.data, b.size))
        self._blobs = []
        check(self.lib.eb_finalize(self._h))
        self.finalized = True

    @property
    def pool_bytes(self) -> int:
        v = c_uint64()
        check(self.lib.eb_pool_bytes(self._h, byref(v)))
        return v.value

    # ------------------------------------------------------------ execution
    def forward(self, x: np.ndarray, input_kind: int, *, topk: int = 0, policy: int = 0,
                policy_k: int = 0, want_logits: bool = False):
        """One native eb_forward call.  x: (B, C*H*W) f32 or (B, H, W, C) u8, host."""
        b = int(x.shape[0])
        x = np.ascontiguousarray(x)
        n = len(self.members)
        labels = np.empty((n, b), dtype=np.int32)
        kmax = max(m[3] for m in self.members)
        logits = np.zeros((n, b, kmax), dtype=np.float32) if want_logits else None
        tk_i = np.empty((n, b, max(topk, 1)), dtype=np.int32)
        tk_p = np.empty((n, b, max(topk, 1)), dtype=np.float32)
        comb = np.empty(max(b, 1), dtype=np.int32)
        check(self.lib.eb_forward(
            self._h, x.ctypes.data, input_kind, b, labels.ctypes.data,
            logits.ctypes.data if logits is not None else None, topk,
            tk_i.ctypes.data, tk_p.ctypes.data, policy, policy_k, comb.ctypes.data))
        out = {"labels": labels}
        if logits is not None:
            out["logits"] = logits
        if topk:
            out["topk_idx"] = tk_i[:, :, :topk]
            out["topk_prob"] = tk_p[:, :, :topk]
        if policy:
            out["combined"] = comb[:b]
        return out

    def forward_batches(self, xs, input_kind: int) -> list:
        """One native eb_forward_batches call: a pipelined sequence of equal-size host
        batches (each batch's H2D overlaps the previous batch's forward).  Returns the
        labels ([N][B] int32) of every batch."""
        import ctypes

        if not xs:
            return []
        b = int(xs[0].shape[0])
        n = len(self.members)
        arrs = [np.ascontiguousarray(x) for x in xs]
        if any(int(a.shape[0]) != b for a in arrs):
            raise ValueError("eb_forward_batches needs equal batch sizes")
        # pinned label buffers: the device->host copies stay asynchronous, so the host
        # enqueues every batch without waiting on the previous one
        need = len(arrs) * n * b
        if getattr(self, "_pinned_labels", None) is None or self._pinned_labels.numel() < need:
            self._pinned_labels = torch.empty(need, dtype=torch.int32, pin_memory=True)  # reused
        pinned = self._pinned_labels[:need].view(len(arrs), n, b)
        ins = (ctypes.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
        outs = (ctypes.c_void_p * len(arrs))(*[pinned[i].data_ptr() for i in range(len(arrs))])
        check(self.lib.eb_forward_batches(self._h, ins, len(arrs), input_kind, b, outs))
        return [pinned[i].numpy().copy() for i in range(len(arrs))]

    def forward_device(self, batch: int, input_kind: int, topk: int = 0, policy: int = 0,
                       policy_k: int = 0):
        check(self.lib.eb_forward_device(self._h, input_kind, batch, topk, policy, policy_k))

    def input_buffer(self, input_kind: int) -> int:
        p = c_void_p()
        check(self.lib.eb_input_buffer(self._h, input_kind, byref(p)))
        return p.value

    def stream(self) -> int:
        p = c_void_p()
        check(self.lib.eb_engine_stream(self._h, byref(p)))
        return p.value

    def profile(self, batch: int, input_kind: int, repeat: int = 1) -> np.ndarray:
        """Per-op device ms of one serialised eager run; with repeat > 1 each op is
        launched that many times back to back and the mean per launch is returned
        (eb_profile_ops_repeat)."""
        ms = np.zeros(self.n_ops, dtype=np.float32)
        check(self.lib.eb_profile_ops_repeat(self._h, input_kind, batch, ms.ctypes.data,
                                             self.n_ops, repeat))
        return ms

    def launch_count(self, input_kind: int, batch: int) -> int:
        v = c_int()
        check(self.lib.eb_launch_count(self._h, input_kind, batch, byref(v)))
        return v.value

    def tensor_view(self, t: TRef, batch: int) -> torch.Tensor:
        """A torch view of an engine tensor (debugging / parity of intermediates)."""
        p = c_void_p()
        h, w, c, dt = c_int(), c_int(), c_int(), c_int()
        check(self.lib.eb_tensor_ptr(self._h, t.id, byref(p), byref(h), byref(w), byref(c), byref(dt)))
        dtype = {0: torch.bfloat16, 1: torch.float32, 2: torch.float64}[dt.value]
        numel = batch * h.value * w.value * c.value
        t_ = _wrap_device_ptr(p.value, numel, dtype, self.device)
        return t_.view(batch, h.value, w.value, c.value)

    def clone(self) -> "Engine":
        """Another execution context on the same device: shared ops and weight pool, its
        own activation arena, streams and graph cache (eb_engine_clone)."""
        if not self.finalized:
            raise RuntimeError("clone needs a finalized engine")
        c = object.__new__(Engine)
        c.__dict__.update({k: v for k, v in self.__dict__.items()
                           if k not in ("_h", "_pinned_labels", "_blobs")})
        c._blobs = []
        c._h = c_void_p()
        check(self.lib.eb_engine_clone(self._h, byref(c._h)))
        return c

    def warmup(self, input_kind: int, max_b: int = 0) -> None:
        """Capture the graph of every batch-size bucket up to max_b (eb_engine_warmup)."""
        check(self.lib.eb_engine_warmup(self._h, input_kind, max_b))

    @property
    def arena_bytes(self) -> int:
        """Device bytes of this context's activation tensors (max_batch deep)."""
        return getattr(self, "_arena_bytes", 0)

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            self.lib.eb_engine_destroy(self._h)
            self._h = c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _wrap_device_ptr(ptr: int, numel: int, dtype, device: int) -> torch.Tensor:
    """Zero-copy torch view of engine-owned device memory."""
    typestr = {torch.bfloat16: "<i2", torch.float32: "<f4", torch.float64: "<f8",
               torch.uint8: "|u1"}[dtype]

    class _Arr:
        __cuda_array_interface__ = {"shape": (numel,), "typestr": typestr, "data": (ptr, False),
                                    "version": 3}

    t = torch.as_tensor(_Arr(), device=f"cuda:{device}")
    return t.view(torch.bfloat16) if dtype == torch.bfloat16 else t


class ContextPool:
    """Execution contexts of one engine leased per request (F2): the
    reference's gateway re-enters forward from ``workers`` pool threads
    (eg/gateway.py:222-257) and requests stay uncoalesced; with one context
    they serialise on its lock, with n contexts up to n forwards run concurrently on the
    GPU (their own arenas, streams and graphs; shared weights).  Same forward contract as
    Engine."""

    def __init__(self, engine: Engine, n: int):
        import queue

        self.contexts = [engine] + [engine.clone() for _ in range(max(0, n - 1))]
        self._free = queue.Queue()
        for c in self.contexts:
            self._free.put(c)
        first = self.contexts[0]
        self.members, self.max_batch, self.device = first.members, first.max_batch, first.device
        self.op_meta, self.n_ops = first.op_meta, first.n_ops

    def _lease(self, fn):
        ctx = self._free.get()
        try:
            return fn(ctx)
        finally:
            self._free.put(ctx)

    def forward(self, x, input_kind: int, **kw):
        return self._lease(lambda c: c.forward(x, input_kind, **kw))

    def forward_batches(self, xs, input_kind: int):
        return self._lease(lambda c: c.forward_batches(xs, input_kind))

    def warmup(self, input_kind: int, max_b: int = 0) -> None:
        for c in self.contexts:
            c.warmup(input_kind, max_b)

    def __getattr__(self, name):  # device-level helpers (bench, profiling): first context
        return getattr(self.contexts[0], name)

    def close(self):
        for c in self.contexts:
            c.close()
