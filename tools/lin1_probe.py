"""Track R's K6 alone: LIN1 scores for B = 256 at D = 150528, sum K = 6 (3 binary members)
and 3000 (3 x K = 1000), through the kernel-level C-ABI -- the command ncu profiles."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2003_01538_b200 import _lib  # noqa: E402
from paper_2003_01538_b200.models import lin1_splits  # noqa: E402

lib = _lib.load()
P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
B, D = 256, 150528
ns = lin1_splits(D)
x = torch.rand(B, D, device="cuda")
for k in [int(a) for a in (sys.argv[1:] or ["6", "3000"])]:
    w = torch.randn(k, D, device="cuda")
    b = torch.randn(k, device="cuda")
    part = torch.empty(ns * B * k, dtype=torch.float64, device="cuda")
    out = torch.empty(B, k, dtype=torch.float64, device="cuda")
    for _ in range(3):
        _lib.check(lib.eb_k_lin1(P(x), P(w), P(b), P(part), P(out), B, k, D, ns, None))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        _lib.check(lib.eb_k_lin1(P(x), P(w), P(b), P(part), P(out), B, k, D, ns, None))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    byt = 4 * B * D + 4 * k * D
    print(f"sumK={k}: {ms * 1e3:.1f} us, {byt / ms / 1e6:.0f} GB/s, {2 * B * D * k / ms / 1e9:.2f} fp64 TFLOP/s")
