"""Time one pooling launch through the kernel-level ABI (eb_k_pool) with CUDA events.

    python tools/pool_bench.py B H W C K S P MODE [--pre] [--iters N]
"""
import argparse
import ctypes
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2003_01538_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
for n in ("B", "H", "W", "C", "K", "S", "P", "MODE"):
    ap.add_argument(n, type=int)
ap.add_argument("--pre", action="store_true")
ap.add_argument("--iters", type=int, default=20)
a = ap.parse_args()
lib = _lib.load()
P = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
x = torch.randn(a.B, a.H, a.W, a.C, device="cuda").to(torch.bfloat16)
Ho = (a.H + 2 * a.P - a.K) // a.S + 1
Wo = (a.W + 2 * a.P - a.K) // a.S + 1
y = torch.empty(a.B, Ho, Wo, a.C, device="cuda", dtype=torch.bfloat16)
sc = torch.rand(a.C, device="cuda") if a.pre else None
sh = torch.rand(a.C, device="cuda") if a.pre else None


def run():
    _lib.check(lib.eb_k_pool(P(x), a.C, P(y), a.C, 0, a.B, a.H, a.W, a.C, a.K, a.S, a.P, a.MODE,
                             P(sc), P(sh), None))


for _ in range(3):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.iters):
    run()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.iters
bytes_ = 2 * (x.numel() + y.numel())
print(f"{ms*1e3:.1f} us  {bytes_/ms/1e6:.0f} GB/s (compulsory)")
