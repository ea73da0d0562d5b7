"""Time one conv layer through the kernel-level ABI (eb_k_conv) with CUDA events.

    python tools/conv_bench.py B H W CIN COUT KH KW S P [--res] [--iters N]
"""
import argparse
import ctypes
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2003_01538_b200 import _lib  # noqa: E402
from paper_2003_01538_b200.packing import conv_mode, pack_conv_weight  # noqa: E402

ap = argparse.ArgumentParser()
for n in ("B", "H", "W", "CIN", "COUT", "KH", "KW", "S", "P"):
    ap.add_argument(n, type=int)
ap.add_argument("--res", action="store_true")
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--block-n", type=int, default=0)
ap.add_argument("--stem", action="store_true", help="CIN<=8 image in NHWC8 (gather mode)")
ap.add_argument("--pre", action="store_true", help="fused BN-ReLU pre-activation on A")
ap.add_argument("--split", type=int, default=0)
ap.add_argument("--groups", type=int, default=1)
ap.add_argument("--relayout", action="store_true", help="stem: padded rows / planes layout (c8_stem=2)")
ap.add_argument("--pool", action="store_true", help="fused 2x2/2 max-pool (eb_k_conv_maxpool2)")
ap.add_argument("--then-pool", action="store_true", help="conv then a separate eb_k_pool (2x2/2 max)")
ap.add_argument("--graph", action="store_true", help="time a CUDA graph of --iters launches (no host cost)")
a = ap.parse_args()
lib = _lib.load()
P = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
LD = 8 if a.stem else a.CIN
x = torch.randn(a.B, a.H, a.W, LD, device="cuda").to(torch.bfloat16)
w = torch.randn(a.COUT, a.CIN, a.KH, a.KW) * 0.05
wp = pack_conv_weight(w, conv_mode(a.KH, a.KW, a.S, a.S, a.P, a.P, a.CIN, a.stem)).cuda()
Ho = (a.H + 2 * a.P - a.KH) // a.S + 1
Wo = (a.W + 2 * a.P - a.KW) // a.S + 1
y = torch.empty(a.B, Ho, Wo, a.COUT, device="cuda", dtype=torch.bfloat16)
res = torch.randn_like(y) if a.res else None
bias = torch.randn(a.COUT, device="cuda")
ws = torch.empty(2 * 148 * 128 * 256, device="cuda")
kp = (a.CIN + 63) // 64 * 64
pre_s = torch.rand(kp, device="cuda") if a.pre else None
pre_t = torch.rand(kp, device="cuda") if a.pre else None


src = x
if a.relayout:
    nb = ctypes.c_uint64(0)
    _lib.check(lib.eb_k_stem_layout(a.B, a.H, a.W, a.KH, a.KW, a.S, a.S, a.P, a.P, ctypes.byref(nb)))
    src = torch.empty(nb.value // 2, device="cuda", dtype=torch.bfloat16)

    def relayout():
        _lib.check(lib.eb_k_stem_relayout(P(x), a.B, a.H, a.W, a.KH, a.KW, a.S, a.S, a.P, a.P, P(src), None))

    relayout()
    torch.cuda.synchronize()
    r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    r0.record()
    for _ in range(a.iters):
        relayout()
    r1.record()
    torch.cuda.synchronize()
    print(f"relayout {r0.elapsed_time(r1) / a.iters * 1e3:.1f} us")
STEM = 2 if a.relayout else int(a.stem)


if a.pool or a.then_pool:
    yp = torch.empty(a.B, Ho // 2, Wo // 2, a.COUT, device="cuda", dtype=torch.bfloat16)


def stream_arg():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def run():
    if a.pool:
        _lib.check(lib.eb_k_conv_maxpool2(P(src), a.B, a.H, a.W, LD, LD, P(wp), P(bias), P(yp), a.COUT, 0,
                                          a.COUT, a.KH, a.KW, a.P, a.P, 1, stream_arg()))
        return
    _lib.check(lib.eb_k_conv(P(src), a.B, a.H, a.W, LD, LD, P(wp), P(bias), P(res),
                             a.COUT if res is not None else 0, P(y), a.COUT, 0, a.COUT, a.KH, a.KW,
                             a.S, a.S, a.P, a.P, 1, 0, STEM, a.split, a.block_n, a.groups, P(ws), P(pre_s), P(pre_t),
                             stream_arg()))
    if a.then_pool:
        _lib.check(lib.eb_k_pool(P(y), a.COUT, P(yp), a.COUT, 0, a.B, Ho, Wo, a.COUT, 2, 2, 0, 0,
                                 None, None, stream_arg()))


for _ in range(3):
    run()
torch.cuda.synchronize()
if a.graph:
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(a.iters):
            run()
    torch.cuda.synchronize()
    body = run

    def run():  # noqa: F811  (one replay = --iters launches; timed per launch below)
        g.replay()

    a_iters = a.iters
    a.iters = 1
# L2 flush buffer (inputs of the big layers exceed L2 anyway; small ones should not hit)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")
times = []
for _ in range(5):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.iters):
        run()
    e1.record()
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1) / a.iters / (a_iters if a.graph else 1))
ms = sorted(times)[len(times) // 2]  # median of 5 repeats
flops = 2 * a.B * Ho * Wo * a.COUT * a.CIN * a.KH * a.KW
bytes_ = 2 * (x.numel() + y.numel() + (res.numel() if res is not None else 0) + wp.numel())
print(f"{ms*1e3:.1f} us  {flops/ms/1e9:.0f} TFLOP/s  {bytes_/ms/1e6:.0f} GB/s")
