"""Wall-clock anatomy of the end-to-end paths at B=256 (C2)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
from paper_2003_01538_b200 import _lib, synth  # noqa: E402
from paper_2003_01538_b200.ensemble import engine_for  # noqa: E402

B, K = 256, 20
eng = engine_for(bench.build_ensemble(B, 0))
kind = _lib.EB_IN_U8_HWC
h1 = torch.from_numpy(synth.images_fast(B, 224, 224, 3, seed0=1)).pin_memory().numpy()
h2 = torch.from_numpy(synth.images_fast(B, 224, 224, 3, seed0=2)).pin_memory().numpy()
xs = [h1 if i % 2 == 0 else h2 for i in range(K)]
for _ in range(3):
    eng.forward(h1, kind)
eng.forward_batches(xs[:2], kind)


res = {}


def t(fn, name):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    res.setdefault(name, []).append((time.perf_counter() - t0) / K * 1e3)


for rep in range(3):  # interleaved: under the power cap later runs would see lower clocks
    t(lambda: [eng.forward_device(B, kind) for _ in range(K)], "forward_device (no copies)")
    t(lambda: [eng.forward(x, kind) for x in xs], "forward (H2D+fwd+D2H per call)")
    t(lambda: eng.forward_batches(xs, kind), "forward_batches (pipelined)")
for name, v in res.items():
    dt = sorted(v)[1]
    print(f"{name:40s} median {dt:.3f} ms/step  {B / dt * 1e3:.0f} img/s   {[round(x, 3) for x in v]}")
