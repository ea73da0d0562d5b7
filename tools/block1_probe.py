"""Fused VGG block 1 vs the unfused pair: per-op serialised profile of a VGG-16-only
ensemble at B (default 256), EB_BLOCK1=1 and 0 engines built side by side and profiled
alternately (the power-capped clock drifts); launch counts."""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
from paper_2003_01538_b200 import _lib  # noqa: E402
from paper_2003_01538_b200.ensemble import engine_for  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
kind = _lib.EB_IN_U8_HWC
engs = {}
for flag in ("1", "0"):
    os.environ["EB_BLOCK1"] = flag
    engs[flag] = engine_for(bench.build_ensemble(B, 0, members=[("vgg16", 4)]))
x = np.random.randint(0, 256, (B, 224 * 224 * 3), dtype=np.uint8)
res = {f: [] for f in engs}
for f, e in engs.items():
    e.forward(x, kind)
for _ in range(5):
    for f, e in engs.items():
        res[f].append(e.profile(B, kind, repeat=5))
for f, e in engs.items():
    ms = np.median(np.stack(res[f]), axis=0)
    print(f"EB_BLOCK1={f}: launches {e.launch_count(kind, B)}, first ops (ms) "
          f"{[round(float(t), 3) for t in ms[:4]]}, block 1 {float(ms[:3].sum()):.3f} ms, "
          f"all ops {float(ms.sum()):.3f} ms", flush=True)
