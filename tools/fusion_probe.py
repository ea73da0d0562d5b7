"""A fused kernel vs the unfused launches it replaces: engines built with the fusion on and
off side by side (ENV=1 / ENV=0), per-op serialised profiles taken alternately (the
power-capped clock drifts), launch counts and the summed time of the listed ops.

    python tools/fusion_probe.py EB_STEM_POOL resnet50:3,densenet121:2 [B]
    python tools/fusion_probe.py EB_BLOCK1 vgg16:4 [B]
"""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
from paper_2003_01538_b200 import _lib  # noqa: E402
from paper_2003_01538_b200.ensemble import engine_for  # noqa: E402

env = sys.argv[1]
members = [(m.split(":")[0], int(m.split(":")[1])) for m in sys.argv[2].split(",")]
B = int(sys.argv[3]) if len(sys.argv) > 3 else 256
kind = _lib.EB_IN_U8_HWC
engs = {}
for flag in ("1", "0"):
    os.environ[env] = flag
    engs[flag] = engine_for(bench.build_ensemble(B, 0, members=members))
x = np.random.randint(0, 256, (B, 224 * 224 * 3), dtype=np.uint8)
res = {f: [] for f in engs}
for e in engs.values():
    e.forward(x, kind)
for _ in range(5):
    for f, e in engs.items():
        res[f].append(e.profile(B, kind, repeat=5))
for f, e in engs.items():
    ms = np.median(np.stack(res[f]), axis=0)
    kinds = [m.get("name") or m.get("kind") for m in e.op_meta]
    print(f"{env}={f}: launches {e.launch_count(kind, B)}, all ops {float(ms.sum()):.3f} ms; "
          f"largest ops {[(i, kinds[i], round(float(ms[i]), 3)) for i in np.argsort(-ms)[:4]]}", flush=True)
