"""Per-op profile of C5 (ResNet-152, DenseNet-201, VGG-19, Inception-v3 @299, ResNeXt-50)
at B = 128 per GPU: per-member serialised time and the slowest layers (TF/s)."""
import collections
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2003_01538_b200 import _lib, synth  # noqa: E402
from paper_2003_01538_b200.ensemble import engine_for  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
members = [("resnet152", 6), ("densenet201", 7), ("vgg19", 8), ("inception_v3", 5), ("resnext50_32x4d", 9)]
ens = bench.build_ensemble(B, 0, members=members)
eng = engine_for(ens)
px = synth.images_fast(B, 299, 299, 3, seed0=77)
eng.forward(px, _lib.EB_IN_U8_HWC)
ms = np.median(np.stack([eng.profile(B, _lib.EB_IN_U8_HWC, repeat=5) for _ in range(3)]), axis=0)
lanes = collections.defaultdict(float)
rows = []
for m, t in zip(eng.op_meta, ms):
    lanes[m.get("lane")] += float(t)
    f = m.get("flops", 0) * B
    rows.append((float(t), m.get("name"), m.get("shape"), m.get("lane"), f / t / 1e9 if f and t else 0,
                 m.get("groups", 1)))
print("total ms", round(float(ms.sum()), 3), "per lane", {k: round(v, 3) for k, v in lanes.items()})
for r in sorted(rows, key=lambda r: -r[0])[:40]:
    print(round(r[0], 3), r[1], r[2], "lane", r[3], "TF/s", round(r[4]))
json.dump([{"ms": float(r[0]), "name": r[1], "shape": r[2], "lane": r[3], "tflops": float(r[4])} for r in rows],
          open(ROOT / "gpurun_out" / "c5_profile.json", "w"))
# the bench.py --profile-json format (tools/ops_roofline.py reads it)
json.dump([{"i": i, **{k: (list(v) if isinstance(v, tuple) else v) for k, v in m.items()}, "ms": float(t)}
           for i, (m, t) in enumerate(zip(eng.op_meta, ms))],
          open(ROOT / "gpurun_out" / "c5_per_op_profile.json", "w"), indent=0)
