"""Device images/s of the C2 ensemble at small batches with the fused kernels on / off
(EB_BLOCK1, EB_STEM_POOL): where the runtime should start using them (they compute the
same bits either way, so the threshold may depend on B)."""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
from paper_2003_01538_b200 import _lib  # noqa: E402
from paper_2003_01538_b200.ensemble import engine_for  # noqa: E402

engs = {}
for label, env in (("fused", "1"), ("unfused", "0")):
    os.environ["EB_BLOCK1"] = env
    os.environ["EB_STEM_POOL"] = env
    e = engine_for(bench.build_ensemble(128, 0))
    engs[label] = (e, torch.cuda.ExternalStream(e.stream()))
for b in (8, 10, 12, 16, 19, 24, 32, 48, 64, 128):
    r = {k: bench.device_rate(e, b, _lib.EB_IN_U8_HWC, s, 5, iters=20) for k, (e, s) in engs.items()}
    r2 = {k: bench.device_rate(e, b, _lib.EB_IN_U8_HWC, s, 5, iters=20) for k, (e, s) in engs.items()}
    print(f"B={b:4d}  fused {max(r['fused'], r2['fused']):8.0f}  unfused {max(r['unfused'], r2['unfused']):8.0f} images/s",
          flush=True)
