"""Cost of the first call at a new batch size (graph capture + instantiate) vs a cached one."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
from paper_2003_01538_b200 import _lib  # noqa: E402
from paper_2003_01538_b200.ensemble import engine_for  # noqa: E402

eng = engine_for(bench.build_ensemble(512, 0))
kind = _lib.EB_IN_U8_HWC
x = np.random.randint(0, 256, (512, 224 * 224 * 3), dtype=np.uint8)
eng.forward(x[:1], kind)
for b in (37, 101, 250, 37, 101, 250, 300):
    t0 = time.perf_counter()
    eng.forward(x[:b], kind)
    print(b, "%.1f ms" % ((time.perf_counter() - t0) * 1e3))
