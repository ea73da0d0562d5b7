"""One fused VGG block-1 forward at B (default 256) for ncu (-k regex:block1)."""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
os.environ.setdefault("EB_BLOCK1", "1")
import bench  # noqa: E402
from paper_2003_01538_b200 import _lib  # noqa: E402
from paper_2003_01538_b200.ensemble import engine_for  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
eng = engine_for(bench.build_ensemble(B, 0, members=[("vgg16", 4)]))
x = np.random.randint(0, 256, (B, 224 * 224 * 3), dtype=np.uint8)
eng.profile(B, _lib.EB_IN_U8_HWC)
