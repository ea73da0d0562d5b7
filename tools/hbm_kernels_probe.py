"""Run bench.hbm_kernels once (K1 preprocess variants, K5 combine at B = 256 and 4096):
the command profiled by ncu for profiles/<round>/ncu_k1_k5*."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402

if __name__ == "__main__":
    pk, src = bench.peaks()
    print(json.dumps(bench.hbm_kernels(256, pk["hbm_gbs"], src)))
