"""B = 1 device time of each C2 member alone (its own engine and graph) next to the
three-member ensemble: which lane bounds the single-image latency.

    python tools/bs1_lanes.py [B]
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
from paper_2003_01538_b200 import _lib  # noqa: E402
from paper_2003_01538_b200.ensemble import engine_for  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
kind = _lib.EB_IN_U8_HWC
for label, members in [("ensemble", bench.MEMBERS)] + [(m[0], [m]) for m in bench.MEMBERS]:
    eng = engine_for(bench.build_ensemble(max(B, 8), 0, members=members))
    stream = torch.cuda.ExternalStream(eng.stream())
    ms = 1e3 / bench.device_rate(eng, B, kind, stream, 5, iters=50) * B
    prof = eng.profile(B, kind, repeat=5)
    print(f"{label:12s} B={B}: {ms:.3f} ms device (graph), {len(prof)} ops, "
          f"serialised per-op sum {float(prof.sum()):.3f} ms")
