"""Device-timed C2 images/s at a few batch sizes (the bench's sweep), for env A/B runs:
    EB_PDL_MAX_BATCH=64 python tools/sweep_probe.py 16 32 64 128"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
from paper_2003_01538_b200 import _lib, synth  # noqa: E402
from paper_2003_01538_b200.ensemble import engine_for  # noqa: E402

bs = [int(a) for a in sys.argv[1:]] or [8, 32, 64, 128]
ens = bench.build_ensemble(max(bs), 0)
eng = engine_for(ens)
stream = torch.cuda.ExternalStream(eng.stream())
eng.forward(synth.images_fast(max(bs), 224, 224, 3, seed0=3), _lib.EB_IN_U8_HWC)
print(" ".join(f"B={b}:{bench.device_rate(eng, b, _lib.EB_IN_U8_HWC, stream, 5, iters=20):.0f}" for b in bs))
