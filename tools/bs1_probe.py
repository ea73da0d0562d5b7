"""B=1 latency anatomy of the C2 ensemble: device-only graph replay time, e2e eb_forward
time, and the serialised per-op profile (which layers dominate a single-image call)."""
import statistics
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
from paper_2003_01538_b200 import _lib  # noqa: E402

ens = bench.build_ensemble(256, 0)
from paper_2003_01538_b200.ensemble import engine_for  # noqa: E402

eng = engine_for(ens)
kind = _lib.EB_IN_U8_HWC
x = np.random.randint(0, 256, (1, 224 * 224 * 3), dtype=np.uint8)
for _ in range(5):
    eng.forward(x, kind)
lat = []
for _ in range(50):
    t0 = time.perf_counter()
    eng.forward(x, kind)
    lat.append((time.perf_counter() - t0) * 1e3)
print("e2e p50 %.3f ms" % statistics.median(lat))
for _ in range(5):
    eng.forward_device(1, kind)
torch.cuda.synchronize()
s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
st = torch.cuda.ExternalStream(eng.stream_handle()) if hasattr(eng, "stream_handle") else torch.cuda.current_stream()
t0 = time.perf_counter()
for _ in range(50):
    eng.forward_device(1, kind)
torch.cuda.synchronize()
print("device replay (host-timed, 50 back-to-back) %.3f ms" % ((time.perf_counter() - t0) * 1e3 / 50))
ms = eng.profile(1, kind)
lanes = {}
for m, t in zip(eng.op_meta, ms):
    lanes[m.get("lane", -1)] = lanes.get(m.get("lane", -1), 0) + float(t)
print("serialised per-op sum %.3f ms, by lane %s, ops %d" % (sum(map(float, ms)), {k: round(v, 3) for k, v in lanes.items()}, len(ms)))
print("median op %.1f us" % (statistics.median(map(float, ms)) * 1e3))
