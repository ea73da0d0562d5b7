"""Per-op roofline of a bench.py per-op profile (profiles/*/bench_per_op_profile.json).

For every conv / FC launch: the tensor bound (algorithmic flops / the sustained bf16 peak)
and the HBM bound (input read once + output written once + residual read + weights, over
the measured copy bandwidth); an op's bound is the larger of the two.  Prints the ops that
lose the most time against their bound, the loss by member and layer class, and two
whole-step lower bounds:
  * sum of per-op bounds (ops serialised, each at its own roofline), and
  * max(total flops / peak, total bytes / HBM) (perfect overlap of compute- and
    memory-bound ops across the members' lanes).
Non-conv ops (pool, GAP, ...) count at their measured time in both.

    python tools/ops_roofline.py profiles/round2/bench_per_op_profile.json [B] [--burst]
        [--names=ResNet-50,DenseNet-121,VGG-16]   (member name of each lane; default C2's)

The tensor bound uses the sustained bf16 peak of MEASURED_PEAKS.json (what a long step
sees, as bench.py's roofline does); --burst uses the burst peak instead (each op of the
profile runs only 5 times back to back, so its compute-bound ops can exceed the sustained
figure -- VGG-16's 28x28 / 56x56 convs do).
"""
import collections
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
ops = json.load(open(sys.argv[1]))  # (first positional argument)
argv = [a for a in sys.argv[1:] if not a.startswith("--")]
B = int(argv[1]) if len(argv) > 1 else 256  # the profile's flops are per image
peaks = json.load(open(ROOT / "MEASURED_PEAKS.json")) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
TC = (peaks.get("bf16_tflops", 1616.7) if "--burst" in sys.argv
      else peaks.get("bf16_tflops_sustained", 1363.1)) * 1e12
HBM = peaks.get("hbm_gbs", 6536.4) * 1e9
_names = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--names=")),
              "ResNet-50,DenseNet-121,VGG-16")
LANES = dict(enumerate(_names.split(",")))

sys.path.insert(0, str(ROOT))
from bench import op_bounds  # noqa: E402  (the same bound bench.py reports)

bounds = op_bounds(ops, [o["ms"] for o in ops], B, TC / 1e12, HBM / 1e9)
rows = [dict(o=r["meta"], ms=r["ms"], tc=r["tensor_ms"], hbm=r["hbm_ms"], bound=r["bound_ms"]) for r in bounds]
other_ms = sum(o["ms"] for o in ops if o.get("name") != "conv")
tot_flops = sum(r["o"]["flops"] * B for r in rows)
tot_bytes = sum(r["bytes"] for r in bounds)

conv_ms = sum(r["ms"] for r in rows)
sum_bound = sum(r["bound"] for r in rows)
overlap_bound = max(tot_flops / TC, tot_bytes / HBM) * 1e3
print(f"tensor peak {TC / 1e12:.1f} TF/s, HBM {HBM / 1e9:.0f} GB/s")
print(f"B = {B}: {len(rows)} conv/FC launches, {conv_ms:.3f} ms serialised (+ {other_ms:.3f} ms other ops)")
print(f"  sum of per-op bounds        {sum_bound:.3f} ms  -> conv class at {sum_bound / conv_ms:.2f} of its per-op roofline")
print(f"  whole-step overlap bound    {overlap_bound:.3f} ms  (flops {tot_flops / 1e12:.2f} T, bytes {tot_bytes / 1e9:.2f} GB)")
print(f"  step lower bounds incl. other ops: {sum_bound + other_ms:.3f} ms (serialised), "
      f"{overlap_bound + other_ms:.3f} ms (overlapped)")
print("\nloss against the per-op bound by member and class:")
cls = collections.defaultdict(lambda: [0, 0.0, 0.0])
for r in rows:
    ho, wo, co, kh, kw, s, ci = r["o"]["shape"]
    k = (LANES.get(r["o"]["lane"], r["o"]["lane"]), f"{ho}x{wo}", f"{kh}x{kw}/{s}")
    cls[k][0] += 1
    cls[k][1] += r["ms"]
    cls[k][2] += r["bound"]
for k, v in sorted(cls.items(), key=lambda kv: -(kv[1][1] - kv[1][2])):
    print(f"  {k[0]:13s} {k[1]:>7s} {k[2]:7s} n={v[0]:3d}  {v[1]:.3f} ms  bound {v[2]:.3f}  "
          f"frac {v[2] / v[1]:.2f}  loss {v[1] - v[2]:.3f}")
print("\ntop single launches by loss:")
for r in sorted(rows, key=lambda r: -(r["ms"] - r["bound"]))[:int(argv[2]) if len(argv) > 2 else 12]:
    o = r["o"]
    print(f"  op {o['i']:3d} {LANES.get(o['lane'], o['lane']):13s} {str(o['shape']):32s} {r['ms']:.3f} ms  "
          f"tensor {r['tc']:.3f}  hbm {r['hbm']:.3f}  frac {r['bound'] / r['ms']:.2f}")
