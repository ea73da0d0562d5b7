"""Summarise a per-op profile JSON written by bench.py --profile-json (optionally vs another)."""
import collections
import json
import sys

BATCH = 256  # profile flops are per image
KIND = {0: "conv", 1: "pool", 2: "bnrelu", 3: "gap", 4: "lin1", 5: "resize"}


def agg(path):
    d = collections.OrderedDict()
    for x in json.load(open(path)):
        k = (KIND.get(x.get("kind"), "?"), tuple(x.get("shape") or []), x.get("lane"))
        a = d.setdefault(k, [0, 0.0, 0])
        a[0] += 1
        a[1] += x["ms"]
        a[2] += x.get("flops", 0)
    return d


new = agg(sys.argv[1])
old = agg(sys.argv[2]) if len(sys.argv) > 2 else {}
lanes = collections.defaultdict(float)
for k, v in new.items():
    lanes[k[2]] += v[1]
print("total ms %.3f  by lane %s" % (sum(v[1] for v in new.values()), {k: round(v, 3) for k, v in lanes.items()}))
for k, v in sorted(new.items(), key=lambda kv: -kv[1][1])[:int(sys.argv[3]) if len(sys.argv) > 3 else 40]:
    o = old.get(k, [0, 0.0, 0])[1]
    tf = BATCH * v[2] / (v[1] * 1e-3) / 1e12 if v[1] else 0
    print(f"{k[0]:6s} lane{k[2]} {str(k[1]):36s} n={v[0]:2d} ms={v[1]:.3f} old={o:.3f} TF/s={tf:6.0f}")
