"""Summarise an EB_TRACE dump: per-role event intervals (SM clock cycles) of CTA 0."""
import collections
import sys

ev = collections.defaultdict(list)
spans = []
for line in open(sys.argv[1]):
    f = list(map(int, line.split()))
    if f[0] == 3:  # CTA span: cta, entry, prologue done, exit (global ns)
        spans.append(f[1:])
        continue
    r, tag, clk, ns = f
    ev[r].append((tag, clk))
if spans:
    t0 = min(s[1] for s in spans)
    q = lambda v: (min(v), sorted(v)[len(v) // 2], max(v))  # noqa: E731
    print(f"CTAs {len(spans)}: entry +ns min/med/max {q([s[1] - t0 for s in spans])}")
    print(f"   prologue ns {q([s[2] - s[1] for s in spans])}  body ns {q([s[3] - s[2] for s in spans])}")
    print(f"   exit +ns {q([s[3] - t0 for s in spans])}")
if not ev:
    sys.exit(0)
t0 = min(v[0][1] for v in ev.values())
names = {0: "producer", 1: "mma", 2: "epilogue(w2)"}
for r in sorted(ev):
    e = ev[r]
    print(f"{names[r]}: {len(e)} events, span {e[-1][1] - e[0][1]} clk, first at +{e[0][1] - t0}")
    # mean delta between consecutive events by (tag_prev, tag_next)
    d = collections.defaultdict(list)
    for (a, ca), (b, cb) in zip(e, e[1:]):
        d[(a, b)].append(cb - ca)
    for k, v in sorted(d.items()):
        v2 = sorted(v)
        print(f"   {k}: n={len(v)} mean={sum(v)/len(v):.0f} med={v2[len(v2)//2]} p90={v2[int(len(v2)*.9)]}")
if len(sys.argv) > 2:
    n = int(sys.argv[2])
    for r in sorted(ev):
        print(names[r], [(t, c - t0) for t, c in ev[r][:n]])
