"""Summarise an EB_TRACE dump: per-role event intervals (SM clock cycles) of CTA 0."""
import collections
import sys

ev = collections.defaultdict(list)
for line in open(sys.argv[1]):
    r, tag, clk, ns = map(int, line.split())
    ev[r].append((tag, clk))
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
