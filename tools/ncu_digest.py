"""Digest an ncu report: key SOL metrics, then SASS stall samples grouped by execution count.

    python tools/ncu_digest.py REPORT.ncu-rep [top_lines]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 16
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
KEYS = ("Duration", "Throughput", "Busy", "Issue", "Eligible", "Hit Rate", "Pipe", "Warp Cycles",
        "Executed Instructions", "Tensor")
for r in csv.DictReader(io.StringIO(det)):
    n = r["Metric Name"]
    if any(k in n for k in KEYS):
        print(f"{r['Section Name'][:26]:26s} {n[:50]:50s} {r['Metric Unit']:10s} {r['Metric Value']}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr, data = rows[1], rows[2:]
ia = hdr.index("Instructions Executed")
isrc = hdr.index("Source")
iss = hdr.index("Warp Stall Sampling (All Samples)")
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
idx = [hdr.index(h) for h in cols]
groups = collections.defaultdict(lambda: [0, 0, 0, collections.Counter()])
for r in data:
    n = int(r[ia] or 0)
    g = groups[n]
    g[0] += 1
    g[1] += n
    g[2] += int(r[iss] or 0)
    for h, i in zip(cols, idx):
        g[3][h[6:]] += int(r[i] or 0)
print("\nexec-count groups (instrs, total executed, stall samples, top reasons)")
for n, v in sorted(groups.items(), key=lambda kv: -kv[1][2])[:10]:
    print(f"{n:10d} n={v[0]:4d} total={v[1]:11d} samples={v[2]:6d} {v[3].most_common(4)}")
print("\ntop stall lines")
for r in sorted(data, key=lambda r: -int(r[iss] or 0))[:top]:
    reasons = {h[6:]: int(r[i]) for h, i in zip(cols, idx) if int(r[i] or 0) > 20}
    print(r[0][-5:], r[ia], r[iss], r[isrc].strip()[:64], reasons)
