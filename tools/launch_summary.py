"""Summarise an ncu --metrics gpu__time_duration.sum CSV: share per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
for r in rows[hdr_i + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    agg[r[ki]][0] += 1
    agg[r[ki]][1] += v
    tot += v
print(sys.argv[2] if len(sys.argv) > 2 else "")
print(f"{'share%':>7} {'launches':>8} {'total_ms':>10}  kernel")
for t, n, k in sorted(((v[1], v[0], k) for k, v in agg.items()), reverse=True):
    print(f"{100 * t / tot:7.2f} {n:8d} {t / 1e6:10.3f}  {k[:110]}")
