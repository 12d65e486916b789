"""Top SASS instructions by warp-stall samples from an ncu report, with the
dominant stall reasons and +-context.  usage: ncu_sass_top.py REPORT [top]"""
import csv
import io
import subprocess
import sys

rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
ci = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[ci["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
order = sorted(range(len(data)), key=lambda i: -int(data[i][ci["Warp Stall Sampling (All Samples)"]] or 0))
print(f"total samples {tot}, instructions {len(data)}")
for i in order[:top]:
    r = data[i]
    s = int(r[ci["Warp Stall Sampling (All Samples)"]] or 0)
    reasons = sorted(((int(r[ci[c]] or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
    prev = data[i - 1][ci["Source"]].strip() if i else ""
    print(f"{100 * s / tot:5.1f}% {int(r[ci['Instructions Executed']] or 0):9d}x  [{i:5d}] {r[ci['Source']].strip()[:60]:60s} "
          + " ".join(f"{n}:{v}" for v, n in reasons if v) + f"   <- {prev[:40]}")
