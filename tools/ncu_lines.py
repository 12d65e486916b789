"""Per-source-line stall samples and executed instructions from an ncu report
(needs -lineinfo).  usage: ncu_lines.py REPORT [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr, rows = "?", None, []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0].isdigit() and len(r) > 5 and r[2] == "-":
        samp = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        inst = int(r[hdr.index("Instructions Executed")] or 0)
        rows.append((samp, inst, f"{fname}:{r[0]}", r[1].strip()[:80]))
ts = sum(r[0] for r in rows) or 1
ti = sum(r[1] for r in rows) or 1
print(f"samples {ts}, warp instructions {ti}")
for s, i, loc, src in sorted(rows, reverse=True)[:top]:
    print(f"{100 * s / ts:5.1f}% smp {100 * i / ti:5.1f}% inst  {loc:22s} {src}")
