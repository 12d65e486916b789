"""Per-source-line warp instructions (per tile) and stall samples from an
ncu report with -lineinfo.  usage: ncu_lines2.py REPORT [tiles] [top]"""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]
tiles = float(sys.argv[2]) if len(sys.argv) > 2 else 31250
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
fname = cur = hdr = None
agg = collections.defaultdict(lambda: [0, 0])
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No":
        hdr = r; continue
    if hdr is None:
        continue
    if len(r) > 2 and r[0].isdigit() and r[2] == "-":
        cur = (fname, int(r[0]), r[1].strip()[:70]); continue
    if len(r) > 7 and r[2].startswith("0x") and cur:
        try:
            agg[cur][0] += int(r[4] or 0); agg[cur][1] += int(r[7] or 0)
        except ValueError:
            pass
ti = sum(v[1] for v in agg.values()); ts = sum(v[0] for v in agg.values()) or 1
print(f"warp instructions per tile {ti / tiles:.0f}; stall samples {ts}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[1] / tiles:8.0f} inst/tile {100 * v[0] / ts:5.1f}% smp  {k[0]}:{k[1]} {k[2]}")
