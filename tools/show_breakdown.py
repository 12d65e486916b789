"""Print a bench breakdown JSON (per function/precision device time)."""
import json, sys
d = json.load(open(sys.argv[1]))
rows = sorted(d["rows"], key=lambda r: (r["precision"], r["fn"]))
tot = sum(r["seconds"] for r in rows)
for p in ("double", "single"):
    line = []
    for r in rows:
        if r["precision"] == p:
            line.append(f'{r["fn"]}:{r["evals_per_s"]/1e6:.0f}')
    print(p, " ".join(line))
print(f"total {tot*1e3:.1f} ms per step; suite rate {len(rows)*d['n_local']/tot/1e6:.1f} M evals/s")
