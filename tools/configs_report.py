"""Assemble profiles/r02/configs.json from tools/run_configs.sh output:
per BASELINE.json config the device-timed throughput, the end-to-end
throughput through the public API, the roofline fractions (dominant launch
and suite = sum T_roof / sum T), the CPU baselines (all cores over
min(N, 20000) rows; one pinned core), all recomputable from the committed
peaks (profiles/r02/peaks.json, MEASURED_PEAKS.json) and breakdowns."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
tag = sys.argv[1] if len(sys.argv) > 1 else "cfg"
src = ROOT / "gpurun_out"
out = {"peaks": json.loads((ROOT / "profiles" / "r02" / "peaks.json").read_text()),
       "hbm_gbs": json.loads((ROOT / "MEASURED_PEAKS.json").read_text()).get("hbm_gbs"),
       "configs": {}}
for c in range(1, 6):
    f = src / f"cfg{c}_{tag}.json"
    if not f.exists():
        continue
    lines = [ln for ln in f.read_text().splitlines() if ln.startswith("{")]
    if not lines:
        continue
    d = json.loads(lines[-1])
    rec = {k: d.get(k) for k in ("config", "value", "unit", "ms_per_step", "dtype", "e2e", "e2e_pinned_tensor", "e2e_numpy",
                                 "latency", "cpu_baseline", "clocks", "per_precision_evals_per_s")}
    rec["roofline"] = {k: d["roofline"].get(k) for k in ("bound", "achieved", "peak", "unit", "frac",
                                                          "kernel", "suite_frac", "peak_source")}
    bd = src / f"cfg{c}_breakdown_{tag}.json"
    if bd.exists():
        rows = json.loads(bd.read_text())["rows"]
        rec["per_function"] = [{k: r[k] for k in ("fn", "precision", "evals_per_s", "frac",
                                                  "t_roof_hbm", "t_roof_fp", "seconds",
                                                  "rotate_flops_per_eval")} for r in rows]
        dst = ROOT / "profiles" / "r02" / f"breakdown_config{c}.json"
        dst.write_text(bd.read_text())
    if d.get("cpu_baseline"):
        rec["speedup_vs_cpu_all_cores"] = d["value"] / d["cpu_baseline"]["value"]
        if d["cpu_baseline"].get("single_core"):
            rec["speedup_vs_cpu_one_core"] = d["value"] / d["cpu_baseline"]["single_core"]["value"]
    out["configs"][str(c)] = rec
ref = src / f"ref_{tag}.json"
if ref.exists():
    lines = [ln for ln in ref.read_text().splitlines() if ln.startswith("{")]
    if lines:
        out["reference_arm"] = json.loads(lines[-1])
(ROOT / "profiles" / "r02" / "configs.json").write_text(json.dumps(out, indent=1))
for c, r in out["configs"].items():
    print(c, f"{r['value'] / 1e6:9.1f} M/s", "e2e", f"{(r['e2e'] or {}).get('value', 0) / 1e6:8.1f}",
          "frac", round(r["roofline"]["frac"], 3), "suite", round(r["roofline"]["suite_frac"], 3),
          "cpu16", round((r.get("cpu_baseline") or {}).get("value", 0)), "x", round(r.get("speedup_vs_cpu_all_cores", 0)))
