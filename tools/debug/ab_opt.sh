# A/B: composition optima staged in shared memory (RB_OPT_SMEM bits) -- breakdown per fn
for m in 3 2 0 3; do
  RB_OPT_SMEM=$m timeout 600 python bench.py --rows 10000000 --steps 2 --warmup 3 --no-cpu --no-e2e --breakdown gpurun_out/abopt_$m.json > gpurun_out/abopt_$m.txt 2>/dev/null
  python - $m <<'PY'
import json, sys
m = sys.argv[1]
d = json.load(open(f"gpurun_out/abopt_{m}.json"))
r = {(x["fn"], x["precision"]): x["evals_per_s"] / 1e6 for x in d["rows"]}
l = [x for x in open(f"gpurun_out/abopt_{m}.txt") if x.startswith("{")][-1]
v = json.loads(l)["value"] / 1e6
print(m, "suite", round(v, 1), "comp f64", [round(r[(f, "double")]) for f in range(29, 37)],
      "comp f32", [round(r[(f, "single")]) for f in range(29, 37)])
PY
done
