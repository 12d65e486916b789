for v in base l4 w21 base; do
  RB_LIB=paper_1407_7737_b200/variants/lib_$v.so timeout 600 python bench.py --rows 10000000 --steps 2 --warmup 3 --no-cpu --no-e2e --breakdown gpurun_out/abu_$v.json > gpurun_out/abu_$v.txt 2>/dev/null
  python - $v <<'PY'
import json, sys
v = sys.argv[1]
d = json.load(open(f"gpurun_out/abu_{v}.json"))
r = {(x["fn"], x["precision"]): x["evals_per_s"] / 1e6 for x in d["rows"]}
l = [x for x in open(f"gpurun_out/abu_{v}.txt") if x.startswith("{")][-1]
j = json.loads(l)
pp = j["per_precision_evals_per_s"]
print(v, "suite", round(j["value"] / 1e6, 1), "f64", round(pp["double"] / 1e6, 1), "f32", round(pp["single"] / 1e6, 1),
      "f64", [round(r[(f, "double")]) for f in (0, 8, 20)], "f32", [round(r[(f, "single")]) for f in (0, 8, 20)], "comp f64", [round(r[(f, "double")]) for f in (29, 32, 35)])
PY
done
