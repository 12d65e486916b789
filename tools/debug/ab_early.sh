for v in cur early cur early; do
  RB_LIB=paper_1407_7737_b200/variants/lib_$v.so timeout 600 python bench.py --config 1 --steps 400 --warmup 20 --no-cpu > gpurun_out/c1_$v.json 2>/dev/null
  RB_LIB=paper_1407_7737_b200/variants/lib_$v.so python tools/latency_probe.py --calls 512 --k 64 > gpurun_out/lp_$v.json 2>/dev/null
  python -c "
import json; l=[x for x in open('gpurun_out/c1_$v.json') if x.startswith('{')][-1]; d=json.loads(l); g=d['latency']['graph']; lp=json.load(open('gpurun_out/lp_$v.json'))
print('$v', 'c1 value', round(d['value']/1e6,1), 'graph dev us', round(g['device_us_per_call_median'],2), 'probe many dev', round(lp['device_many_us'],2), 'blocking', round(lp['blocking_dev_us'],1))"
done
AB_EXTRA="--config 2" bash tools/ab.sh e2 0 cur early 2>&1 | grep -E "^==|total"
bash tools/ab.sh e5 10000000 cur early 2>&1 | grep -E "^==|total"
RB_LIB=paper_1407_7737_b200/variants/lib_early.so timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -1
