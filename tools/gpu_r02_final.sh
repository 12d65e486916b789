#!/bin/bash
# Round-2 GPU evidence (under gpurun): parity tests, smoke, BASELINE configs
# 1-5 with CPU baselines and the reference arm (tools/run_configs.sh), the
# driver's default bench line and reference arm, a launch list of one step,
# ncu --set full captures (summary, per-line and per-SASS hot spots) and
# DRAM traffic of the dominant launches.
# usage: bash tools/gpu_r02_final.sh TAG "FN:PREC ..."
TAG=${1:-r02}; CAPS=${2:-"32:single 32:double 0:double 0:single"}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_$TAG.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1
bash tools/run_configs.sh $TAG
timeout 1200 python bench.py --breakdown gpurun_out/breakdown_full_$TAG.json \
    > gpurun_out/bench_full_$TAG.txt 2> gpurun_out/bench_full_$TAG.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --rows 1000000 --steps 1 --warmup 3 \
    --no-cpu --no-e2e > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_$TAG.csv > gpurun_out/launches_summary_$TAG.txt 2>&1
for c in $CAPS; do
  FN=${c%%:*}; PREC=${c##*:}
  REP=gpurun_out/prof_${TAG}_fn${FN}_${PREC}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:evaluate_kernel -s 1 -c 1 \
      -o $REP python tools/profile_one.py 100 1000000 $FN $PREC 2 > gpurun_out/ncu_${TAG}_fn${FN}_${PREC}.log 2>&1
  python tools/ncu_summary.py $REP.ncu-rep > gpurun_out/ncu_full_${TAG}_fn${FN}_${PREC}.txt 2>&1
  python tools/ncu_lines2.py $REP.ncu-rep 31250 30 > gpurun_out/ncu_lines_${TAG}_fn${FN}_${PREC}.txt 2>&1
  python tools/ncu_sass_top.py $REP.ncu-rep 30 > gpurun_out/ncu_sass_${TAG}_fn${FN}_${PREC}.txt 2>&1
done
timeout 900 python tools/traffic.py 32:single 33:single 32:double 33:double 0:double 0:single > gpurun_out/traffic_$TAG.txt 2>&1
cp profiles/r02/ncu_traffic.json gpurun_out/ncu_traffic_$TAG.json 2>/dev/null
rm -f gpurun_out/*.ncu-rep
tail -2 gpurun_out/pytest_$TAG.txt; tail -1 gpurun_out/smoke_$TAG.txt
