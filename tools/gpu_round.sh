#!/bin/bash
# One GPU round trip: parity tests, smoke, full bench line, reference arm,
# launch list, and ncu --set full captures of the given (fn, precision) pairs.
# usage (under gpurun): bash tools/gpu_round.sh TAG "FN:PREC FN:PREC ..."
TAG=${1:-r01}; CAPS=${2:-"32:double"}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_$TAG.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1
timeout 1200 python bench.py --breakdown gpurun_out/breakdown_full_$TAG.json \
    > gpurun_out/bench_full_$TAG.txt 2> gpurun_out/bench_full_$TAG.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --rows 1000000 --steps 1 --warmup 1 \
    --no-cpu --no-e2e > /dev/null 2>&1
for c in $CAPS; do
  FN=${c%%:*}; PREC=${c##*:}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:evaluate_kernel -s 1 -c 1 \
      -o gpurun_out/prof_${TAG}_fn${FN}_${PREC} python tools/profile_one.py 100 1000000 $FN $PREC 2 \
      > gpurun_out/ncu_${TAG}_fn${FN}_${PREC}.log 2>&1
done
tail -5 gpurun_out/pytest_$TAG.txt; cat gpurun_out/smoke_$TAG.txt | tail -3
tail -c 3000 gpurun_out/bench_full_$TAG.txt; tail -c 1500 gpurun_out/bench_ref_$TAG.txt
