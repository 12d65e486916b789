#!/bin/bash
# Quick GPU round trip: parity tests, N=1e6 breakdown, optional ncu captures.
# usage (under gpurun): bash tools/gpu_quick.sh TAG "FN:PREC ..." [N]
TAG=${1:-q}; CAPS=${2:-""}; N=${3:-1000000}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_$TAG.txt 2>&1
timeout 600 python bench.py --rows $N --steps 2 --warmup 1 --no-cpu --no-e2e \
    --breakdown gpurun_out/breakdown_$TAG.json > gpurun_out/bench_$TAG.txt 2>&1
for c in $CAPS; do
  FN=${c%%:*}; PREC=${c##*:}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:evaluate_kernel -s 1 -c 1 \
      -o gpurun_out/prof_${TAG}_fn${FN}_${PREC} python tools/profile_one.py 100 1000000 $FN $PREC 2 \
      > gpurun_out/ncu_${TAG}_fn${FN}_${PREC}.log 2>&1
done
tail -15 gpurun_out/pytest_$TAG.txt; python tools/show_breakdown.py gpurun_out/breakdown_$TAG.json
