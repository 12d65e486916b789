#!/bin/bash
# Full bench line + ncu evidence (launch list, one --set full capture).
# usage (under gpurun): bash tools/gpu_full.sh TAG DOM_FN DOM_PREC
TAG=${1:-r01}; FN=${2:-32}; PREC=${3:-double}
mkdir -p gpurun_out
timeout 1200 python bench.py --breakdown gpurun_out/breakdown_full_$TAG.json > gpurun_out/bench_full_$TAG.txt 2> gpurun_out/bench_full_$TAG.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --n 1000000 --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:evaluate_kernel -s 1 -c 1 \
    -o gpurun_out/prof_${TAG}_fn${FN}_${PREC} python tools/profile_one.py 100 1000000 $FN $PREC 2 > gpurun_out/ncu_${TAG}.log 2>&1
tail -c 3000 gpurun_out/bench_full_$TAG.txt; tail -c 1500 gpurun_out/bench_ref_$TAG.txt
