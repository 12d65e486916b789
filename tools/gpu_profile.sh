#!/bin/bash
# ncu --set full captures of chosen (fn, precision) launches at D=100,
# N=1e6 (one launch each), with summaries and per-line hot spots.
# usage (under gpurun): bash tools/gpu_profile.sh TAG "FN:PREC ..."
TAG=${1:-p}; CAPS=${2:-"0:double"}
mkdir -p gpurun_out
for c in $CAPS; do
  FN=${c%%:*}; PREC=${c##*:}
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:evaluate_kernel -s 1 -c 1 \
      -o gpurun_out/prof_${TAG}_fn${FN}_${PREC} python tools/profile_one.py 100 1000000 $FN $PREC 2 \
      > gpurun_out/ncu_${TAG}_fn${FN}_${PREC}.log 2>&1
  python tools/ncu_summary.py gpurun_out/prof_${TAG}_fn${FN}_${PREC}.ncu-rep > gpurun_out/ncu_full_${TAG}_fn${FN}_${PREC}.txt 2>&1
  python tools/ncu_lines2.py gpurun_out/prof_${TAG}_fn${FN}_${PREC}.ncu-rep 31250 40 > gpurun_out/ncu_lines_${TAG}_fn${FN}_${PREC}.txt 2>&1
done
