#!/bin/bash
# ncu evidence for one round (under gpurun), small enough to come back
# (< 64 MiB): launch list of a bench step, --set full captures summarised to
# text on the box (.ncu-rep kept only for the first capture).
# usage: bash tools/gpu_evidence.sh TAG "FN:PREC FN:PREC ..."
TAG=${1:-r01}; CAPS=${2:-"32:single"}
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --rows 1000000 --steps 1 --warmup 1 \
    --no-cpu --no-e2e > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_$TAG.csv > gpurun_out/launches_summary_$TAG.txt 2>&1
first=1
for c in $CAPS; do
  FN=${c%%:*}; PREC=${c##*:}
  REP=gpurun_out/prof_${TAG}_fn${FN}_${PREC}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:evaluate_kernel -s 1 -c 1 \
      -o $REP python tools/profile_one.py 100 1000000 $FN $PREC 2 > gpurun_out/ncu_${TAG}_fn${FN}_${PREC}.log 2>&1
  python tools/ncu_summary.py $REP.ncu-rep > gpurun_out/ncu_full_${TAG}_fn${FN}_${PREC}.txt 2>&1
  python tools/ncu_lines2.py $REP.ncu-rep 31250 30 > gpurun_out/ncu_lines_${TAG}_fn${FN}_${PREC}.txt 2>&1
  [ $first = 1 ] || rm -f $REP.ncu-rep
  first=0
done
rm -f gpurun_out/launches_$TAG.csv.gz
ls -la gpurun_out | tail -20
