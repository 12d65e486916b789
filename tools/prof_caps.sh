mkdir -p gpurun_out
for c in $CAPS; do
  FN=${c%%:*}; PREC=${c##*:}
  REP=gpurun_out/prof_${TAG}_fn${FN}_${PREC}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:evaluate_kernel -s 1 -c 1 \
      -o $REP python tools/profile_one.py 100 1000000 $FN $PREC 2 > gpurun_out/ncu_${TAG}_fn${FN}_${PREC}.log 2>&1
  python tools/ncu_summary.py $REP.ncu-rep > gpurun_out/ncu_full_${TAG}_fn${FN}_${PREC}.txt 2>&1
  python tools/ncu_lines2.py $REP.ncu-rep 31250 40 > gpurun_out/ncu_lines_${TAG}_fn${FN}_${PREC}.txt 2>&1
  python tools/ncu_sass_top.py $REP.ncu-rep 40 > gpurun_out/ncu_sass_${TAG}_fn${FN}_${PREC}.txt 2>&1
done
rm -f gpurun_out/*.ncu-rep
