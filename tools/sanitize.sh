#!/bin/bash
# compute-sanitizer over one launch per kernel family (tools/sanitize_one.py),
# each tool, plus the generic (non-specialised) kernels and the
# large-dimension kernel forced (RB_BIG=1); logs under gpurun_out/.
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 0 --print-limit 50 \
      python tools/sanitize_one.py > gpurun_out/sanitize_$tool.txt 2>&1
  RB_SPEC=0 timeout 1200 compute-sanitizer --tool $tool --error-exitcode 0 --print-limit 50 \
      python tools/sanitize_one.py > gpurun_out/sanitize_${tool}_generic.txt 2>&1
  RB_BIG=1 timeout 1200 compute-sanitizer --tool $tool --error-exitcode 0 --print-limit 50 \
      python tools/sanitize_one.py > gpurun_out/sanitize_${tool}_bigdim.txt 2>&1
done
tail -n 3 gpurun_out/sanitize_*.txt
