#!/bin/bash
# BASELINE.json configs 1-5 on one GPU (under gpurun): peaks microbenchmark,
# one bench line per config (with its CPU baselines: all cores over
# min(N, 20000) rows and one pinned core), the reference arm; then
# tools/configs_report.py TAG assembles profiles/r02/configs.json.
# usage: bash tools/run_configs.sh TAG
TAG=${1:-cfg}
mkdir -p gpurun_out profiles/r02
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/peaks tools/peaks_microbench.cu && \
  /tmp/peaks > gpurun_out/peaks_$TAG.json && cp gpurun_out/peaks_$TAG.json profiles/r02/peaks.json
timeout 900 python bench.py --config 1 --steps 400 --warmup 20 --cpu-rows-1core 1000 \
    > gpurun_out/cfg1_$TAG.json 2> gpurun_out/cfg1_$TAG.err
for c in 2 3 4; do
  timeout 1200 python bench.py --config $c --steps 5 --warmup 3 --cpu-rows-1core 20000 \
      --breakdown gpurun_out/cfg${c}_breakdown_$TAG.json > gpurun_out/cfg${c}_$TAG.json 2> gpurun_out/cfg${c}_$TAG.err
done
timeout 1500 python bench.py --config 5 --steps 5 --warmup 3 --cpu-rows-1core 2000 --e2e-numpy \
    --breakdown gpurun_out/cfg5_breakdown_$TAG.json > gpurun_out/cfg5_$TAG.json 2> gpurun_out/cfg5_$TAG.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_$TAG.json 2>&1
