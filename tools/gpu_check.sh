#!/bin/bash
# GPU round trip: tests, small-N bench breakdown (and optional extra command).
# usage (under gpurun): bash tools/gpu_check.sh TAG [N]
TAG=${1:-run}; N=${2:-1000000}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 > gpurun_out/pytest_$TAG.txt
timeout 600 python bench.py --n $N --steps 2 --warmup 1 --no-cpu --no-e2e \
    --breakdown gpurun_out/breakdown_$TAG.json > gpurun_out/bench_$TAG.txt 2>&1
cat gpurun_out/pytest_$TAG.txt; tail -c 600 gpurun_out/bench_$TAG.txt
