#!/bin/bash
# Round-end GPU evidence (under gpurun): parity tests, smoke, the bench line
# (+ per-function breakdown), the reference arm, then tools/gpu_evidence.sh.
# usage: bash tools/gpu_final.sh TAG "FN:PREC ..."
TAG=${1:-r01}; CAPS=${2:-"32:single 32:double"}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_$TAG.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1
timeout 1200 python bench.py --breakdown gpurun_out/breakdown_full_$TAG.json \
    > gpurun_out/bench_full_$TAG.txt 2> gpurun_out/bench_full_$TAG.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.txt 2>&1
bash tools/gpu_evidence.sh $TAG "$CAPS" > /dev/null 2>&1
rm -f gpurun_out/*.ncu-rep
tail -3 gpurun_out/pytest_$TAG.txt; tail -2 gpurun_out/smoke_$TAG.txt
tail -c 3000 gpurun_out/bench_full_$TAG.txt; tail -c 1500 gpurun_out/bench_ref_$TAG.txt
