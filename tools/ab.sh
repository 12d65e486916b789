#!/bin/bash
# A/B the library variants built by tools/variants.sh (under gpurun).
#   bash tools/ab.sh TAG N name1 name2 ...
TAG=$1; N=$2; shift 2
mkdir -p gpurun_out
for v in "$@"; do
  RB_LIB=paper_1407_7737_b200/variants/lib_$v.so timeout 600 python bench.py --rows $N --steps 2 --warmup 1 $AB_EXTRA \
     --no-cpu --no-e2e --breakdown gpurun_out/ab_${TAG}_$v.json > gpurun_out/ab_${TAG}_$v.txt 2>&1
  echo "== $v"; python tools/show_breakdown.py gpurun_out/ab_${TAG}_$v.json
done
