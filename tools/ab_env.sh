#!/bin/bash
# A/B environment knobs of the library (under gpurun):
#   bash tools/ab_env.sh TAG N "NAME:VAR=VAL,VAR=VAL" ...   (NAME:- for defaults)
TAG=$1; N=$2; shift 2
mkdir -p gpurun_out
for spec in "$@"; do
  name=${spec%%:*}; vars=${spec#*:}
  envs=""; [ "$vars" != "-" ] && envs=$(echo "$vars" | tr ',' ' ')
  env $envs timeout 600 python bench.py --rows $N --steps 2 --warmup 1 --no-cpu --no-e2e \
     --breakdown gpurun_out/ab_${TAG}_$name.json > gpurun_out/ab_${TAG}_$name.txt 2>&1
  echo "== $name ($vars)"; python tools/show_breakdown.py gpurun_out/ab_${TAG}_$name.json
done
