#!/bin/bash
# Build tuning variants of the library side by side (here, on CPU):
#   bash tools/variants.sh NAME "-DKNOB=VAL ..." [NAME "-D..."]...
cd "$(dirname "$0")/../paper_1407_7737_b200" && mkdir -p variants
while [ $# -ge 2 ]; do
  python build.py --out "variants/lib_$1.so" $2 || exit 1
  shift 2
done
