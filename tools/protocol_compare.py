"""Side-by-side of two protocol reports (paper_1407_7737_b200.protocol TSV
vs the reference's `robench bench` TSV): batch ns/eval and the speed-up per
(fn, dim), geometric mean per dimension.
usage: protocol_compare.py OURS.tsv REFERENCE.tsv"""
import csv
import math
import sys
from collections import defaultdict


def load(path):
    with open(path) as fh:
        return {(int(r["fn"]), int(r["dim"])): r for r in csv.DictReader(fh, delimiter="\t")}


ours, ref = load(sys.argv[1]), load(sys.argv[2])
per_dim = defaultdict(list)
print("fn\tdim\tprecision\tgpu_batch_ns_per_eval\tref_batch_ns_per_eval\tspeedup")
for key in sorted(ours):
    if key not in ref:
        continue
    g, c = float(ours[key]["batch_ns_per_eval"]), float(ref[key]["batch_ns_per_eval"])
    per_dim[key[1]].append(c / g)
    print(f"{key[0]}\t{key[1]}\t{ours[key]['precision']}\t{g:.1f}\t{c:.1f}\t{c / g:.1f}")
for d, v in sorted(per_dim.items()):
    print(f"# dim {d}: geometric-mean speed-up {math.exp(sum(map(math.log, v)) / len(v)):.1f}x "
          f"over {len(v)} functions")
