"""Debug: is every function's value independent of the row's tile position?"""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1407_7737_b200 as rb
from oracle.robench_oracle import population
dim = int(sys.argv[1]) if len(sys.argv) > 1 else 30
eng = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=1000, seed=2))
x = population(dim, 1000, seed=5)
for fn in eng.enabled_ids:
    for prec in ("double", "single"):
        whole = eng.evaluate(fn, x, precision=prec).values
        for sh in (500, 5, 1):
            part = eng.evaluate(fn, x[sh:], precision=prec).values
            bad = np.flatnonzero(whole[sh:] != part)
            if len(bad):
                i = bad[0] + sh
                print(f"fn {fn} {prec} shift {sh}: {len(bad)} rows differ, first row {i}: "
                      f"{whole[i]!r} vs {part[i - sh]!r}")
print("done")
