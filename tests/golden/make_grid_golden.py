"""Golden landscape grids from the live reference (scalar_evaluator, the
engine of ``robench grid``, cli.py:72-91): fixtures for tests/test_fileio.py.
Run here (needs /root/reference): python tests/golden/make_grid_golden.py"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from robench.engine import scalar_evaluator  # noqa: E402

FNS = (0, 8, 14, 20, 29, 31, 33)
STEPS, LO, HI, SEED = 7, -100.0, 100.0, 3

out = {}
nodes = np.linspace(LO, HI, STEPS)
for fn in FNS:
    ev = scalar_evaluator(fn, 2, SEED)
    vals = np.empty((STEPS, STEPS))
    for i in range(STEPS):
        for j in range(STEPS):
            vals[i, j] = ev(np.array([nodes[i], nodes[j]]))
    out[f"grid/{fn}"] = vals
out["meta"] = np.array([STEPS, LO, HI, SEED])
np.savez(Path(__file__).with_name("grid.npz"), fns=np.array(FNS), **out)
print("wrote", len(FNS), "grids")
