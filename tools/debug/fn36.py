import sys, numpy as np
sys.path.insert(0, ".")
import paper_1407_7737_b200 as rb
from oracle.robench_oracle import Oracle
from tests.test_parity_sweep_gpu import _special_points
dim, seed = 10, 1
eng = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=4096, seed=seed))
orc = Oracle(dim, seed)
x = np.random.default_rng(seed).uniform(-100, 100, (64, dim))
for fn in (29, 30, 33, 34, 35, 36):
    sp, far = _special_points(fn, dim, seed)
    pts = np.vstack([x, sp])
    for prec in ("single", "double"):
        got = eng.evaluate(fn, pts, precision=prec).values
        want = orc.evaluate(fn, pts, prec)
        bad = np.flatnonzero(~np.isclose(got, want, rtol=1e-5, equal_nan=True))
        print(fn, prec, "bad rows", bad[:8], got[bad[:3]], want[bad[:3]])
        one = eng.evaluate(fn, pts[74:75], precision=prec).values
        print("   row 74 alone", one, "in batch", got[74], "want", want[74])
