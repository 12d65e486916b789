import sys; sys.path.insert(0, '.')
import numpy as np
import paper_1407_7737_b200 as rb
from paper_1407_7737_b200 import instances
from oracle.robench_oracle import Oracle
g = np.load('tests/golden/values.npz')
for dim in (2, 3, 10):
    eng = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=64, seed=int(g['seed'])))
    orc = Oracle(dim, int(g['seed']))
    for fn in eng.enabled_ids:
        opt = g[f"opt/{dim}/{fn}"][None, :]
        x = np.vstack([g[f"x/{dim}"], opt])
        got = eng.evaluate(fn, x, precision="double").values
        want = orc.evaluate(fn, x, "double")
        err = np.abs(got - want)
        if err.max() > 1e-10:
            print(dim, fn, "maxerr", err.max(), "at", np.argmax(err), got[np.argmax(err)], want[np.argmax(err)])
    eng.dispose()
print("done")
