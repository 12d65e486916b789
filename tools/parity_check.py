"""Quick GPU-vs-oracle sweep: prints max relative error per (dim, fn, precision)."""
import sys, time, json
import numpy as np
sys.path.insert(0, ".")
import paper_1407_7737_b200 as rb
from oracle.robench_oracle import Oracle, population

dims = [int(a) for a in sys.argv[1].split(",")] if len(sys.argv) > 1 else [10, 30, 50, 100]
npts = int(sys.argv[2]) if len(sys.argv) > 2 else 200
worst = {}
for dim in dims:
    t0 = time.time()
    eng = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=100000, seed=0))
    orc = Oracle(dim, 0)
    X = population(dim, npts, seed=0)
    for fn in eng.enabled_ids:
        for prec in ("double", "single"):
            got = eng.evaluate(fn, X, precision=prec).values
            want = orc.evaluate(fn, X, prec)
            den = np.maximum(np.abs(want.astype(np.float64)), 1.0 if prec == "double" else 0.0)
            err = np.abs(got.astype(np.float64) - want.astype(np.float64)) / np.where(den == 0, 1, den)
            rel = float(np.max(err))
            nbit = int(np.sum(got != want))
            tol = 1e-12 if prec == "double" else 1e-5
            flag = "" if rel <= tol else "  <-- FAIL"
            print(f"D={dim:3d} fn={fn:2d} {prec:6s} maxrel={rel:.3e} nonbitexact={nbit}/{npts}{flag}", flush=True)
    eng.dispose()
    print(f"dim {dim} done in {time.time()-t0:.1f}s", flush=True)
