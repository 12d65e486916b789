"""Host many-call API throughput: python tools/many_bench.py DIM N REPS"""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_1407_7737_b200 as rb
dim, n, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
eng = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=n, seed=0))
x = np.random.default_rng(0).uniform(-100, 100, (n, dim))
calls = [(fn, p) for p in ("double", "single") for fn in eng.enabled_ids]
eng.evaluate_many(calls, x)
t0 = time.perf_counter()
for _ in range(reps):
    eng.evaluate_many(calls, x)
dt = (time.perf_counter() - t0) / reps
print(f"{len(calls) * n / dt / 1e6:.1f} M evals/s, {dt * 1e3:.0f} ms per suite step")
