"""NumPy host-path throughput (rb_h_func_evaluate[_x64]) at one size:
python tools/host_path_bench.py DIM N [FN ...]"""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_1407_7737_b200 as rb
dim, n = int(sys.argv[1]), int(sys.argv[2])
fns = [int(f) for f in sys.argv[3:]] or [0]
eng = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=n, seed=0))
x = np.random.default_rng(0).uniform(-100, 100, (n, dim))
for prec in ("double", "single"):
    eng.evaluate(fns[0], x, prec)
    t0 = time.perf_counter()
    for fn in fns:
        eng.evaluate(fn, x, prec)
    dt = time.perf_counter() - t0
    print(prec, f"{len(fns) * n / dt / 1e6:.1f} M evals/s", f"{len(fns) * x.nbytes / dt / 1e9:.1f} GB/s of float64 X")
