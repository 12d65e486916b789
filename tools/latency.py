"""Per-call latency of small batches (the paper protocol's batch of 50):
host-pointer path, device-tensor path, and the kernel alone (CUDA events).
usage: latency.py [DIM] [BATCH] [FN,FN..]"""
import sys
import time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1407_7737_b200 as rb

dim = int(sys.argv[1]) if len(sys.argv) > 1 else 32
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 50
fns = [int(f) for f in sys.argv[3].split(",")] if len(sys.argv) > 3 else [3, 8, 30]
eng = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=batch, seed=0))
x = np.random.default_rng(0).uniform(-100, 100, (batch, dim))
xt = torch.from_numpy(x).cuda()
out = torch.empty(batch, dtype=torch.float64, device="cuda")
for fn in fns:
    for _ in range(20):
        eng.evaluate(fn, x)
    reps = 200
    t0 = time.perf_counter()
    for _ in range(reps):
        eng.evaluate(fn, x)
    host_us = (time.perf_counter() - t0) / reps * 1e6
    t0 = time.perf_counter()
    for _ in range(reps):
        eng.evaluate(fn, xt, out=out)
    dev_us = (time.perf_counter() - t0) / reps * 1e6
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        eng.evaluate(fn, xt, out=out)
    b.record()
    torch.cuda.synchronize()
    ev_us = a.elapsed_time(b) / reps * 1e3
    print(f"fn {fn:2d} D={dim} batch={batch}: host path {host_us:6.1f} us/call, "
          f"device path {dev_us:6.1f} us/call (events {ev_us:6.1f})")
eng.dispose()
