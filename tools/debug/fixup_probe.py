"""Which calls run a full fixup pass (rows marked) -- run under ncu
--metrics gpu__time_duration.sum; prints values digest per mode."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.getcwd())
import paper_1407_7737_b200 as rb

dim, n, fn, mode = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
eng = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=n, seed=0))
x = np.random.default_rng(0).uniform(-100, 100, (n, dim))
xd = torch.from_numpy(x).cuda()
out = torch.empty(n, dtype=torch.float64, device="cuda")
for _ in range(3):
    if mode == "blocking":
        v = eng.evaluate(fn, xd, "double").values
    elif mode == "async":
        v = eng.evaluate_async(fn, xd, "double", out=out).result().values
    else:
        v = eng.evaluate(fn, x, "double").values
    torch.cuda.synchronize()
v = v.cpu().numpy() if hasattr(v, "cpu") else v
print(mode, float(np.sum(v)), int(np.sum(np.isnan(v))))
