"""Run one (fn, precision) evaluation a few times on device-resident data
(for ncu captures).  usage: profile_one.py DIM N FN PREC [REPS]"""
import sys
import torch
sys.path.insert(0, ".")
import paper_1407_7737_b200 as rb

dim, n, fn, prec = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 2
eng = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=n, seed=0))
g = torch.Generator(device="cuda"); g.manual_seed(1)
x = torch.rand((n, dim), dtype=torch.float64, device="cuda", generator=g) * 200 - 100
if prec == "single":
    x = x.float()
for fns in [[int(f) for f in sys.argv[3].split(",")]]:
    for _ in range(reps):
        for f in fns:
            eng.evaluate(f, x, prec)
torch.cuda.synchronize()
eng.dispose()
