"""Small-N launches for ncu (config 1/2 latency): DIM N FN PREC REPS"""
import sys
import torch
sys.path.insert(0, ".")
import paper_1407_7737_b200 as rb
dim, n, fn, prec, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], int(sys.argv[5])
eng = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=n, seed=0))
x = torch.rand((n, dim), dtype=torch.float64, device="cuda") * 200 - 100
if prec == "single":
    x = x.float()
for _ in range(reps):
    eng.evaluate(fn, x, prec)
torch.cuda.synchronize()
