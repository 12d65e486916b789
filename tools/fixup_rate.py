"""Throughput when every row is next to an optimum (late-stage optimizer
populations): float64 HappyCat / HGBat rows are then all marked and
re-evaluated in exact order by fixup_kernel.
    python tools/fixup_rate.py [DIM] [N]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
import paper_1407_7737_b200 as rb  # noqa: E402
from paper_1407_7737_b200 import instances  # noqa: E402

dim = int(sys.argv[1]) if len(sys.argv) > 1 else 100
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
eng = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=n, seed=0))
rng = np.random.default_rng(0)
for fn in (20, 21, 28, 32):
    inst = instances.build(fn, dim, 0)
    o = np.asarray(inst.shift if hasattr(inst, "shift") else inst.members[1].shift)
    near = torch.from_numpy(o + 1e-9 * rng.standard_normal((n, dim))).cuda()
    rand = torch.from_numpy(rng.uniform(-100, 100, (n, dim))).cuda()
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    res = {}
    for name, x in (("random", rand), ("near_optimum", near)):
        for _ in range(2):
            eng.evaluate_async(fn, x, "double", out=out).result()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(3):
            p = eng.evaluate_async(fn, x, "double", out=out)
        e.record()
        p.result()
        res[name] = n * 3 / (s.elapsed_time(e) / 1e3) / 1e6
    print(f"fn {fn} D={dim} N={n}: random {res['random']:.1f} M evals/s, "
          f"all rows near the optimum {res['near_optimum']:.1f} M evals/s")
