"""With a -DRB_DEBUG_FIXUP library: f[0] = -1000 - flag[1] when the fixup
pass did not exit early."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.getcwd())
import paper_1407_7737_b200 as rb
dim, n, fn = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
eng = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=n, seed=0))
x = np.random.default_rng(0).uniform(-100, 100, (n, dim))
xd = torch.from_numpy(x).cuda()
b = eng.evaluate(fn, xd, "double").values
a = eng.evaluate_async(fn, xd, "double").result().values
m = eng.evaluate_many([(fn, "double")], [xd])[0].result().values
print("blocking f0", float(b[0]), "async f0", float(a[0]), "many f0", float(m[0]))
