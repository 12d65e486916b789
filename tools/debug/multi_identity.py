"""Debug: host path vs device path vs MultiDeviceEngine for every function."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1407_7737_b200 as rb
from paper_1407_7737_b200.dist import MultiDeviceEngine
from oracle.robench_oracle import population
dim, n = 30, 1000
cfg = rb.EngineConfig(dim=dim, max_concurrency=n, seed=2)
one = rb.initialize(cfg)
multi = MultiDeviceEngine(cfg, [0, 0])
x = population(dim, n, seed=5)
xt = torch.from_numpy(x).cuda()
for fn in one.enabled_ids:
    for prec in ("double", "single"):
        host = one.evaluate(fn, x, precision=prec).values
        dev = one.evaluate(fn, xt, precision=prec).values.cpu().numpy()
        dev2 = one.evaluate(fn, xt[500:], precision=prec).values.cpu().numpy()
        outs = [o.cpu().numpy() for o in multi.evaluate(fn, [xt[:500], xt[500:]], prec)]
        msg = []
        if not np.array_equal(host, dev): msg.append(f"host!=dev ({np.sum(host != dev)})")
        if not np.array_equal(host[500:], dev2): msg.append("dev shifted")
        for g, o in enumerate(outs):
            if not np.array_equal(host, o):
                b = np.flatnonzero(host != o)
                msg.append(f"multi[{g}] {len(b)} rows, first {b[0]}: {host[b[0]]!r} vs {o[b[0]]!r}")
        if msg: print(fn, prec, "; ".join(msg))
print("done")
