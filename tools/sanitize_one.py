"""One small launch of every kernel family, for compute-sanitizer
(tools/sanitize.sh): basic (fn 0, 20 with its fixup pass, 8), hybrid-spec
(24), composition-spec (32, 36), the generic kernel (RB_SPEC=0 run), both
precisions; the async path, a captured graph, the host pipeline, the sharded P2P-store gather
and the on-device population source."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
import paper_1407_7737_b200 as rb  # noqa: E402
from paper_1407_7737_b200 import instances  # noqa: E402
from paper_1407_7737_b200.dist import MultiDeviceEngine  # noqa: E402
from paper_1407_7737_b200.population import uniform_population, workload_entropy  # noqa: E402

dim, n = 30, 70
eng = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=256, seed=0))
x = np.random.default_rng(1).uniform(-100, 100, (n, dim))
x[3] = instances.build(20, dim, 0).shift            # marked row -> fixup_kernel
for fn in (0, 8, 20, 24, 32, 36):
    for prec in ("double", "single"):
        eng.evaluate(fn, x, precision=prec)
xt = torch.from_numpy(x).cuda()
for p in [eng.evaluate_async(fn, xt, "double") for fn in (20, 33)]:
    p.result()
cap = eng.capture(20, xt, "double")                 # CUDA graph: reset, kernel, fixup
cap.launch().result()
cap.close()
multi = MultiDeviceEngine(rb.EngineConfig(dim=dim, max_concurrency=256, seed=0), [0, 0])
multi.evaluate(29, [xt[:35], xt[35:]], "double")
multi.dispose()
uniform_population(dim, 33, workload_entropy(dim, 33), device=0, dtypes=("double", "single"))
torch.cuda.synchronize()
eng.dispose()
print("sanitize_one ok")
