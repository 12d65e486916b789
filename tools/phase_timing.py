"""Per-phase clock split of the evaluation kernels (needs a library built
with -DRB_PHASE_TIMING, e.g. tools/variants.sh phase "-DRB_PHASE_TIMING",
then RB_LIB=paper_1407_7737_b200/variants/lib_phase.so).
usage: phase_timing.py DIM N FN[,FN..] [PREC]"""
import sys
import torch
sys.path.insert(0, ".")
import paper_1407_7737_b200 as rb
from paper_1407_7737_b200 import _lib

dim, n = int(sys.argv[1]), int(sys.argv[2])
fns = [int(f) for f in sys.argv[3].split(",")]
precs = sys.argv[4].split(",") if len(sys.argv) > 4 else ["double", "single"]
eng = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=n, seed=0))
g = torch.Generator(device="cuda")
g.manual_seed(1)
x64 = torch.rand((n, dim), dtype=torch.float64, device="cuda", generator=g) * 200 - 100
xs = {"double": x64, "single": x64.float()}
for prec in precs:
    for fn in fns:
        eng.evaluate(fn, xs[prec], prec)
        torch.cuda.synchronize()
        _lib.debug_phases(prec, reset=True)
        eng.evaluate(fn, xs[prec], prec)
        torch.cuda.synchronize()
        ph = _lib.debug_phases(prec, reset=True)
        tiles = max(ph[4], 1)
        load, stage, kern, tot, _, wts = (ph[i] / tiles for i in range(6))
        other = tot - load - stage - kern - wts
        print(f"fn {fn:2d} {prec:6s} clk/tile/CTA {tot:8.0f}: load {load:7.0f} ({100*load/tot:4.1f}%)  "
              f"z-stage {stage:7.0f} ({100*stage/tot:4.1f}%)  kernel {kern:7.0f} ({100*kern/tot:4.1f}%)  "
              f"weights {wts:7.0f} ({100*wts/tot:4.1f}%)  other {other:7.0f} ({100*other/tot:4.1f}%)")
eng.dispose()
