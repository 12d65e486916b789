"""Throughput of the large-dimension path (rb_device.cuh evaluate_big_kernel)
next to the shared-memory kernels.

    python tools/big_dim_bench.py --dims 100,420,640,1000 --rows 200000

Per dimension and precision: every function evaluated on device-resident
rows (evaluate_async into a preallocated output, CUDA events on the
launching stream, 3 warm-up + 5 timed calls per function), reported as
M evals/s and the X-read bandwidth N*D*s / t.  RB_BIG=1 in the environment
forces the large-dimension kernel at every dimension (same-D comparison)."""

import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.getcwd())
import paper_1407_7737_b200 as rb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", default="420,640,1000")
    ap.add_argument("--rows", type=int, default=200_000)
    ap.add_argument("--fns", default="")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    res = []
    for dim in [int(d) for d in args.dims.split(",")]:
        t0 = time.time()
        eng = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=args.rows, seed=0))
        build = time.time() - t0
        g = torch.Generator(device="cuda").manual_seed(dim)
        x64 = (torch.rand(args.rows, dim, device="cuda", dtype=torch.float64, generator=g) * 200 - 100)
        x32 = x64.float()
        fns = [int(f) for f in args.fns.split(",")] if args.fns else list(eng.enabled_ids)
        for prec, x in (("double", x64), ("single", x32)):
            out = torch.empty(args.rows, dtype=x.dtype, device="cuda")
            for fn in fns:
                for _ in range(3):
                    eng.evaluate_async(fn, x, prec, out=out).result()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                s.record()
                for _ in range(5):
                    p = eng.evaluate_async(fn, x, prec, out=out)
                e.record()
                p.result()
                ms = s.elapsed_time(e) / 5
                r = {"dim": dim, "fn": fn, "precision": prec, "ms": round(ms, 4),
                     "M_evals_s": round(args.rows / ms / 1e3, 3),
                     "x_GBs": round(args.rows * dim * x.element_size() / ms / 1e6, 1)}
                res.append(r)
                print(json.dumps(r), flush=True)
        eng.dispose()
        print(json.dumps({"dim": dim, "engine_init_s": round(build, 1)}), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
