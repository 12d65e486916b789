"""Small-batch latency breakdown (BASELINE config 1: sphere, D=10, N=1000).

    python tools/latency_probe.py [--dim 10] [--n 1000] [--fn 0] [--calls 400]

Prints, per path, microseconds per evaluation:
  enqueue_async   host time to queue one evaluate_async call (Python + native)
  enqueue_native  host time per call inside ONE rb_func_evaluate_many of K calls
  device_async    device time per call, K async calls queued (CUDA events)
  device_many     device time per call, K calls in one native call (one output)
  device_many_distinct  the same with a distinct output per call (two streams)
  blocking_dev    Engine.evaluate on a CUDA tensor (blocking, status read)
  blocking_numpy  Engine.evaluate on a NumPy array (H2D + kernel + D2H)
Run the same command under ncu (--metrics gpu__time_duration.sum) for the
kernel's own duration."""

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
import paper_1407_7737_b200 as rb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, default=10)
    ap.add_argument("--n", type=int, default=1000)
    ap.add_argument("--fn", type=int, default=0)
    ap.add_argument("--prec", default="double")
    ap.add_argument("--calls", type=int, default=512)
    ap.add_argument("--k", type=int, default=64)
    args = ap.parse_args()
    eng = rb.initialize(rb.EngineConfig(dim=args.dim, max_concurrency=args.n, seed=0))
    dt = torch.float64 if args.prec == "double" else torch.float32
    xh = np.random.default_rng(0).uniform(-100, 100, (args.n, args.dim))
    xd = torch.from_numpy(xh).to("cuda", dt)
    out = torch.empty(args.n, dtype=dt, device="cuda")
    fn, p, K = args.fn, args.prec, args.k
    res = {}
    for _ in range(20):
        eng.evaluate(fn, xd, p)
    torch.cuda.synchronize()

    def timed(queue):
        enq, dev = [], []
        for _ in range(max(1, args.calls // K)):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            s.record()
            t0 = time.perf_counter()
            pend = queue()
            t1 = time.perf_counter()
            e.record()
            for q in pend:
                q.result()
            enq.append((t1 - t0) / K * 1e6)
            dev.append(s.elapsed_time(e) / K * 1e3)
        return statistics.median(enq), statistics.median(dev)

    res["enqueue_async_us"], res["device_async_us"] = timed(
        lambda: [eng.evaluate_async(fn, xd, p, out=out) for _ in range(K)])
    res["enqueue_native_us"], res["device_many_us"] = timed(
        lambda: eng.evaluate_many([(fn, p)] * K, [xd] * K, outs=[out] * K))
    outs = [torch.empty_like(out) for _ in range(K)]      # distinct outputs: two streams
    res["enqueue_native_distinct_us"], res["device_many_distinct_us"] = timed(
        lambda: eng.evaluate_many([(fn, p)] * K, [xd] * K, outs=outs))

    for name, x in (("blocking_dev_us", xd), ("blocking_numpy_us", xh)):
        ts = []
        for _ in range(args.calls):
            t0 = time.perf_counter()
            eng.evaluate(fn, x, p)
            ts.append((time.perf_counter() - t0) * 1e6)
        res[name] = statistics.median(ts)
    res.update(dim=args.dim, n=args.n, fn=fn, precision=p)
    print(json.dumps(res))
    eng.dispose()


if __name__ == "__main__":
    main()
