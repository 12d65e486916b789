"""Engines coexisting in one process, and dimensions past the shared-memory
tile: the reference lets any number of engines of any dims live side by side
(engine.py:144-159, 225-228) and has no dimension cap (engine.py:42-44)."""

import numpy as np
import pytest

from tests.conftest import cuda_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

import paper_1407_7737_b200 as rb  # noqa: E402
from oracle.robench_oracle import Oracle, population  # noqa: E402


def _check(eng, orc, fns, n=24):
    x = population(eng.dim, n, seed=3)
    for fn in fns:
        for prec, rel, ab in (("double", 1e-12, 1e-10), ("single", 1e-5, 0.0)):
            got = eng.evaluate(fn, x, precision=prec).values.astype(np.float64)
            want = orc.evaluate(fn, x, prec).astype(np.float64)
            assert np.all(np.abs(got - want) <= np.maximum(rel * np.abs(want), ab)), (eng.dim, fn, prec)


def test_smaller_engine_created_later_does_not_shrink_the_first():
    # the per-kernel dynamic shared-memory limit is process-wide: a dim-10
    # engine built after a dim-100 one must not lower it
    big = rb.initialize(rb.EngineConfig(dim=100, max_concurrency=64, seed=0))
    small = rb.initialize(rb.EngineConfig(dim=10, max_concurrency=64, seed=0))
    fns = (0, 8, 20, 21, 24, 29, 32, 36)
    _check(big, Oracle(100, 0), fns)
    _check(small, Oracle(10, 0), fns)
    small.dispose()
    _check(big, Oracle(100, 0), fns)
    big.dispose()


def test_dimension_past_the_tile_serves_every_function():
    # float64 compositions stop fitting the shared-memory tile first
    # (D ~ 400); they move to the large-dimension kernel (tiles in global
    # scratch, rb_device.cuh evaluate_big_kernel) and nothing is refused
    dim = 420
    eng = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=16, seed=0))
    orc = Oracle(dim, 0)
    x = population(dim, 8, seed=1)
    served = []
    for fn in eng.enabled_ids:
        for prec in ("double", "single"):
            got = eng.evaluate(fn, x, precision=prec).values.astype(np.float64)
            want = orc.evaluate(fn, x, prec).astype(np.float64)
            rel, ab = (1e-12, 1e-10) if prec == "double" else (1e-5, 0.0)
            assert np.all(np.abs(got - want) <= np.maximum(rel * np.abs(want), ab)), (fn, prec)
            served.append((fn, prec))
    eng.dispose()
    assert len(served) == 2 * len(eng.enabled_ids)


@pytest.mark.parametrize("dim", [10, 30, 100])
def test_near_optimum_rows_take_the_exact_order_pass(dim):
    # float64 HappyCat / HGBat members next to their optimum: the main kernel
    # marks the rows, the fixup pass re-evaluates them with NumPy-order z
    # (rb_device.cuh exact64_kernel); host arrays and device tensors, batch
    # and single rows agree bit for bit, and meet the bar
    import torch
    from paper_1407_7737_b200 import _lib, instances
    eng = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=4096, seed=4))
    orc = Oracle(dim, 4)
    rng = np.random.default_rng(dim)
    for fn in (20, 21, 24, 26, 27, 28, 30, 32, 33, 34, 35, 36):
        inst = instances.build(fn, dim, 4)
        optima = [m.shift for m in inst.members] if hasattr(inst, "members") else [inst.shift]
        rows = [rng.uniform(-100, 100, dim)]
        for o in optima:
            o = np.asarray(o, dtype=np.float64)
            rows += [o, o + 1e-12 * rng.standard_normal(dim), o + 1e-9 * rng.standard_normal(dim),
                     o + 1e-6 * rng.standard_normal(dim)]
        x = np.vstack(rows + [rng.uniform(-100, 100, (40, dim))])
        want = orc.evaluate(fn, x, "double")
        n0 = _lib.launch_count()
        host = eng.evaluate(fn, x).values
        dev = eng.evaluate(fn, torch.from_numpy(x).cuda()).values.cpu().numpy()
        assert np.array_equal(host, dev), fn
        assert np.all(np.abs(host - want) <= np.maximum(1e-12 * np.abs(want), 1e-10)), \
            (dim, fn, np.max(np.abs(host - want)))
        for i in (1, 2, 3):
            assert eng.evaluate(fn, x[i:i + 1]).values[0] == host[i], (fn, i)
        assert _lib.launch_count() - n0 >= 3          # main kernel + fixup passes ran
    eng.dispose()


def test_host_pipeline_chunks_match_the_device_path():
    # rb_h_func_evaluate[f] / _x64 pipeline rows in ~32 MB chunks (41 943
    # rows at D=100): a 3-chunk batch equals the device-tensor evaluation bit
    # for bit in both precisions (float32 from float64 rows = the host cast
    # of engine.py:201); a NaN in the last chunk raises; a HappyCat optimum in
    # the second chunk takes the fixup pass
    import torch
    from paper_1407_7737_b200 import instances
    dim, n = 100, 100_003
    eng = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=n, seed=0))
    x = population(dim, n, seed=9)
    x[50_000] = instances.build(20, dim, 0).shift
    xt = torch.from_numpy(x).cuda()
    for fn in (0, 20, 33):
        for prec in ("double", "single"):
            host = eng.evaluate(fn, x, precision=prec).values
            dev = eng.evaluate(fn, xt, precision=prec).values.cpu().numpy()
            assert host.dtype == (np.float64 if prec == "double" else np.float32)
            assert np.array_equal(host, dev), (fn, prec)
    x32 = x.astype(np.float32)
    assert np.array_equal(eng.evaluate(8, x32, precision="single").values,
                          eng.evaluate(8, x, precision="single").values)
    assert eng.evaluate(20, x).values[50_000] == 100.0
    bad = x.copy()
    bad[n - 2, 7] = np.nan
    for prec in ("double", "single"):
        with pytest.raises(rb.NonFiniteInput):
            eng.evaluate(0, bad, precision=prec)
    eng.dispose()


def test_host_evaluate_many_matches_single_calls():
    # one host population, many functions: rows uploaded once per chunk
    # (rb_h_func_evaluate_many; ~128 MB chunks = 167 772 rows at D=100: 2 chunks)
    dim, n = 100, 200_003
    eng = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=n, seed=1))
    x = population(dim, n, seed=3)
    from paper_1407_7737_b200 import instances
    x[180_000] = instances.build(21, dim, 1).shift         # an exact-order fixup row (chunk 2)
    calls = [(fn, p) for p in ("double", "single") for fn in (0, 8, 21, 24, 33)]
    res = eng.evaluate_many(calls, x)
    for (fn, p), r in zip(calls, res):
        assert np.array_equal(r.values, eng.evaluate(fn, x, precision=p).values), (fn, p)
    assert res[2].values[180_000] == 100.0
    bad = x.copy()
    bad[n - 1, 0] = np.inf
    with pytest.raises(rb.NonFiniteInput):
        eng.evaluate_many(calls, bad)
    with pytest.raises(rb.UnknownFunction):
        eng.evaluate_many([(0, "double"), (99, "single")], x)
    eng.dispose()


def test_two_engines_from_threads_share_the_staging_pool():
    # the host pipeline's worker pool is process-wide: engines of different
    # dims called from several threads at once give the single-thread values
    import threading
    engs = [rb.initialize(rb.EngineConfig(dim=d, max_concurrency=200_000, seed=1)) for d in (30, 100)]
    xs = [population(d, 150_000, seed=d) for d in (30, 100)]
    want = [[e.evaluate(fn, x, precision=p).values for fn in (0, 21, 33) for p in ("double", "single")]
            for e, x in zip(engs, xs)]
    got, errs = [None, None, None, None], []

    def run(i):
        try:
            e, x = engs[i % 2], xs[i % 2]
            got[i] = [e.evaluate(fn, x, precision=p).values for fn in (0, 21, 33) for p in ("double", "single")]
        except Exception as ex:           # pragma: no cover - reported below
            errs.append(ex)

    ts = [threading.Thread(target=run, args=(i,)) for i in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for i in range(4):
        for a, b in zip(got[i], want[i % 2]):
            assert np.array_equal(a, b)
    for e in engs:
        e.dispose()


def test_many_call_fork_keeps_stream_order_and_values():
    # rb_func_evaluate_many runs short calls with disjoint outputs on two
    # streams (forked from the caller's and joined back): the values equal
    # one call at a time, and work queued after it on the caller's stream
    # sees every value; overlapping outputs keep one stream (last call wins)
    import torch
    dim, n = 30, 5000
    eng = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=n, seed=1))
    x = torch.from_numpy(population(dim, n, seed=11)).cuda()
    x32 = x.float()
    calls = [(fn, p) for p in ("double", "single") for fn in eng.enabled_ids]
    batches = {"double": x, "single": x32}
    outs = [torch.full((n,), float("nan"), dtype=batches[p].dtype, device="cuda") for _, p in calls]
    eng.evaluate_many(calls, batches, outs=outs)
    sums = torch.stack([o.double().sum() for o in outs])          # queued behind the join
    for (fn, p), o in zip(calls, outs):
        want = eng.evaluate(fn, batches[p], p).values
        assert torch.equal(o, want), (fn, p)
    assert torch.isfinite(sums).all()
    shared = torch.empty(n, dtype=torch.float64, device="cuda")
    pend = eng.evaluate_many([(0, "double"), (8, "double"), (29, "double")], x, outs=[shared] * 3)
    pend[-1].result()
    assert torch.equal(shared, eng.evaluate(29, x, "double").values)
    # an output inside a later call's input: not forked, calls stay in order
    # (call 0 writes column 0 of the buffer call 1 then reads)
    buf = x.clone()
    col0 = torch.empty(n, dtype=torch.float64, device="cuda")
    ref = eng.evaluate(3, x, "double").values
    ins = [x, buf]
    outs2 = [buf.view(-1)[:n], col0]
    eng.evaluate_many([(3, "double"), (0, "double")], ins, outs=outs2)[1].result()
    after = x.clone().view(-1)
    after[:n] = ref
    assert torch.equal(col0, eng.evaluate(0, after.view(n, dim), "double").values)
    eng.dispose()
