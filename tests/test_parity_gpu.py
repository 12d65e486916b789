"""CUDA path vs the CPU oracle (and the reference's golden vectors), through
the public API and the C ABI.  Tolerances (BASELINE.json north_star):
float64 |f - f_ref| <= max(1e-12 |f_ref|, 1e-10); float32 |f - f_ref| <=
1e-5 |f_ref| against the reference evaluated in float32."""

import numpy as np
import pytest

from tests.conftest import cuda_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

import paper_1407_7737_b200 as rb  # noqa: E402
from oracle.robench_oracle import Oracle, population  # noqa: E402

TOL = {"double": (1e-12, 1e-10), "single": (1e-5, 0.0)}


def assert_close(got, want, prec, what=""):
    rel, ab = TOL[prec]
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    bound = np.maximum(rel * np.abs(want), ab)
    bad = np.abs(got - want) > bound
    assert not bad.any(), (what, prec, np.flatnonzero(bad)[:5], got[bad][:5], want[bad][:5])


@pytest.fixture(scope="module", params=[2, 10, 30, 32, 50, 64, 96, 100, 200, 250, 300])
def pair(request):
    dim = request.param
    eng = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=4096, seed=0))
    yield eng, Oracle(dim, 0)
    eng.dispose()


def test_parity_every_function(pair):
    eng, orc = pair
    x = population(eng.dim, 96, seed=0)
    x[-1] *= 9.0           # far point: schwefel's outer branches, tiny composition weights
    for fn in eng.enabled_ids:
        for prec in ("double", "single"):
            got = eng.evaluate(fn, x, precision=prec).values
            want = orc.evaluate(fn, x, prec)
            assert got.dtype == want.dtype
            assert_close(got, want, prec, f"D={eng.dim} fn={fn}")


def test_golden_vectors(golden):
    seed = int(golden["seed"])
    for dim in (2, 10, 13, 30, 50, 100):
        eng = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=64, seed=seed))
        x = golden[f"x/{dim}"]
        for fn in eng.enabled_ids:
            pts = np.vstack([x, golden[f"opt/{dim}/{fn}"][None, :]])
            for prec in ("double", "single"):
                assert_close(eng.evaluate(fn, pts, precision=prec).values,
                             golden[f"f/{dim}/{fn}/{prec}"], prec, f"golden D={dim} fn={fn}")
        eng.dispose()


def test_sphere_at_optimum_is_exactly_bias():
    # test_engine.py:44-47
    from paper_1407_7737_b200 import instances
    eng = rb.initialize(rb.EngineConfig(dim=10, seed=1))
    opt = instances.build(0, 10, 1).shift
    assert eng.evaluate(0, opt[None, :]).values[0] == 100.0
    eng.dispose()


def test_optimum_value_reproduction(golden):
    # acceptance criterion 1 (test_acceptance.py:61-74) on the golden optima
    loose = {15, 16, 23, 25, 26, 27, 28, 30, 31, 32, 33, 34, 35, 36}
    seed = int(golden["seed"])
    for dim in (10, 30, 100):
        eng = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=4, seed=seed))
        for fn in range(37):
            v = eng.evaluate(fn, golden[f"opt/{dim}/{fn}"][None, :]).values[0]
            tol = 3e-4 * dim if fn in loose else 1e-8
            assert abs(v - 100.0) <= tol, (dim, fn, v)
        eng.dispose()


def test_batch_equals_single_point_calls():
    # test_engine.py:73-80 — bit identical regardless of batch / tile position
    eng = rb.initialize(rb.EngineConfig(dim=32, max_concurrency=200, seed=2))
    x = np.random.default_rng(3).uniform(-100, 100, (77, 32))
    for fn in (0, 8, 14, 17, 25, 33, 36):
        for prec in ("double", "single"):
            whole = eng.evaluate(fn, x, precision=prec).values
            shifted = eng.evaluate(fn, x[5:], precision=prec).values
            assert np.array_equal(whole[5:], shifted)
            for i in (0, 31, 32, 76):
                alone = eng.evaluate(fn, x[i:i + 1], precision=prec).values[0]
                assert alone == whole[i]
    eng.dispose()


def test_device_tensor_path_matches_host_path():
    import torch
    eng = rb.initialize(rb.EngineConfig(dim=30, max_concurrency=1000, seed=4))
    x = population(30, 500, seed=4)
    xt = torch.from_numpy(x).cuda()
    for fn in (0, 11, 24, 31):
        for prec in ("double", "single"):
            host = eng.evaluate(fn, x, precision=prec).values
            dev = eng.evaluate(fn, xt, precision=prec).values
            assert dev.is_cuda
            assert np.array_equal(dev.cpu().numpy(), host)
    eng.dispose()


def test_errors_in_reference_order():
    # test_engine.py:109-119, 150-155
    eng = rb.initialize(rb.EngineConfig(dim=10, max_concurrency=50, seed=1))
    with pytest.raises(rb.BatchTooLarge):
        eng.evaluate(0, np.zeros((51, 10)))
    with pytest.raises(rb.DimensionMismatch):
        eng.evaluate(0, np.zeros((2, 9)))
    with pytest.raises(rb.UnknownFunction):
        eng.evaluate(37, np.zeros((1, 10)))
    bad = np.zeros((2, 10))
    bad[1, 3] = np.inf
    with pytest.raises(rb.NonFiniteInput):
        eng.evaluate(0, bad)
    with pytest.raises(rb.NonFiniteInput):
        eng.evaluate(30, bad, precision="single")
    with pytest.raises(ValueError):
        eng.evaluate(0, np.zeros((1, 10)), precision="half")
    # finite x whose transform overflows: the kernels' own check (kernels.py:45-49)
    huge = np.full((1, 10), 1e308)
    with pytest.raises(rb.NonFiniteInput):
        eng.evaluate(16, huge)
    eng.dispose()
    eng.dispose()
    with pytest.raises(rb.UseAfterDispose):
        eng.evaluate(0, np.zeros((1, 10)))
    small = rb.initialize(rb.EngineConfig(dim=2, seed=1))
    assert small.enabled_ids == tuple(range(23))
    with pytest.raises(rb.DisabledFunction):
        small.evaluate(23, np.zeros((1, 2)))
    small.dispose()


def test_large_batch_properties():
    # full-size batch: sampled rows equal the oracle and equal their own
    # single-row evaluation (size-independence)
    import torch
    dim, n = 100, 2_000_000
    eng = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=n, seed=0))
    orc = Oracle(dim, 0)
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    x = torch.rand((n, dim), dtype=torch.float64, device="cuda", generator=g) * 200 - 100
    rows = np.array([0, 1, 31, 32, 33, 999_999, n - 1])
    xs = x[torch.from_numpy(rows).cuda()].cpu().numpy()
    for fn in (0, 8, 23, 29):
        for prec in ("double", "single"):
            xx = x if prec == "double" else x.float()
            full = eng.evaluate(fn, xx, precision=prec).values
            assert torch.isfinite(full).all()
            sub = full[torch.from_numpy(rows).cuda()].cpu().numpy()
            assert_close(sub, orc.evaluate(fn, xs, prec), prec, f"large fn={fn}")
            alone = eng.evaluate(fn, xs, precision=prec).values
            assert np.array_equal(alone, sub)
    eng.dispose()


def test_unaligned_device_rows_take_the_per_row_copy_path():
    # a device view whose base is not 16-byte aligned cannot use the bulk
    # tile copy (Args.tma = 0): same values as the aligned buffer
    import torch
    dim, n = 30, 300
    eng = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=n, seed=5))
    x = population(dim, n, seed=5)
    for prec, tdt in (("double", torch.float64), ("single", torch.float32)):
        flat = torch.empty(n * dim + 1, dtype=tdt, device="cuda")
        flat[1:] = torch.from_numpy(x.reshape(-1)).to(tdt).cuda()
        xu = flat[1:].view(n, dim)
        assert xu.data_ptr() % 16 != 0
        for fn in (0, 8, 26, 34):
            got = eng.evaluate(fn, xu, precision=prec).values.cpu().numpy()
            want = eng.evaluate(fn, x, precision=prec).values
            assert np.array_equal(got, want), (fn, prec)
    eng.dispose()


def test_c_abi_rejects_an_empty_batch():
    # PointBatch(np.zeros((0, 10))) is a ValueError (test_engine.py:120-124):
    # the C ABI answers RB_E_INVALID_ARGUMENT and writes nothing
    import ctypes
    from paper_1407_7737_b200 import _lib
    eng = rb.initialize(rb.EngineConfig(dim=10, max_concurrency=8, seed=1))
    lib = _lib.load()
    f = np.full(1, 7.0)
    x = np.zeros((1, 10))
    st = lib.rb_h_func_evaluate(eng._handle, 0, x.ctypes.data_as(ctypes.c_void_p), 0,
                                f.ctypes.data_as(ctypes.c_void_p))
    assert st == 7 and f[0] == 7.0
    eng.dispose()


def test_concurrent_calls_from_threads():
    # SURVEY.md 8b threading: the engine is immutable after init and
    # evaluate may be called concurrently (host arrays and device tensors on
    # separate streams); results are bit-identical to sequential calls
    import threading
    import torch
    eng = rb.initialize(rb.EngineConfig(dim=30, max_concurrency=2048, seed=6))
    x = population(30, 1500, seed=6)
    fns = (0, 9, 24, 31)
    want = {(fn, p): eng.evaluate(fn, x, precision=p).values for fn in fns for p in ("double", "single")}
    errors = []

    def worker(k):
        try:
            stream = torch.cuda.Stream()
            xt = torch.from_numpy(x).cuda()
            torch.cuda.synchronize()              # xt is read on `stream` below
            for rep in range(6):
                for fn in fns:
                    for p in ("double", "single"):
                        if (rep + k) % 2:
                            got = eng.evaluate(fn, x, precision=p).values
                        else:
                            with torch.cuda.stream(stream):
                                got = eng.evaluate(fn, xt, precision=p).values.cpu().numpy()
                        if not np.array_equal(got, want[(fn, p)]):
                            errors.append((k, rep, fn, p))
        except Exception as exc:          # pragma: no cover - reported below
            errors.append(repr(exc))

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    eng.dispose()
    assert not errors, errors[:5]
