"""Dimensions whose tile does not fit in shared memory (rb_device.cuh
evaluate_big_kernel): the reference has no dimension cap (engine.py:42-44),
so every function is served at any dimension -- past ~400 (float64) the
engine keeps only the plan in shared memory and the X / V / z tiles in
global scratch.  Checked against the oracle at D = 420 and 640 (random and
near-optimum points), and against the shared-memory kernels at small D with
the large-dimension path forced (RB_BIG=1)."""

import os

import numpy as np
import pytest

from tests.conftest import cuda_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

import paper_1407_7737_b200 as rb  # noqa: E402
from oracle.robench_oracle import NonFinite, Oracle, population  # noqa: E402
from tests.test_parity_sweep_gpu import _excess, _optima  # noqa: E402


def _points(fn, dim, seed, n=40):
    x = population(dim, n, seed=5)
    rng = np.random.default_rng(77 + fn)
    extra = []
    for o in _optima(fn, dim, seed)[:2]:
        o = np.asarray(o, dtype=np.float64)
        extra += [o, o + 1e-9 * rng.standard_normal(dim), o + 1e-3 * rng.standard_normal(dim)]
    return np.vstack([x] + extra)


@pytest.mark.parametrize("dim", [420, 640])
def test_every_function_served_past_the_tile(dim):
    seed = 0
    eng = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=4096, seed=seed))
    orc = Oracle(dim, seed)
    bad, report = [], []
    for fn in eng.enabled_ids:
        pts = _points(fn, dim, seed)
        for prec in ("double", "single"):
            got = eng.evaluate(fn, pts, precision=prec).values    # raises if refused
            want = orc.evaluate(fn, pts, prec)
            ex = _excess(got, want, prec)
            report.append(f"D={dim} fn={fn:2d} {prec:6s} worst/bar {ex.max():.3g}")
            if not (ex <= 1.0).all():
                i = int(np.argmax(ex))
                bad.append((fn, prec, i, float(got[i]), float(want[i])))
    eng.dispose()
    print("\n".join(report))
    assert len(report) == 2 * 37
    assert not bad, bad[:10]


@pytest.fixture
def forced_big(monkeypatch):
    monkeypatch.setenv("RB_BIG", "1")
    yield
    monkeypatch.delenv("RB_BIG", raising=False)


@pytest.mark.parametrize("dim", [10, 30, 100])
def test_forced_large_dimension_path_matches_tile_kernels(dim, forced_big):
    # the same functions through both kernels: float32 bit for bit (same
    # NumPy-order arithmetic), float64 within the bar (the large-dimension
    # path evaluates HappyCat / HGBat members in exact order for every row,
    # as the fixup pass does for marked rows); batches spanning several
    # waves of the grid, with a ragged last tile
    big = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=1 << 16, seed=2))
    os.environ.pop("RB_BIG")
    tile = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=1 << 16, seed=2))
    orc = Oracle(dim, 2)
    x = np.random.default_rng(dim).uniform(-100, 100, (20_011, dim))
    for fn in big.enabled_ids:
        a = big.evaluate(fn, x, precision="single").values
        b = tile.evaluate(fn, x, precision="single").values
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), (dim, fn)
        a = big.evaluate(fn, x, precision="double").values
        b = tile.evaluate(fn, x, precision="double").values
        assert (_excess(a, b, "double") <= 1.0).all(), (dim, fn)
        head = x[:64]
        for prec in ("double", "single"):
            assert (_excess(big.evaluate(fn, head, precision=prec).values,
                            orc.evaluate(fn, head, prec), prec) <= 1.0).all(), (dim, fn, prec)
    big.dispose()
    tile.dispose()


def test_large_dimension_path_raises_non_finite_and_serves_async():
    import torch
    dim = 420
    eng = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=4096, seed=0))
    x = population(dim, 100, seed=9)
    bad = x.copy()
    bad[37, 5] = np.nan
    orc = Oracle(dim, 0)
    for fn in (29, 32, 36):                   # compositions: past the tile in both precisions
        for prec in ("double", "single"):
            with pytest.raises(rb.NonFiniteInput):
                eng.evaluate(fn, bad, precision=prec)
            with pytest.raises(NonFinite):
                orc.evaluate(fn, bad, prec)
            dt = torch.float64 if prec == "double" else torch.float32
            xt = torch.from_numpy(x).to("cuda", dt)
            pend = eng.evaluate_async(fn, xt, prec)
            got = pend.result().values.cpu().numpy()
            assert (_excess(got, orc.evaluate(fn, x, prec), prec) <= 1.0).all(), (fn, prec)
    calls = [(fn, p) for fn in (0, 21, 29, 36) for p in ("double", "single")]
    many = eng.evaluate_many(calls, x)
    for (fn, p), r in zip(calls, many):
        assert (_excess(r.values, orc.evaluate(fn, x, p), p) <= 1.0).all(), (fn, p)
    eng.dispose()
