"""Captured evaluations (Engine.capture -> rb_graph_capture / rb_graph_launch):
a CUDA graph replays one evaluation of the current buffer contents.  The
values must equal the per-call path's, bit for bit, for every replay;
NonFiniteInput is reported per replay (the graph resets its own status
words); float64 HappyCat / HGBat rows next to an optimum get the exact-order
fixup pass inside the graph; the large-dimension kernel captures too."""

import numpy as np
import pytest

from tests.conftest import cuda_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

import paper_1407_7737_b200 as rb  # noqa: E402
from paper_1407_7737_b200 import instances  # noqa: E402


def _same(a, b):
    a = a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)
    b = b.cpu().numpy() if hasattr(b, "cpu") else np.asarray(b)
    return a.dtype == b.dtype and np.array_equal(a.view(np.uint8), b.view(np.uint8))


@pytest.mark.parametrize("prec", ["double", "single"])
@pytest.mark.parametrize("fn", [0, 8, 20, 24, 32])
def test_replays_equal_per_call_values(fn, prec):
    import torch
    dim, n = 30, 1000
    eng = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=n, seed=0))
    dt = torch.float64 if prec == "double" else torch.float32
    rng = np.random.default_rng(fn)
    x = torch.from_numpy(rng.uniform(-100, 100, (n, dim))).to("cuda", dt)
    cap = eng.capture(fn, x, prec)
    for step in range(3):
        x.copy_(torch.from_numpy(rng.uniform(-100, 100, (n, dim))).to(dt))
        got = cap.launch().result().values.clone()
        want = eng.evaluate(fn, x, prec).values
        assert _same(got, want), (fn, prec, step)
    cap.close()
    cap.close()                                  # idempotent
    with pytest.raises(rb.UseAfterDispose):
        cap.launch()
    eng.dispose()


def test_non_finite_status_is_per_replay():
    import torch
    dim, n = 10, 256
    eng = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=n, seed=0))
    x = torch.from_numpy(np.random.default_rng(1).uniform(-100, 100, (n, dim))).cuda()
    for prec in ("double", "single"):
        xs = x if prec == "double" else x.float()
        cap = eng.capture(3, xs, prec)
        cap.launch().result()
        xs[17, 4] = float("nan")
        with pytest.raises(rb.NonFiniteInput):
            cap.launch().result()
        xs[17, 4] = 1.0
        want = eng.evaluate(3, xs, prec).values
        assert _same(cap.launch().result().values, want)
        cap.close()
    eng.dispose()


def test_near_optimum_rows_take_the_fixup_pass_inside_the_graph():
    import torch
    dim, n = 30, 96
    eng = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=n, seed=4))
    for fn in (20, 21, 28):
        inst = instances.build(fn, dim, 4)
        o = np.asarray(inst.shift if hasattr(inst, "shift") else inst.members[0].shift, dtype=np.float64)
        rng = np.random.default_rng(fn)
        rows = np.vstack([o + s * rng.standard_normal((n // 3, dim)) for s in (0.0, 1e-9, 1e-6)])
        x = torch.from_numpy(rows).cuda()
        cap = eng.capture(fn, x, "double")
        got = cap.launch().result().values
        want = eng.evaluate(fn, rows, "double").values
        assert _same(got.cpu().numpy(), want), fn
        cap.close()
    eng.dispose()


def test_capture_validates_like_evaluate():
    import torch
    eng = rb.initialize(rb.EngineConfig(dim=10, max_concurrency=64, seed=0))
    x = torch.zeros((8, 10), dtype=torch.float64, device="cuda")
    with pytest.raises(rb.DimensionMismatch):
        eng.capture(0, torch.zeros((8, 11), dtype=torch.float64, device="cuda"))
    with pytest.raises(rb.BatchTooLarge):
        eng.capture(0, torch.zeros((65, 10), dtype=torch.float64, device="cuda"))
    with pytest.raises(rb.UnknownFunction):
        eng.capture(37, x)
    with pytest.raises(ValueError):
        eng.capture(0, x, "single")        # a float32 copy would not see later updates
    eng.dispose()


def test_large_dimension_kernel_captures(monkeypatch):
    import torch
    monkeypatch.setenv("RB_BIG", "1")
    dim, n = 30, 300
    big = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=n, seed=0))
    monkeypatch.delenv("RB_BIG")
    x = torch.from_numpy(np.random.default_rng(2).uniform(-100, 100, (n, dim))).cuda()
    for fn, prec in ((0, "double"), (29, "single"), (36, "double")):
        xs = x if prec == "double" else x.float()
        cap = big.capture(fn, xs, prec)
        for _ in range(2):
            assert _same(cap.launch().result().values, big.evaluate(fn, xs, prec).values), (fn, prec)
        cap.close()
    big.dispose()


def test_dispose_closes_captures():
    import torch
    eng = rb.initialize(rb.EngineConfig(dim=10, max_concurrency=64, seed=0))
    x = torch.zeros((8, 10), dtype=torch.float64, device="cuda")
    cap = eng.capture(0, x)
    cap.launch().result()
    eng.dispose()
    with pytest.raises(rb.UseAfterDispose):
        cap.launch()
