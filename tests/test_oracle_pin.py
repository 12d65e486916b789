"""Pin the CPU oracle (oracle/robench_oracle.py) to the reference: bit-exact
against the committed golden vectors (made by tests/golden/make_golden.py
from the live reference) and, when mounted, against the live reference."""

import numpy as np
import pytest

from oracle.robench_oracle import Oracle

DIMS = (2, 10, 13, 30, 50, 100)


@pytest.mark.parametrize("dim", DIMS)
def test_oracle_matches_golden_bit_exact(golden, dim):
    seed = int(golden["seed"])
    orc = Oracle(dim, seed)
    x = golden[f"x/{dim}"]
    for fn in range(37):
        key = f"f/{dim}/{fn}/double"
        if key not in golden.files:
            continue
        pts = np.vstack([x, golden[f"opt/{dim}/{fn}"][None, :]])
        for prec in ("double", "single"):
            want = golden[f"f/{dim}/{fn}/{prec}"]
            got = orc.evaluate(fn, pts, prec)
            assert got.dtype == want.dtype
            assert np.array_equal(got, want), (fn, prec, got - want)


def test_oracle_known_answers(golden):
    # F(optimum) = 100 (test_engine.py:44-47; test_acceptance.py:61-74)
    for dim in (10, 30, 100):
        orc = Oracle(dim, int(golden["seed"]))
        opt = golden[f"opt/{dim}/0"]
        assert orc.evaluate(0, opt[None, :])[0] == 100.0


def test_oracle_matches_live_reference(reference):
    rng = np.random.default_rng(77)
    for dim in (10, 31):
        eng = reference.initialize(reference.EngineConfig(dim=dim, max_concurrency=64, seed=2))
        orc = Oracle(dim, 2)
        x = rng.uniform(-100, 100, (16, dim))
        for fn in range(37):
            for prec in ("double", "single"):
                assert np.array_equal(eng.evaluate(fn, x, precision=prec).values,
                                      orc.evaluate(fn, x, prec)), (dim, fn, prec)
        eng.dispose()
