"""Drop-in for robench callers, on the CPU: the reference's own EngineConfig,
PointBatch and exception classes are accepted / raised by this package
(engine.py:34-84, errors.py:4-52), and tests/refshim.py routes
robench.initialize here (the GPU side runs the reference's own tests:
tests/test_reference_suite_gpu.py)."""

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_1407_7737_b200 as rb
from paper_1407_7737_b200 import engine as E
from paper_1407_7737_b200 import errors

ROOT = Path(__file__).resolve().parent.parent


def _bare_engine(dim=10, max_conc=4):
    """An Engine whose device path is replaced by a recorder (no GPU)."""
    eng = object.__new__(E.Engine)
    eng.config = E.EngineConfig(dim=dim, max_concurrency=max_conc)
    eng._disposed = False
    eng._disabled = frozenset()
    seen = []
    eng._evaluate_host = lambda fn, data, prec: seen.append((fn, data, prec)) or np.zeros(len(data))
    return eng, seen


def test_reference_exception_classes_are_raised(reference):
    e = errors.BatchTooLarge("x")
    assert isinstance(e, reference.BatchTooLarge) and isinstance(e, rb.BatchTooLarge)
    assert isinstance(e, reference.BenchmarkError) and isinstance(e, rb.BenchmarkError)
    with pytest.raises(reference.UnknownFunction):
        rb.lookup(99)
    with pytest.raises(reference.BenchmarkError):      # no reference analogue: still caught
        raise errors.DeviceError("cuda")
    with pytest.raises(reference.DimensionTooSmall):
        rb.EngineConfig(dim=1)


def test_reference_point_batch_and_config_are_accepted(reference):
    eng, seen = _bare_engine()
    x = np.random.default_rng(0).uniform(-100, 100, (3, 10))
    eng.evaluate(4, reference.PointBatch(x), "single")
    fn, data, prec = seen[-1]
    assert fn == 4 and prec == "single" and np.array_equal(data, x)
    with pytest.raises(reference.BatchTooLarge):
        eng.evaluate(0, reference.PointBatch(np.zeros((5, 10))))
    with pytest.raises(reference.DimensionMismatch):
        eng.evaluate(0, reference.PointBatch(np.zeros((2, 9))))
    cfg = E._config(reference.EngineConfig(dim=32, max_concurrency=7, seed=3, precision="single",
                                           threads=8))
    assert (cfg.dim, cfg.max_concurrency, cfg.seed, cfg.precision, cfg.threads, cfg.device) == \
        (32, 7, 3, "single", 8, 0)


def test_refshim_routes_robench_initialize_here(reference):
    code = ("import tests.refshim as s; s.pytest_configure(None); import robench, robench.bench, "
            "paper_1407_7737_b200 as rb; "
            "assert robench.initialize.__doc__.startswith('robench.initialize routed'); "
            "assert robench.engine.initialize is robench.initialize; "
            "assert robench.bench.initialize is robench.initialize; print('ok')")
    env = dict(os.environ, PYTHONPATH=f"{reference.__path__[0].rsplit('/', 1)[0]}{os.pathsep}{ROOT}")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True,
                         text=True, timeout=300)
    assert out.stdout.strip().endswith("ok"), out.stderr[-2000:]
