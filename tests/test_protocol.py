"""The paper's protocol on this engine (paper_1407_7737_b200/protocol.py): the
reference's own harness (bench.py:119-150) with the GPU engine injected --
values within the parity bar, checksums stable across runs, and the
reference's engine restored afterwards."""

import numpy as np
import pytest

from paper_1407_7737_b200 import protocol as PR
from tests.conftest import cuda_available


def _rb():
    try:
        return PR.reference_bench()
    except ImportError:
        pytest.skip("reference package not installed (tools/install_reference.sh)")


def test_adapter_swaps_and_restores_the_reference_engine(monkeypatch):
    rb = _rb()
    original = rb.initialize
    seen = []

    def fake_run(**kw):
        seen.append((rb.initialize is not original, kw))
        raise RuntimeError("stop")

    monkeypatch.setattr(rb, "run_protocol", fake_run)
    with pytest.raises(RuntimeError):
        PR.run_protocol(fns=(3,), dims=(10,), runs=2)
    assert seen and seen[0][0], "the GPU engine was not injected"
    assert seen[0][1] == {"runs": 2, "seed": 0, "precision": "double", "fns": (3,), "dims": (10,)}
    assert rb.initialize is original


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")
def test_protocol_on_gpu_values_and_checksums():
    from oracle.robench_oracle import Oracle
    import paper_1407_7737_b200 as rb
    bench = _rb()
    fns, dims = (3, 8, 23, 29), (10, 32)
    a = PR.run_protocol(fns=fns, dims=dims, runs=4)
    b = PR.run_protocol(fns=fns, dims=dims, runs=4)
    assert PR.checksums(a) == PR.checksums(b)          # timing never changes a value
    assert len(a.rows) == len(fns) * len(dims) and all(r.ratio > 0 for r in a.rows)
    for dim in dims:
        eng = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=50, seed=0))
        orc = Oracle(dim, 0)
        for fn in fns:
            pts = bench.protocol_points(fn, dim, 0, 4, 50)
            vals = [eng.evaluate(fn, pts[r]).values for r in range(4)]
            assert bench._checksum(vals) == PR.checksums(a)[(fn, dim)]
            want = np.concatenate([orc.evaluate(fn, pts[r], "double") for r in range(4)])
            got = np.concatenate(vals)
            assert np.all(np.abs(got - want) <= np.maximum(1e-12 * np.abs(want), 1e-10))
        eng.dispose()
