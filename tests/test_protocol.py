"""The paper's protocol on this engine (paper_1407_7737_b200/protocol.py,
reference bench.py:23-150): same points, same checksum function, same report
format; on the GPU, values within the parity bar and stable checksums."""

import hashlib

import numpy as np
import pytest

from paper_1407_7737_b200 import protocol as PR
from tests.conftest import cuda_available


def test_protocol_points_pinned():
    # sha256 prefix of the reference's protocol_points(3, 10, seed=0, runs=4, batch=50)
    pts = PR.protocol_points(3, 10, 0, 4, 50)
    assert pts.shape == (4, 50, 10)
    assert hashlib.sha256(pts.tobytes()).hexdigest()[:16] == "a025b18c426b0d1f"
    assert PR.checksum([pts[0]]) == "1059fb3f37767354"


def test_protocol_matches_live_reference(reference):
    from robench import bench as RB
    for fn, dim in ((3, 10), (36, 32), (8, 96)):
        assert np.array_equal(PR.protocol_points(fn, dim, 2, 3, 50), RB.protocol_points(fn, dim, 2, 3, 50))
    assert PR.CEC14_OVERLAP_IDS == RB.CEC14_OVERLAP_IDS
    assert PR.PROTOCOL_DIMS == RB.PROTOCOL_DIMS and PR.PROTOCOL_BATCH == RB.PROTOCOL_BATCH
    row = dict(fn_id=3, dim=10, precision="double", batch=50, runs=4, total_evals=200,
               batch_ns_per_eval=12.25, min_batch_ns=500.0, baseline_ns_per_eval=99.5,
               ratio=8.1224, checksum="0123456789abcdef")
    assert PR.EvalReport((PR.ReportRow(**row),)).to_tsv() == RB.EvalReport((RB.ReportRow(**row),)).to_tsv()


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")
def test_protocol_on_gpu_values_and_checksums():
    from oracle.robench_oracle import Oracle
    import paper_1407_7737_b200 as rb
    fns, dims = (3, 8, 23, 29), (10, 32)
    a = PR.run_protocol(fns=fns, dims=dims, runs=4)
    b = PR.run_protocol(fns=fns, dims=dims, runs=4)
    assert a.checksums() == b.checksums()          # timing never changes a value
    assert len(a.rows) == len(fns) * len(dims) and all(r.ratio > 0 for r in a.rows)
    for dim in dims:
        eng = rb.initialize(rb.EngineConfig(dim=dim, max_concurrency=50, seed=0))
        orc = Oracle(dim, 0)
        for fn in fns:
            pts = PR.protocol_points(fn, dim, 0, 4, 50)
            vals = [eng.evaluate(fn, pts[r]).values for r in range(4)]
            assert PR.checksum(vals) == a.checksums()[(fn, dim)]
            want = np.concatenate([orc.evaluate(fn, pts[r], "double") for r in range(4)])
            got = np.concatenate(vals)
            assert np.all(np.abs(got - want) <= np.maximum(1e-12 * np.abs(want), 1e-10))
        eng.dispose()
