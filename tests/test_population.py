"""On-device population source (paper_1407_7737_b200/population.py): the
§8d workload population drawn on the device equals numpy's Philox draw bit
for bit, for any row range (shards, sampled rows)."""

import numpy as np
import pytest

from paper_1407_7737_b200 import population as pop
from tests.conftest import cuda_available

M0, M1 = 0xD2E7470EE14C6C93, 0xCA5A826395121157
W0, W1 = 0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B
MASK = (1 << 64) - 1


def _philox_block(counter, key):
    """Philox4x64-10 (the restatement the CUDA kernel follows)."""
    c, k = list(counter), list(key)
    for _ in range(10):
        p0, p1 = M0 * c[0], M1 * c[2]
        c = [((p1 >> 64) ^ c[1] ^ k[0]) & MASK, p1 & MASK, ((p0 >> 64) ^ c[3] ^ k[1]) & MASK,
             p0 & MASK]
        k = [(k[0] + W0) & MASK, (k[1] + W1) & MASK]
    return c


def test_philox_restatement_matches_numpy():
    ent = pop.workload_entropy(100, 1000)
    key = pop.philox_key(ent)
    raw = np.random.Philox(np.random.SeedSequence(ent)).random_raw(12)
    mine = [w for b in range(3) for w in _philox_block([b + 1, 0, 0, 0], key)]
    assert [int(v) for v in raw] == mine


@pytest.mark.parametrize("first_row", [0, 1, 7, 999])
def test_host_rows_follow_the_stream(first_row):
    ent = pop.workload_entropy(100, 1000)
    full = np.random.Generator(np.random.Philox(np.random.SeedSequence(ent))).uniform(
        -100, 100, (1000, 100))
    assert np.array_equal(pop.host_rows(100, ent, first_row, 1)[0], full[first_row])


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")
@pytest.mark.parametrize("dim,n,first,count", [(100, 1000, 0, 1000), (100, 1000, 3, 17),
                                               (13, 500, 5, 101), (2, 64, 1, 63)])
def test_device_population_is_numpy_draw(dim, n, first, count):
    ent = pop.workload_entropy(dim, n)
    want = np.random.Generator(np.random.Philox(np.random.SeedSequence(ent))).uniform(
        -100, 100, (n, dim))[first:first + count]
    got = pop.uniform_population(dim, count, ent, first_row=first, dtypes=("double", "single"))
    assert np.array_equal(got["double"].cpu().numpy(), want)
    assert np.array_equal(got["single"].cpu().numpy(), want.astype(np.float32))
