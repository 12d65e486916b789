"""Host instance generation is bit-identical to the reference
(transforms.py:37-230, hybrid.py:72-95, composition.py:75-111)."""

import json

import numpy as np
import pytest

from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
from paper_1407_7737_b200 import catalog, instances
from tests.golden.digest import digest

GOLDEN = json.loads((ROOT / "tests" / "golden" / "instances.json").read_text())


def arrays(fn, dim, seed):
    inst = instances.build(fn, dim, seed)
    if isinstance(inst, instances.BasicInstance):
        rot = inst.rotation or instances.grouped_rotation(fn, dim, seed)
        return [inst.shift, rot.perm, rot.dense()]
    if isinstance(inst, instances.HybridInstance):
        return [inst.shift, inst.split_perm, np.asarray(inst.sizes), *inst.chunk_rotations]
    out = []
    for m in inst.members:
        out.append(m.shift)
        if m.rotation is not None:
            out.append(m.rotation.dense())
        else:
            out += [m.hybrid.split_perm, np.asarray(m.hybrid.sizes), *m.hybrid.chunk_rotations]
    return out


@pytest.mark.parametrize("key", sorted(GOLDEN))
def test_instance_digest_matches_reference(key):
    fn, dim, seed = map(int, key.split("/"))
    assert digest(arrays(fn, dim, seed)) == GOLDEN[key]


def test_live_reference_instances(reference):
    from robench import composition, hybrid, transforms
    for dim in (3, 17, 64):
        for fn in (0, 5, 16, 22):
            ref = transforms.generate_instance(fn, dim, 11)
            mine = instances.build(fn, dim, 11)
            assert np.array_equal(ref.x_opt, mine.shift)
            assert np.array_equal(ref.rotation, mine.rotation.dense())
        for fn in ((23, 28) if dim >= 10 else ()):
            ref = hybrid.build_hybrid(fn, dim, 11)
            mine = instances.build(fn, dim, 11)
            assert ref.sizes == mine.sizes
            assert np.array_equal(ref.split_perm, mine.split_perm)
            assert all(np.array_equal(a, b) for a, b in zip(ref.chunk_rotations, mine.chunk_rotations))
        ref = composition.build_composition(33, dim, 11)
        mine = instances.build(33, dim, 11)
        for a, b in zip(ref.members, mine.members):
            assert np.array_equal(a.x_opt, b.shift)
            assert np.array_equal(a.rotation, b.rotation.dense())


def test_chunk_sizes_partition_the_dimension():
    # reference criterion 4 (test_acceptance.py:133-141)
    for fn in range(23, 29):
        for dim in range(10, 257):
            sizes = instances.chunk_sizes(catalog.lookup(fn).fractions, dim)
            assert sum(sizes) == dim and min(sizes) >= 1
    assert instances.chunk_sizes((0.3, 0.3, 0.4), 50) == (15, 15, 20)
    assert instances.chunk_sizes((0.1, 0.2, 0.2, 0.2, 0.3), 100) == (10, 20, 20, 20, 30)


def test_group_sizes():
    assert instances.group_sizes(100) == (34, 33, 33)
    assert instances.group_sizes(10) == (4, 3, 3)
    assert instances.group_sizes(2) == (1, 1)


def test_rotations_orthonormal():
    for dim in (2, 10, 50):
        rot = instances.grouped_rotation(0, dim, 3)
        r = rot.dense()
        assert np.max(np.abs(r.T @ r - np.eye(dim))) < 1e-10
        assert sorted(rot.perm.tolist()) == list(range(dim))
