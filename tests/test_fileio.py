"""Instance files -> device pack, points / values / grid formats
(paper_1407_7737_b200/fileio.py, grid.py; reference fileio.py, cli.py)."""

from pathlib import Path

import numpy as np
import pytest

from paper_1407_7737_b200 import fileio as F
from paper_1407_7737_b200 import pack as P
from paper_1407_7737_b200.errors import CorruptInstance, ParseError, UnsupportedAtDim2
from tests.conftest import cuda_available

GOLDEN = Path(__file__).with_name("golden") / "grid.npz"


@pytest.mark.parametrize("fn", [0, 10, 16, 23, 28, 30, 35])
def test_instance_file_round_trip(tmp_path, fn):
    f = F.instance_file(fn, 13, 4)
    path = tmp_path / "inst.txt"
    F.store_instance(f, path)
    g = F.load_instance(path)
    for name in ("x_opt", "group_perm", "split_perm"):
        a, b = getattr(f, name), getattr(g, name)
        assert (a is None and b is None) or np.array_equal(a, b)
    for name in ("blocks", "chunk_rotations", "member_optima"):
        a, b = getattr(f, name), getattr(g, name)
        assert (a is None and b is None) or all(np.array_equal(x, y) for x, y in zip(a, b))


@pytest.mark.parametrize("dim", [10, 30])
def test_pack_from_files_is_pack_from_seed(tmp_path, dim):
    # the loader feeds the device exactly the data generation would
    overrides = {}
    for fn in range(37):
        path = tmp_path / f"instance_f{fn:02d}_d{dim}_s1.txt"
        F.store_instance(F.instance_file(fn, dim, 1), path)
        overrides[fn] = F.to_instance(F.load_instance(path))
    a, b = P.Pack(dim, 1), P.Pack(dim, 1, overrides=overrides)
    assert np.array_equal(a.values_f64, b.values_f64)
    assert np.array_equal(a.values_f32, b.values_f32)
    assert np.array_equal(a.index, b.index)
    assert a.groups.tobytes() == b.groups.tobytes() and a.segments.tobytes() == b.segments.tobytes()


def test_gates(tmp_path):
    path = tmp_path / "i.txt"
    F.store_instance(F.instance_file(3, 10, 0), path)
    text = path.read_text()
    bad = tmp_path / "bad.txt"
    lines = text.splitlines()
    perm_line = next(i for i, l in enumerate(lines) if l.startswith("perm "))
    lines[perm_line] = "perm " + " ".join(["0"] * 10)
    bad.write_text("\n".join(lines) + "\n")
    with pytest.raises(CorruptInstance):
        F.load_instance(bad)
    lines = text.splitlines()
    blk = next(i for i, l in enumerate(lines) if l.startswith("block 0"))
    lines[blk + 1] = " ".join(str(2.0 * float(v)) for v in lines[blk + 1].split())
    bad.write_text("\n".join(lines) + "\n")
    with pytest.raises(CorruptInstance):
        F.load_instance(bad)
    bad.write_text(text.replace("robench-instance 1", "robench-instance 2"))
    with pytest.raises(ParseError):
        F.load_instance(bad)
    bad.write_text("\n".join(text.splitlines()[:-2]) + "\n")
    with pytest.raises(ParseError):
        F.load_instance(bad)


def test_reference_files_interoperate(tmp_path, reference):
    from robench import fileio as RF
    from robench.transforms import generate_instance
    for fn in (5, 11, 24, 32, 36):
        ref_path, our_path = tmp_path / f"r{fn}.txt", tmp_path / f"o{fn}.txt"
        RF.store_instance(generate_instance(fn, 20, 2), ref_path)
        F.store_instance(F.instance_file(fn, 20, 2), our_path)
        assert ref_path.read_text() == our_path.read_text()
        RF.load_instance(our_path)
        F.load_instance(ref_path)


def test_points_values_grid_formats(tmp_path):
    from paper_1407_7737_b200 import PointBatch
    x = np.random.default_rng(0).uniform(-100, 100, (5, 3))
    F.write_points(PointBatch(x), tmp_path / "p.txt")
    assert np.array_equal(F.read_points(tmp_path / "p.txt", 3).data, x)
    v = np.random.default_rng(1).uniform(100, 1e6, 9).astype(np.float32)
    F.write_values(v, tmp_path / "v.txt")
    assert np.array_equal(F.read_values(tmp_path / "v.txt", "single"), v)
    g = np.random.default_rng(2).uniform(size=(4, 4))
    F.write_grid(tmp_path / "g.txt", 8, 3, -5.0, 5.0, g)
    fn, seed, lo, hi, back = F.read_grid(tmp_path / "g.txt")
    assert (fn, seed, lo, hi) == (8, 3, -5.0, 5.0) and np.array_equal(back, g)


def test_grid_rejects_hybrids():
    from paper_1407_7737_b200.grid import landscape
    for fn in (23, 35):
        with pytest.raises(UnsupportedAtDim2):
            landscape(fn)


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")
def test_engine_from_files_matches_seeded(tmp_path):
    import paper_1407_7737_b200 as rb
    paths = []
    for fn in (0, 10, 16, 24, 29, 36):
        p = tmp_path / f"instance_f{fn:02d}_d30_s2.txt"
        F.store_instance(F.instance_file(fn, 30, 2), p)
        paths.append(p)
    cfg = rb.EngineConfig(dim=30, max_concurrency=64, seed=2)
    a, b = rb.initialize(cfg), F.initialize_from_files(cfg, paths)
    x = np.random.default_rng(5).uniform(-100, 100, (64, 30))
    from oracle.robench_oracle import Oracle
    orc = Oracle(30, 2)                 # the seeded instances: pins the file engine to the reference
    for fn in (0, 10, 16, 24, 29, 36):
        for prec in ("double", "single"):
            got = b.evaluate(fn, x, precision=prec).values
            assert np.array_equal(a.evaluate(fn, x, precision=prec).values, got)
            want = orc.evaluate(fn, x, prec).astype(np.float64)
            rel, ab = (1e-12, 1e-10) if prec == "double" else (1e-5, 0.0)
            assert np.all(np.abs(got.astype(np.float64) - want) <= np.maximum(rel * np.abs(want), ab))
    a.dispose()
    b.dispose()


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")
def test_landscape_matches_reference_scalar_evaluator(tmp_path):
    from paper_1407_7737_b200.grid import export_grid
    gold = np.load(GOLDEN)
    steps, lo, hi, seed = gold["meta"]
    for fn in gold["fns"]:
        want = gold[f"grid/{int(fn)}"]
        got = export_grid(tmp_path / f"g{int(fn)}.txt", int(fn), int(seed), float(lo), float(hi),
                          int(steps))
        assert np.all(np.abs(got - want) <= np.maximum(1e-12 * np.abs(want), 1e-10)), int(fn)
        assert np.array_equal(F.read_grid(tmp_path / f"g{int(fn)}.txt")[4], got)
