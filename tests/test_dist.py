"""Row sharding + fitness all-gather (dist.py) on world_size 2 with gloo on
CPU; the per-rank evaluator is the CPU oracle, so the check is the
plumbing: partition, rank order, bit-identity with one process."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1407_7737_b200.dist import Shard, ShardedEngine


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class OracleEngine:
    def __init__(self, dim):
        from oracle.robench_oracle import Oracle
        self.orc = Oracle(dim, 0)

    def evaluate(self, fn, pts, precision=None):
        class R:
            pass
        r = R()
        r.values = torch.from_numpy(self.orc.evaluate(fn, pts.numpy(), precision or "double"))
        return r


def _worker(rank, world, port, n, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.robench_oracle import population
    x = population(10, n, seed=3)
    sh = Shard(rank, world, n)
    eng = ShardedEngine(OracleEngine(10), sh)
    local = torch.from_numpy(x[sh.start:sh.start + sh.count])
    for fn in (0, 23, 30):
        full = eng.evaluate(fn, local, "double").values
        if rank == 0:
            np.save(f"{out}_{fn}.npy", full.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [10, 11])
def test_sharded_evaluation_matches_single_process(tmp_path, n):
    out = str(tmp_path / "f")
    mp.spawn(_worker, args=(2, free_port(), n, out), nprocs=2, join=True)
    from oracle.robench_oracle import Oracle, population
    x = population(10, n, seed=3)
    orc = Oracle(10, 0)
    for fn in (0, 23, 30):
        assert np.array_equal(np.load(f"{out}_{fn}.npy"), orc.evaluate(fn, x, "double"))


def test_shard_partition():
    for n in (1, 7, 10, 10_000_000):
        for w in (1, 2, 4, 8):
            shards = [Shard(r, w, n) for r in range(w)]
            assert sum(s.count for s in shards) == n
            assert [s.start for s in shards] == list(np.cumsum([0] + [s.count for s in shards])[:-1])


def _pop_worker(rank, world, port, dim, n, out):
    # each rank draws only its shard of the 8d population (what bench.py does
    # on the device with population.uniform_population(first_row=shard.start))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1407_7737_b200.population import host_rows, workload_entropy
    sh = Shard(rank, world, n)
    local = torch.from_numpy(host_rows(dim, workload_entropy(dim, n), sh.start, sh.count)).reshape(-1)
    width = max(sh.sizes) * dim                       # gloo gathers equal sizes: pad
    padded = torch.zeros(width, dtype=torch.float64)
    padded[: local.numel()] = local
    rows = [torch.empty(width, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(rows, padded)
    if rank == 0:
        full = torch.cat([rows[r][: c * dim] for r, c in enumerate(sh.sizes)])
        np.save(out, full.numpy().reshape(n, dim))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 12), (4, 10)])
def test_sharded_population_is_the_single_process_draw(tmp_path, world, n):
    from paper_1407_7737_b200.population import workload_entropy
    out = str(tmp_path / "x.npy")
    mp.spawn(_pop_worker, args=(world, free_port(), 100, n, out), nprocs=world, join=True)
    want = np.random.Generator(np.random.Philox(np.random.SeedSequence(
        workload_entropy(100, n)))).uniform(-100, 100, (n, 100))
    assert np.array_equal(np.load(out), want)
