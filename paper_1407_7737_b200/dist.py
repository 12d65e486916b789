"""Row sharding across GPUs, one process per GPU (torch.distributed).

The population is the only thing that is split: rank r owns rows
[r*N/W, (r+1)*N/W) (remainder to the leading ranks), every rank holds a full
replica of the instance pack, and the only exchange is one all-gather of the
fitness vector so every rank ends with all N values — the engine contract
(engine.py:174-214) returns a value per input row.  Values are bit-identical
to a single-GPU evaluation: rows never interact (engine.py:207-209).

The reference has no distributed code at all; its only
parallelism is a GIL-bound thread pool over rows (engine.py:211-213).
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    n_total: int

    @property
    def sizes(self) -> list[int]:
        base, extra = divmod(self.n_total, self.world)
        return [base + (1 if r < extra else 0) for r in range(self.world)]

    @property
    def start(self) -> int:
        return sum(self.sizes[: self.rank])

    @property
    def count(self) -> int:
        return self.sizes[self.rank]

    @property
    def even(self) -> bool:
        return self.n_total % self.world == 0


def gather_fitness(local, shard: Shard, group=None):
    """All-gather per-rank fitness into the full N-vector (rank order).

    Uses the single-buffer ``all_gather_into_tensor`` (NCCL all-gather over
    NVLink) when shards are even, else a padded gather + trim.
    """
    import torch
    import torch.distributed as dist

    if shard.world == 1:
        return local
    if shard.even:
        out = torch.empty(shard.n_total, dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(out, local.contiguous(), group=group)
        return out
    width = max(shard.sizes)
    padded = torch.zeros(width, dtype=local.dtype, device=local.device)
    padded[: local.numel()] = local
    out = torch.empty(width * shard.world, dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, padded, group=group)
    return torch.cat([out[r * width: r * width + n] for r, n in enumerate(shard.sizes)])


class ShardedEngine:
    """Evaluate a row-sharded population: local rows on this rank's GPU,
    then the fitness all-gather.  ``engine`` is any object with the
    Engine.evaluate signature (tests pass a CPU stand-in under gloo)."""

    def __init__(self, engine, shard: Shard, group=None):
        self.engine, self.shard, self.group = engine, shard, group

    def evaluate(self, fn_id: int, local_points, precision: str | None = None):
        local = self.engine.evaluate(fn_id, local_points, precision).values
        return gather_fitness(local, self.shard, self.group)
