"""Row sharding across GPUs.

The population is the only thing that is split: device r owns rows
[r*N/W, (r+1)*N/W) (remainder to the leading devices), every device holds a
full replica of the instance pack, and the only exchange is the all-gather of
the fitness vector so every device ends with all N values -- the engine
contract (engine.py:174-214) returns a value per input row.  Values are
bit-identical to a single-GPU evaluation: rows never interact
(engine.py:207-209).

Two process models, both behind the same row rule (Shard):

* ``ShardedEngine``: one process per GPU (torchrun / torch.distributed).
  ``submit`` queues the local evaluation (Engine.evaluate_async, no host
  synchronisation) and the NCCL all-gather of its fitness on a separate
  communication stream, so the gather of function k overlaps the evaluation
  of function k+1 (NVLink / NVSwitch); ``Pending.result`` checks every
  rank's status.  Under gloo (CPU tests) the gather is a host all_gather.
* ``MultiDeviceEngine``: one process driving several GPUs through the C ABI's
  rb_initialize_sharded / rb_func_evaluate_sharded: each device evaluates its
  rows and stores its slice into every peer's full-length output with P2P
  stores (peer_scatter_kernel) -- the collective fused into the evaluation
  stream, no NCCL call.

The reference has no distributed code at all; its only
parallelism is a GIL-bound thread pool over rows (engine.py:211-213).
"""

from __future__ import annotations

import ctypes
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


def _backend(group=None) -> str:
    import torch.distributed as dist
    return dist.get_backend(group)


def gather_fitness(local, shard: Shard, group=None, out=None):
    """All-gather per-rank fitness into the full N-vector (rank order).

    NCCL: ``all_gather_into_tensor`` (in place when shards are even, else a
    padded gather + trim).  gloo: a host ``all_gather`` of CPU copies, the
    result moved back to ``local``'s device."""
    import torch
    import torch.distributed as dist

    if shard.world == 1:
        if out is not None:
            out.copy_(local)
            return out
        return local
    if _backend(group) == "gloo":
        host = local.detach().cpu()
        width = max(shard.sizes)
        padded = torch.zeros(width, dtype=host.dtype)
        padded[: host.numel()] = host
        parts = [torch.empty_like(padded) for _ in range(shard.world)]
        dist.all_gather(parts, padded, group=group)
        full = torch.cat([parts[r][:n] for r, n in enumerate(shard.sizes)]).to(local.device)
        if out is not None:
            out.copy_(full)
            return out
        return full
    if shard.even:
        if out is None:
            out = torch.empty(shard.n_total, dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(out, local.contiguous(), group=group)
        return out
    width = max(shard.sizes)
    padded = torch.zeros(width, dtype=local.dtype, device=local.device)
    padded[: local.numel()] = local
    tmp = torch.empty(width * shard.world, dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(tmp, padded, group=group)
    full = torch.cat([tmp[r * width: r * width + n] for r, n in enumerate(shard.sizes)])
    if out is not None:
        out.copy_(full)
        return out
    return full


class ShardedEngine:
    """Evaluate a row-sharded population, one process per GPU.

    ``engine``: this package's Engine on this rank's GPU (or, in CPU tests, any
    object with the Engine.evaluate signature)."""

    def __init__(self, engine, shard: Shard, group=None):
        self.engine, self.shard, self.group = engine, shard, group
        self._comm = None

    def _comm_stream(self, device):
        import torch
        if self._comm is None:
            self._comm = torch.cuda.Stream(device=device)
        return self._comm

    def evaluate(self, fn_id: int, local_points, precision: str | None = None):
        """Synchronous: every row's value, on every rank."""
        from .engine import EvalResult
        if not hasattr(self.engine, "evaluate_async") or not _is_cuda(local_points):
            local = self.engine.evaluate(fn_id, local_points, precision).values
            return EvalResult(gather_fitness(local, self.shard, self.group))
        return self.submit(fn_id, local_points, precision).result()

    def submit(self, fn_id: int, local_points, precision: str | None = None, *, out=None,
               local_out=None):
        """Queue this rank's rows (no host synchronisation) and the fitness
        all-gather behind them on the communication stream; returns a
        Pending whose ``values`` is the full N-vector (``out`` if given).
        The next submit's evaluation overlaps this one's gather."""
        import torch

        from .engine import Pending
        pend = self.engine.evaluate_async(fn_id, local_points, precision, out=local_out)
        local = pend.values
        if self.shard.world == 1:
            if out is not None:
                out.copy_(local)
                local = out
            return Pending(local, pend._tickets, pend.done, keep=pend._keep)
        comm = self._comm_stream(local.device)
        comm.wait_event(pend.done)
        with torch.cuda.stream(comm):
            full = gather_fitness(local, self.shard, self.group, out=out)
            local.record_stream(comm)
            if out is not None:
                out.record_stream(comm)
            done = torch.cuda.Event()
            done.record(comm)
        return Pending(full, pend._tickets, done, keep=pend._keep + (local,))


def _is_cuda(x) -> bool:
    return type(x).__module__.startswith("torch") and getattr(x, "is_cuda", False)


class MultiDeviceEngine:
    """One process, several GPUs: the C ABI's sharded engine
    (rb_initialize_sharded), a pack replica per device.

    ``evaluate(fn, shards)``: ``shards[g]`` is device g's rows (a CUDA tensor
    on ``devices[g]``, Shard's row rule over the total); returns one
    full-length fitness tensor per device, all equal.  The all-gather is P2P
    stores from each device's evaluation stream (peer_scatter_kernel)."""

    def __init__(self, config, devices):
        from . import _lib, catalog
        from .engine import _config
        from .pack import Pack
        self.config = _config(config)
        self.devices = [int(d) for d in devices]
        self._lib = _lib
        dim = self.config.dim
        if dim >= catalog.MIN_CONSTRUCTED_DIMENSION:
            disabled = frozenset()
        else:
            disabled = frozenset(r.fn_id for r in catalog.FUNCTIONS
                                 if r.category in (catalog.HYBRID, catalog.COMPOSITION))
        self.disabled_ids = disabled
        self._pack = Pack(dim, self.config.seed, disabled)
        devs = (ctypes.c_int32 * len(self.devices))(*self.devices)
        handle = ctypes.c_void_p()
        _lib.check(_lib.load().rb_initialize_sharded(
            ctypes.byref(_lib.make_pack(self._pack)), int(self.config.max_concurrency), devs,
            len(self.devices), ctypes.byref(handle)))
        self._handle = handle

    def evaluate(self, fn_id: int, shards, precision: str | None = None, *, outs=None,
                 wait: bool = True):
        import torch

        from .engine import Pending
        precision = precision or self.config.precision
        dt = torch.float64 if precision == "double" else torch.float32
        G = len(self.devices)
        if len(shards) != G:
            raise ValueError(f"{G} shards expected")
        xs = [s.to(dt).contiguous() for s in shards]
        n_total = sum(int(x.shape[0]) for x in xs)
        want = Shard(0, G, n_total).sizes
        for g, x in enumerate(xs):
            if x.shape[0] != want[g] or x.device.index != self.devices[g]:
                raise ValueError(f"shard {g}: {want[g]} rows on cuda:{self.devices[g]} expected")
        if outs is None:
            outs = [torch.empty(n_total, dtype=dt, device=f"cuda:{d}") for d in self.devices]
        vp = ctypes.c_void_p
        xp = (vp * G)(*[x.data_ptr() for x in xs])
        fp = (vp * G)(*[o.data_ptr() for o in outs])
        streams = [torch.cuda.current_stream(d) for d in self.devices]
        sp = (vp * G)(*[s.cuda_stream for s in streams])
        tickets = (ctypes.c_int64 * G)()
        _lib = self._lib
        _lib.check(_lib.load().rb_func_evaluate_sharded(
            self._handle, int(fn_id), _lib.RB_DOUBLE if precision == "double" else _lib.RB_SINGLE,
            xp, n_total, fp, sp, tickets))
        done = []
        for g, d in enumerate(self.devices):
            ev = torch.cuda.Event()
            ev.record(streams[g])
            done.append(ev)
        pend = _ShardedPending(outs, self, list(tickets), done, keep=tuple(xs))
        return pend.result() if wait else pend

    def ticket_status(self, device_index: int, ticket: int) -> None:
        self._lib.check(self._lib.load().rb_sharded_ticket_status(self._handle, int(device_index),
                                                                  int(ticket)))

    def dispose(self) -> None:
        if getattr(self, "_handle", None) is not None and self._handle.value:
            self._lib.check(self._lib.load().rb_dispose_sharded(ctypes.byref(self._handle)))

    def __del__(self):
        try:
            self.dispose()
        except Exception:
            pass


class _ShardedPending:
    def __init__(self, outs, owner, tickets, done, keep=()):
        self.values, self._owner, self._tickets, self._done, self._keep = outs, owner, tickets, done, keep

    def result(self):
        for ev in self._done:
            ev.synchronize()
        for g, t in enumerate(self._tickets):
            self._owner.ticket_status(g, t)
        self._keep = ()
        return self.values
