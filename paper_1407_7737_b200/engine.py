"""Drop-in engine: the reference's ``initialize / Engine.evaluate /
evaluate_single_precision / dispose`` API (engine.py:34-228) over the
native C ABI.

Same types (EngineConfig, PointBatch, EvalResult), same validation order and
exception classes (engine.py:180-203), same values (+100 bias, the batch
dtype).  Differences, all additive:

* ``EngineConfig.device`` selects the GPU; ``threads`` is accepted and
  ignored (the per-point parallelism lives on the device).
* ``evaluate`` also accepts a CUDA ``torch.Tensor`` (N x D); the points then
  never leave the device and ``EvalResult.values`` is a CUDA tensor.  NumPy
  input goes through the host wrappers (rb_h_func_evaluate[f]) and returns
  NumPy, exactly like the reference.

Every evaluation runs on the GPU; there is no CPU path.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib, catalog
from .errors import (BatchTooLarge, DimensionMismatch, DimensionTooSmall, DisabledFunction,
                     UseAfterDispose)
from .pack import Pack

_DTYPES = {"double": np.float64, "single": np.float32}


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch") and hasattr(x, "is_cuda")


@dataclass(frozen=True)
class EngineConfig:
    """engine.py:34-52, plus ``device``.

    ``dim``: any value >= 2, as in the reference (engine.py:42-44).  Up to
    D ~ 340 every function runs from shared-memory tiles.  Past that, the
    functions whose tile no longer fits use the large-dimension kernel
    (tiles in global scratch).  That kernel is slower
    but gives the same values."""

    dim: int
    max_concurrency: int = 50
    seed: int = 0
    precision: str = "double"
    threads: int = 1
    device: int = 0

    def __post_init__(self):
        if self.dim < catalog.MIN_DIMENSION:
            raise DimensionTooSmall(f"dim must be >= {catalog.MIN_DIMENSION}, got {self.dim}")
        if self.max_concurrency < 1:
            raise ValueError("max_concurrency must be >= 1")
        if self.seed < 0:
            raise ValueError("seed must be a non-negative integer")
        if self.precision not in _DTYPES:
            raise ValueError(f"precision must be one of {sorted(_DTYPES)}")
        if self.threads < 1:
            raise ValueError("threads must be >= 1")


@dataclass(frozen=True)
class PointBatch:
    """N x D points (engine.py:55-77); NumPy array or CUDA torch tensor."""

    data: object

    def __post_init__(self):
        arr = self.data if _is_torch(self.data) else np.asarray(self.data)
        if arr.ndim != 2 or arr.shape[0] < 1:
            raise ValueError("batch data must be a non-empty 2-D array")
        object.__setattr__(self, "data", arr)

    @property
    def count(self) -> int:
        return int(self.data.shape[0])

    @property
    def dim(self) -> int:
        return int(self.data.shape[1])

    @property
    def precision(self) -> str:
        dt = self.data.dtype
        if _is_torch(self.data):
            import torch
            return "single" if dt == torch.float32 else "double"
        return "single" if dt == np.float32 else "double"


@dataclass(frozen=True)
class EvalResult:
    values: object


class Engine:
    """All 37 instances of one (dim, seed), resident on one GPU."""

    def __init__(self, config: EngineConfig, *, instances=None, enabled=None):
        """``instances``: {fn: instance} overriding the seeded ones (see
        fileio.initialize_from_files); ``enabled``: the function ids to
        build instead of the reference's rule (grid.py needs basic-member
        compositions at dimension 2, as scalar_evaluator does,
        engine.py:121-138)."""
        self.config = config = _config(config)
        self._disposed = False
        dim = config.dim
        if enabled is not None:
            self._disabled = frozenset(range(catalog.FUNCTION_COUNT)) - frozenset(enabled)
        elif dim >= catalog.MIN_CONSTRUCTED_DIMENSION:
            self._disabled = frozenset()
        else:                                               # engine.py:148-154
            self._disabled = frozenset(r.fn_id for r in catalog.FUNCTIONS
                                       if r.category in (catalog.HYBRID, catalog.COMPOSITION))
        lib = _lib.load()
        self._pack = Pack(dim, config.seed, self._disabled, instances)
        handle = ctypes.c_void_p()
        _lib.check(lib.rb_initialize(ctypes.byref(_lib.make_pack(self._pack)),
                                     int(config.max_concurrency), int(config.device),
                                     ctypes.byref(handle)))
        self._handle = handle
        import weakref
        self._captures = weakref.WeakSet()      # graphs reference the device pack: closed by dispose()
        # engine.py:155-159 keeps one per-point evaluator per (fn, precision);
        # here each is a handle onto the device-resident instance
        self._evaluators = {(fn, prec): _PointEvaluator(self, fn, prec)
                            for fn in self.enabled_ids for prec in _DTYPES}

    @property
    def dim(self) -> int:
        return self.config.dim

    @property
    def disabled_ids(self) -> frozenset:
        return self._disabled

    @property
    def enabled_ids(self) -> tuple:
        return tuple(fn for fn in range(catalog.FUNCTION_COUNT) if fn not in self._disabled)

    def evaluate(self, fn_id: int, batch, precision: str | None = None, *, out=None) -> EvalResult:
        """Score every point of ``batch`` against ``fn_id`` (engine.py:174-214).

        ``batch``: this package's PointBatch, any object with a 2-D ``data``
        array (the reference's own ``robench.PointBatch``), a NumPy array or
        a CUDA tensor.
        ``out`` (addition, CUDA batches only): a contiguous device tensor of
        the batch's length and the precision's dtype that receives the values
        (pipelines that keep results resident, e.g. bench.py's e2e step)."""
        if self._disposed:
            raise UseAfterDispose("engine was disposed")
        if not isinstance(batch, PointBatch):
            data = batch
            if not isinstance(batch, np.ndarray) and not _is_torch(batch) and hasattr(batch, "data"):
                data = batch.data                            # robench.PointBatch and friends
            batch = PointBatch(data)
        catalog.lookup(fn_id)
        fn_id = int(fn_id)
        if fn_id in self._disabled:
            raise DisabledFunction(
                f"function {fn_id} needs dimension >= {catalog.MIN_CONSTRUCTED_DIMENSION}")
        if batch.count > self.config.max_concurrency:
            raise BatchTooLarge(f"batch of {batch.count} exceeds "
                                f"max_concurrency={self.config.max_concurrency}")
        if batch.dim != self.config.dim:
            raise DimensionMismatch(f"batch dim {batch.dim} != engine dim {self.config.dim}")
        precision = precision or self.config.precision
        if precision not in _DTYPES:
            raise ValueError(f"precision must be one of {sorted(_DTYPES)}")
        if _is_torch(batch.data):
            return EvalResult(self._evaluate_device(fn_id, batch.data, precision, out))
        if out is not None:
            raise ValueError("out= is only supported for CUDA tensor batches")
        return EvalResult(self._evaluate_host(fn_id, batch.data, precision))

    def evaluate_async(self, fn_id: int, batch, precision: str | None = None, *,
                       out=None) -> "Pending":
        """Queue the evaluation of a CUDA-tensor batch on the current stream
        and return at once (rb_func_evaluate_async): argument errors are
        raised now, in the reference's order; NonFiniteInput is raised by
        ``Pending.result()``, which waits for the values.  No host
        synchronisation per call, so callers can overlap many functions with
        copies or collectives (dist.ShardedEngine, bench.py)."""
        import torch
        if self._disposed:
            raise UseAfterDispose("engine was disposed")
        if not isinstance(batch, PointBatch):
            batch = PointBatch(batch)
        if not _is_torch(batch.data):
            raise ValueError("evaluate_async takes CUDA tensor batches (host arrays: evaluate)")
        catalog.lookup(fn_id)
        fn_id = int(fn_id)
        if fn_id in self._disabled:
            raise DisabledFunction(
                f"function {fn_id} needs dimension >= {catalog.MIN_CONSTRUCTED_DIMENSION}")
        if batch.count > self.config.max_concurrency:
            raise BatchTooLarge(f"batch of {batch.count} exceeds "
                                f"max_concurrency={self.config.max_concurrency}")
        if batch.dim != self.config.dim:
            raise DimensionMismatch(f"batch dim {batch.dim} != engine dim {self.config.dim}")
        precision = precision or self.config.precision
        if precision not in _DTYPES:
            raise ValueError(f"precision must be one of {sorted(_DTYPES)}")
        pts, out = self._device_args(batch.data, precision, out)
        stream = torch.cuda.current_stream(pts.device)
        ticket = ctypes.c_int64(-1)
        _lib.check(_lib.load().rb_func_evaluate_async(
            self._handle, fn_id, _lib.RB_DOUBLE if precision == "double" else _lib.RB_SINGLE,
            pts.data_ptr(), pts.shape[0], out.data_ptr(), stream.cuda_stream, ctypes.byref(ticket)))
        done = torch.cuda.Event()
        done.record(stream)
        return Pending(out, [(self, ticket.value)], done, keep=(pts,))

    def capture(self, fn_id: int, batch, precision: str | None = None, *,
                out=None) -> "CapturedEvaluation":
        """Capture one evaluation of a CUDA-tensor batch as a CUDA graph
        (rb_graph_capture) for repeated use on the same buffers: each
        ``launch()`` evaluates the tensor's CURRENT contents with one
        cudaGraphLaunch, no per-call validation or flag bookkeeping (small
        populations in an optimizer loop are launch-bound).  Argument
        errors are raised here, in the reference's order; NonFiniteInput by
        ``result()`` after each launch."""
        if self._disposed:
            raise UseAfterDispose("engine was disposed")
        if not isinstance(batch, PointBatch):
            batch = PointBatch(batch)
        if not _is_torch(batch.data):
            raise ValueError("capture takes CUDA tensor batches")
        catalog.lookup(fn_id)
        fn_id = int(fn_id)
        if fn_id in self._disabled:
            raise DisabledFunction(
                f"function {fn_id} needs dimension >= {catalog.MIN_CONSTRUCTED_DIMENSION}")
        if batch.count > self.config.max_concurrency:
            raise BatchTooLarge(f"batch of {batch.count} exceeds "
                                f"max_concurrency={self.config.max_concurrency}")
        if batch.dim != self.config.dim:
            raise DimensionMismatch(f"batch dim {batch.dim} != engine dim {self.config.dim}")
        precision = precision or self.config.precision
        if precision not in _DTYPES:
            raise ValueError(f"precision must be one of {sorted(_DTYPES)}")
        pts, out = self._device_args(batch.data, precision, out)
        if pts.data_ptr() != batch.data.data_ptr():
            raise ValueError("capture needs a contiguous tensor of the evaluation dtype "
                             "(a converted copy would not see later updates)")
        handle = ctypes.c_void_p()
        _lib.check(_lib.load().rb_graph_capture(
            self._handle, fn_id, _lib.RB_DOUBLE if precision == "double" else _lib.RB_SINGLE,
            pts.data_ptr(), pts.shape[0], out.data_ptr(), ctypes.byref(handle)))
        cap = CapturedEvaluation(self, handle, pts, out)
        self._captures.add(cap)
        return cap

    def evaluate_many(self, calls, batches, *, outs=None) -> "list[Pending]":
        """Several evaluations in ONE native call: ``calls`` = [(fn_id,
        precision), ...].  Host rows (a NumPy array / PointBatch): returns
        [EvalResult] synchronously, the rows crossing PCIe once for all calls
        (rb_h_func_evaluate_many; float32 calls evaluate float32(X) as
        engine.py:201).  CUDA tensors (rb_func_evaluate_many): ``batches`` =
        {precision: tensor (N x D)}, a list with one tensor per call, or one
        tensor;
        ``outs`` = optional output tensors, one per call.  Same checks and
        values as evaluate_async per call, without Python work per launch --
        e.g. the whole suite on one population (bench.py's step)."""
        if self._disposed:
            raise UseAfterDispose("engine was disposed")
        if not isinstance(batches, (dict, list, tuple)) and not _is_torch(batches):
            return self._evaluate_many_host(calls, batches)
        import torch
        k = len(calls)
        i32, i64, vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p
        fns, precs, xs, ns, fs = (i32 * k)(), (i32 * k)(), (vp * k)(), (i64 * k)(), (vp * k)()
        keep, results = [], []
        for i, (fn, prec) in enumerate(calls):
            prec = prec or self.config.precision
            if prec not in _DTYPES:
                raise ValueError(f"precision must be one of {sorted(_DTYPES)}")
            data = (batches[prec] if isinstance(batches, dict) else
                    batches[i] if isinstance(batches, (list, tuple)) else batches)
            if not _is_torch(data) or data.ndim != 2:
                raise ValueError("evaluate_many takes CUDA tensor batches")
            if data.shape[1] != self.config.dim:
                raise DimensionMismatch(f"batch dim {data.shape[1]} != engine dim {self.config.dim}")
            pts, out = self._device_args(data, prec, outs[i] if outs is not None else None)
            keep.append(pts)
            results.append(out)
            fns[i], precs[i] = int(fn), _lib.RB_DOUBLE if prec == "double" else _lib.RB_SINGLE
            xs[i], ns[i], fs[i] = pts.data_ptr(), pts.shape[0], out.data_ptr()
        stream = torch.cuda.current_stream(torch.device("cuda", self.config.device))
        tickets = (i64 * k)()
        _lib.check(_lib.load().rb_func_evaluate_many(self._handle, k, fns, precs, xs, ns, fs,
                                                     stream.cuda_stream, tickets))
        done = torch.cuda.Event()
        done.record(stream)
        return [Pending(results[i], [(self, tickets[i])], done, keep=(keep[i],)) for i in range(k)]

    def _evaluate_many_host(self, calls, batch) -> "list[EvalResult]":
        """Host rows (NumPy / PointBatch): every call's values, the rows
        crossing PCIe once for all calls (rb_h_func_evaluate_many)."""
        if not isinstance(batch, PointBatch):
            batch = PointBatch(batch.data if hasattr(batch, "data") and not isinstance(batch, np.ndarray)
                               else batch)
        if batch.dim != self.config.dim:
            raise DimensionMismatch(f"batch dim {batch.dim} != engine dim {self.config.dim}")
        pts = np.ascontiguousarray(batch.data, dtype=np.float64)
        k = len(calls)
        i32, vp = ctypes.c_int32, ctypes.c_void_p
        fns, precs, fs = (i32 * k)(), (i32 * k)(), (vp * k)()
        outs = []
        for i, (fn, prec) in enumerate(calls):
            prec = prec or self.config.precision
            if prec not in _DTYPES:
                raise ValueError(f"precision must be one of {sorted(_DTYPES)}")
            out = np.empty(pts.shape[0], dtype=_DTYPES[prec])
            outs.append(out)
            fns[i], precs[i] = int(fn), _lib.RB_DOUBLE if prec == "double" else _lib.RB_SINGLE
            fs[i] = out.ctypes.data
        _lib.check(_lib.load().rb_h_func_evaluate_many(self._handle, k, fns, precs, _lib.ptr(pts),
                                                       pts.shape[0], fs))
        return [EvalResult(o) for o in outs]

    def ticket_status(self, ticket: int) -> None:
        """Raise NonFiniteInput if the completed call behind ``ticket`` saw a
        non-finite input (rb_ticket_status)."""
        _lib.check(_lib.load().rb_ticket_status(self._handle, int(ticket)))

    def evaluate_single_precision(self, fn_id: int, batch) -> EvalResult:
        return self.evaluate(fn_id, batch, precision="single")

    def dispose(self) -> None:
        """Free the device pack; a second dispose is a no-op (engine.py:219-222)."""
        if not self._disposed:
            for cap in list(getattr(self, "_captures", ())):
                cap.close()
            _lib.check(_lib.load().rb_dispose(ctypes.byref(self._handle)))
            self._pack = None
            self._evaluators = None
        self._disposed = True

    def __del__(self):
        try:
            self.dispose()
        except Exception:
            pass

    # -- paths
    def _evaluate_host(self, fn_id, data, precision):
        dt = _DTYPES[precision]
        lib = _lib.load()
        if dt is np.float32 and data.dtype == np.float64:
            # engine.py:201's float32 cast, done per row chunk inside the
            # native transfer pipeline (rb_h_func_evaluate_x64)
            pts = np.ascontiguousarray(data)
            out = np.empty(pts.shape[0], dtype=dt)
            _lib.check(lib.rb_h_func_evaluate_x64(self._handle, fn_id, _lib.RB_SINGLE, _lib.ptr(pts),
                                                  pts.shape[0], _lib.ptr(out)))
            return out
        pts = np.ascontiguousarray(data, dtype=dt)          # engine.py:201
        out = np.empty(pts.shape[0], dtype=dt)
        call = lib.rb_h_func_evaluate if dt is np.float64 else lib.rb_h_func_evaluatef
        _lib.check(call(self._handle, fn_id, _lib.ptr(pts), pts.shape[0], _lib.ptr(out)))
        return out

    def _device_args(self, data, precision, out):
        import torch
        if not data.is_cuda or data.device.index != self.config.device:
            raise ValueError(f"tensor must live on cuda:{self.config.device}")
        dt = torch.float64 if precision == "double" else torch.float32
        pts = data.to(dt).contiguous()
        if out is None:
            out = torch.empty(pts.shape[0], dtype=dt, device=pts.device)
        elif (out.dtype != dt or out.device != pts.device or not out.is_contiguous()
              or out.numel() != pts.shape[0]):
            raise ValueError("out must be a contiguous device tensor of the batch's length and dtype")
        return pts, out

    def _evaluate_device(self, fn_id, data, precision, out=None):
        import torch
        pts, out = self._device_args(data, precision, out)
        stream = torch.cuda.current_stream(pts.device).cuda_stream
        call = _lib.load().rb_func_evaluate if pts.dtype == torch.float64 else _lib.load().rb_func_evaluatef
        _lib.check(call(self._handle, fn_id, pts.data_ptr(), pts.shape[0], out.data_ptr(), stream))
        return out


class Pending:
    """An evaluation queued on a stream (Engine.evaluate_async,
    dist.ShardedEngine.submit): ``values`` fills in once ``done`` completes;
    ``result()`` waits for it and raises the reference's NonFiniteInput if
    any contributing call saw a non-finite input."""

    def __init__(self, values, tickets, done, keep=()):
        self.values, self._tickets, self.done, self._keep = values, tickets, done, keep

    def result(self) -> EvalResult:
        self.done.synchronize()
        for eng, ticket in self._tickets:
            eng.ticket_status(ticket)
        self._keep = ()
        return EvalResult(self.values)


class CapturedEvaluation:
    """An evaluation captured as a CUDA graph (Engine.capture).  ``launch()``
    queues one replay on the current stream; ``result()`` waits for the
    latest replay and raises NonFiniteInput if it saw a non-finite input.
    Replays of one capture must not overlap (they share its status words);
    the captured tensors are kept alive here."""

    def __init__(self, engine, handle, points, values):
        self._engine, self._handle, self.points, self.values = engine, handle, points, values
        self._done = None

    def launch(self) -> "CapturedEvaluation":
        import torch
        if self._handle is None or not self._handle.value:
            raise UseAfterDispose("captured evaluation was closed")
        stream = torch.cuda.current_stream(self.values.device)
        _lib.check(_lib.load().rb_graph_launch(self._handle, stream.cuda_stream))
        if self._done is None:
            self._done = torch.cuda.Event()
        self._done.record(stream)
        return self

    def result(self) -> EvalResult:
        if self._done is not None:
            self._done.synchronize()
        _lib.check(_lib.load().rb_graph_status(self._handle))
        return EvalResult(self.values)

    def close(self) -> None:
        if self._handle is not None and self._handle.value:
            _lib.check(_lib.load().rb_graph_destroy(ctypes.byref(self._handle)))
        self._handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _PointEvaluator:
    """``Engine._evaluators[(fn, precision)]`` (engine.py:87-118): calling it
    on one point returns that point's value without the bias, like the
    reference's per-point evaluators, computed on the device.  It holds the
    engine weakly: dispose() releases it (test_engine.py:158-166)."""

    __slots__ = ("_engine", "fn_id", "precision", "__weakref__")

    def __init__(self, engine: Engine, fn_id: int, precision: str):
        import weakref
        self._engine = weakref.ref(engine)
        self.fn_id, self.precision = fn_id, precision

    def __call__(self, x):
        # the device value carries the bias; it is removed here (rounded), so
        # evaluator(x) + 100 may differ from evaluate() in the last ulp
        eng = self._engine()
        if eng is None:
            raise UseAfterDispose("engine was disposed")
        dt = _DTYPES[self.precision]
        row = np.asarray(x, dtype=dt).reshape(1, -1)
        return eng.evaluate(self.fn_id, row, self.precision).values[0] - dt(catalog.VALUE_BIAS)


def _config(config) -> EngineConfig:
    """This package's EngineConfig from any config carrying the reference's
    fields (robench.EngineConfig, engine.py:34-52)."""
    if isinstance(config, EngineConfig):
        return config
    return EngineConfig(dim=config.dim, max_concurrency=config.max_concurrency, seed=config.seed,
                        precision=config.precision, threads=config.threads,
                        device=getattr(config, "device", 0))


def initialize(config) -> Engine:
    """Build every instance on the host, upload the pack, return the engine
    (engine.py:225-228).  ``config``: this package's EngineConfig or the
    reference's (a robench caller's ``robench.initialize`` can be pointed here
    unchanged)."""
    return Engine(_config(config))
