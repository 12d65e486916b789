"""B200-native batched evaluation of the cuROB / robench test-function suite.

Drop-in for the reference package's evaluation API
(/root/reference/pkg/src/robench/__init__.py:30-37): ``initialize``,
``EngineConfig``, ``PointBatch``, ``EvalResult``, ``Engine.evaluate``,
``Engine.evaluate_single_precision``, ``Engine.dispose`` and the error
classes.  Evaluation runs in hand-written sm_100a kernels (csrc/rb_device.cuh,
rb_kernels.cuh, rb_fnspec.cuh; instantiated in csrc/rb_kern_*.cu) behind the
C ABI of include/robench_b200.h (csrc/rb_capi.cu).  Multi-GPU: dist.py.
"""

from .catalog import (FUNCTION_COUNT, FUNCTIONS, SEARCH_DOMAIN, SHIFT_DOMAIN, VALUE_BIAS,
                      lookup)
from .errors import (BatchTooLarge, BenchmarkError, CorruptInstance, DeviceError,
                     DimensionMismatch, DimensionTooSmall, DisabledFunction, NonFiniteInput,
                     ParseError, RankDeficiency, UnknownFunction, UnsupportedAtDim2,
                     UseAfterDispose)
from .engine import (CapturedEvaluation, Engine, EngineConfig, EvalResult, Pending, PointBatch,
                     initialize)

__version__ = "0.1.0"
