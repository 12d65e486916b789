"""CPU ORACLE — test infrastructure only, never part of the product path.

A NumPy restatement of the reference's evaluation path
(/root/reference/pkg/src/robench/engine.py:174-214 and everything below it):
the shift/scale/rotate pipeline (engine.py:96-104, transforms.py:42-48), the
21 kernels (kernels.py:52-228), hybrids (hybrid.py:98-116) and compositions
(composition.py:114-166).  Every expression keeps the reference's operand
order and its NumPy call shapes (array vs scalar, ``**2`` vs ``np.power``)
so single precision reproduces the reference's float32 rounding bit for bit
under the same NumPy (NEP 50 weak Python scalars, pairwise ``sum``).

Instance data comes from :mod:`paper_1407_7737_b200.instances` — shared
input, as in the reference's own oracle (pkg/tests/reference.py:1-8); those
generators are pinned bit-exact to the reference by tests/test_instances.py
and tests/golden/instances.json.

Pinning: tests/test_oracle_pin.py compares this module bit-for-bit with the
live reference (when /root/reference is mounted) and with the committed
golden vectors in tests/golden/ (always).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline leg may
import this module.
"""

from __future__ import annotations

import numpy as np

from paper_1407_7737_b200 import catalog, instances

BIAS = 100.0
DTYPES = {"double": np.float64, "single": np.float32}

# kernels.py:22-42
W_A, W_B, W_KMAX = 0.5, 3.0, 20
SCHWEFEL_SHIFT, SCHWEFEL_OFFSET = 420.9687462275036, 418.9829
KATSUURA_TERMS = 32
LUN_MU1, LUN_MU2, LUN_D, LUN_S = 2.5, -2.5, 1.0, 0.9
COND, SHARP_W = 1.0e6, 100.0


class NonFinite(ValueError):
    pass


def _finite(z):
    z = np.asarray(z)
    if not np.all(np.isfinite(z)):
        raise NonFinite("kernel input contains NaN or infinity")  # kernels.py:45-49
    return z


# ----------------------------------------------------------------- kernels
# One function per kernel; z is the transformed 1-D vector.  Line numbers
# refer to /root/reference/pkg/src/robench/kernels.py.

def k_sphere(z):                                   # :52-54
    return np.sum(z * z)


def k_ellipsoid(z):                                # :57-60
    w = np.arange(1, z.shape[-1] + 1, dtype=z.dtype)
    return np.sum(w * z * z)


def k_elliptic(z):                                 # :63-67
    d = z.shape[-1]
    e = np.arange(d, dtype=z.dtype) / max(d - 1, 1)
    return np.sum(COND**e * z * z)


def k_discus(z):                                   # :70-72
    return COND * z[0] * z[0] + np.sum(z[1:] * z[1:])


def k_cigar(z):                                    # :75-77
    return z[0] * z[0] + COND * np.sum(z[1:] * z[1:])


def k_powers(z):                                   # :80-84
    d = z.shape[-1]
    e = 2.0 + 4.0 * np.arange(d, dtype=z.dtype) / max(d - 1, 1)
    return np.sqrt(np.sum(np.abs(z) ** e))


def k_sharp_valley(z):                             # :87-89
    return z[0] * z[0] + SHARP_W * np.sqrt(np.sum(z[1:] * z[1:]))


def k_step(z):                                     # :92-95
    r = np.floor(z + 0.5)
    return np.sum(r * r)


def k_weierstrass(z):                              # :98-106
    k = np.arange(W_KMAX + 1, dtype=z.dtype)
    ak, bk = W_A**k, W_B**k
    grid = ak * np.cos(2.0 * np.pi * bk * (z[:, None] + 0.5))
    base = np.sum(ak * np.cos(np.pi * bk))
    return np.sum(grid) - z.shape[-1] * base


def k_griewank(z):                                 # :109-112
    w = np.arange(1, z.shape[-1] + 1, dtype=z.dtype)
    return np.sum(z * z) / 4000.0 - np.prod(np.cos(z / np.sqrt(w))) + 1.0


def k_rastrigin(z):                                # :115-117
    return np.sum(z * z - 10.0 * np.cos(2.0 * np.pi * z) + 10.0)


def k_schaffers_f7(z):                             # :120-127
    d = z.shape[-1]
    if d < 2:
        return z.dtype.type(0)
    w = np.sqrt(z[:-1] ** 2 + z[1:] ** 2)
    t = np.sqrt(w) * (1.0 + np.sin(50.0 * w**0.2) ** 2)
    return (np.sum(t) / (d - 1)) ** 2


def _rosen_link(x, y):                             # :130-132
    return 100.0 * (x * x - y) ** 2 + (x - 1.0) ** 2


def _griewank_1d(x):                               # :135-137
    return x * x / 4000.0 - np.cos(x) + 1.0


def k_grie_rosen(z):                               # :140-142
    return np.sum(_griewank_1d(_rosen_link(z, np.roll(z, -1))))


def k_rosenbrock(z):                               # :145-149
    a, b = z[:-1], z[1:]
    return np.sum(100.0 * (a * a - b) ** 2 + (a - 1.0) ** 2)


def _schwefel_term(w, d):                          # :152-165
    aw = np.abs(w)
    mid = w * np.sin(np.sqrt(aw))
    top = 500.0 - np.mod(w, 500.0)
    hi = top * np.sin(np.sqrt(top)) - (w - 500.0) ** 2 / (10000.0 * d)
    rem = np.mod(-w, 500.0)
    lo = (rem - 500.0) * np.sin(np.sqrt(500.0 - rem)) - (w + 500.0) ** 2 / (10000.0 * d)
    return np.where(aw <= 500.0, mid, np.where(w > 500.0, hi, lo))


def k_schwefel(z):                                 # :168-171
    d = z.shape[-1]
    return SCHWEFEL_OFFSET * d - np.sum(_schwefel_term(z + SCHWEFEL_SHIFT, d))


def k_katsuura(z):                                 # :174-184
    d = z.shape[-1]
    p2 = 2.0 ** np.arange(1, KATSUURA_TERMS + 1, dtype=z.dtype)
    w = p2 * z[:, None]
    s = np.sum(np.abs(w - np.floor(w + 0.5)) / p2, axis=1)
    t = 1.0 + np.arange(1, d + 1, dtype=z.dtype) * s
    lp = (10.0 / d**1.2) * np.sum(np.log(t))
    return (10.0 / (d * d)) * np.expm1(lp)


def k_lunacek(z):                                  # :187-193
    d = z.shape[-1]
    a, b = z - LUN_MU1, z - LUN_MU2
    funnel = np.minimum(np.sum(a * a), LUN_D * d + LUN_S * np.sum(b * b))
    return funnel + 10.0 * (d - np.sum(np.cos(2.0 * np.pi * a)))


def k_ackley(z):                                   # :196-201
    d = z.shape[-1]
    rms = np.sqrt(np.sum(z * z) / d)
    mc = np.sum(np.cos(2.0 * np.pi * z)) / d
    return -20.0 * np.exp(-0.2 * rms) - np.exp(mc) + 20.0 + np.e


def k_happycat(z):                                 # :204-209
    d = z.shape[-1]
    r2, sz = np.sum(z * z), np.sum(z)
    return np.abs(r2 - d) ** 0.25 + (0.5 * r2 + sz) / d + 0.5


def k_hgbat(z):                                    # :212-217
    d = z.shape[-1]
    r2, sz = np.sum(z * z), np.sum(z)
    return np.sqrt(np.abs(r2 * r2 - sz * sz)) + (0.5 * r2 + sz) / d + 0.5


def _f6_link(x, y):                                # :220-223
    q = x * x + y * y
    return (np.sin(np.sqrt(q)) ** 2 - 0.5) / (1.0 + 0.001 * q) ** 2 + 0.5


def k_schaffers_f6(z):                             # :226-228
    return np.sum(_f6_link(z, np.roll(z, -1)))


KERNELS = {name: globals()["k_" + name] for name in catalog.KERNEL_NAMES}


def kernel(name, z):
    return KERNELS[name](_finite(z))


# -------------------------------------------------------------- pipeline

def rotate(mat, v):
    """transforms.matvec (transforms.py:42-48): rounded products, then the
    pairwise row sum."""
    return (mat * v).sum(axis=1)


def _pipeline(name, x_minus_o, mat):
    """engine._BasicEvaluator.__call__ (engine.py:96-104) / composition
    _member_value (composition.py:147-154) / one hybrid chunk
    (hybrid.py:108-114): scale, +pre, rotate, +post."""
    scale, pre, post = catalog.KERNEL_PIPELINE[name]
    v = scale * x_minus_o
    if pre:
        v = v + pre
    if mat is not None:
        v = rotate(mat, v)
    if post:
        v = v + post
    return kernel(name, v)


class _Basic:
    def __init__(self, inst, dt):
        self.name = inst.kernel
        self.o = inst.shift.astype(dt)
        self.mat = None if inst.rotation is None else inst.rotation.dense().astype(dt)

    def __call__(self, x):
        return _pipeline(self.name, x - self.o, self.mat)


class _Hybrid:
    def __init__(self, inst, dt):
        self.inst = inst
        self.o = inst.shift.astype(dt)
        self.mats = tuple(r.astype(dt) for r in inst.chunk_rotations)

    def __call__(self, x):                         # hybrid.py:98-116
        s = (x - self.o)[self.inst.split_perm]
        total = x.dtype.type(0)
        off = 0
        for name, n, mat in zip(self.inst.kernels, self.inst.sizes, self.mats):
            scale, pre, post = catalog.KERNEL_PIPELINE[name]
            v = scale * s[off:off + n]
            if pre:
                v = v + pre
            z = rotate(mat, v)
            if post:
                z = z + post
            total = total + kernel(name, z)
            off += n
        return total


class _Composition:
    def __init__(self, inst, dt):
        self.dim = inst.members[0].shift.shape[0]
        self.sigma = inst.sigma.astype(dt)
        self.heights = inst.heights.astype(dt)
        self.biases = inst.biases.astype(dt)
        self.opt = tuple(m.shift.astype(dt) for m in inst.members)
        self.parts = []
        for m in inst.members:
            if m.hybrid is not None:
                self.parts.append(_Hybrid(m.hybrid, dt))
            else:
                self.parts.append((m.kernel, m.shift.astype(dt), m.rotation.dense().astype(dt)))

    def weights(self, x):                          # composition.py:114-141
        n = len(self.opt)
        d2 = np.empty(n, dtype=x.dtype)
        for k, o in enumerate(self.opt):
            dx = x - o
            d2[k] = np.sum(dx * dx)
        om = np.zeros(n, dtype=x.dtype)
        if np.min(d2) < 1e-12**2:
            om[int(np.argmin(d2))] = 1
            return om
        w = d2**-0.5 * np.exp(-d2 / (2.0 * self.dim * self.sigma**2))
        tot = np.sum(w)
        if tot == 0:
            om[:] = 1.0 / n
            return om
        return w / tot

    def __call__(self, x):                         # composition.py:157-166
        om = self.weights(x)
        total = x.dtype.type(0)
        for k, part in enumerate(self.parts):
            if om[k] == 0:
                continue
            if isinstance(part, _Hybrid):
                g = part(x)
            else:
                name, o, mat = part
                g = _pipeline(name, x - o, mat)
            total = total + om[k] * (self.heights[k] * g + self.biases[k])
        return total


def evaluator(fn_id, dim, seed, precision="double"):
    """Per-point callable without the bias (engine._prepare, engine.py:107-118)."""
    dt = DTYPES[precision]
    inst = instances.build(fn_id, dim, seed)
    if isinstance(inst, instances.BasicInstance):
        return _Basic(inst, dt)
    if isinstance(inst, instances.HybridInstance):
        return _Hybrid(inst, dt)
    return _Composition(inst, dt)


class Oracle:
    """All evaluators of one (dim, seed), built lazily."""

    def __init__(self, dim, seed=0):
        self.dim, self.seed = int(dim), int(seed)
        self._cache = {}

    def evaluator(self, fn_id, precision):
        key = (int(fn_id), precision)
        if key not in self._cache:
            self._cache[key] = evaluator(fn_id, self.dim, self.seed, precision)
        return self._cache[key]

    def evaluate(self, fn_id, X, precision="double"):
        """Engine.evaluate's hot loop (engine.py:201-209): cast, finiteness
        check, one evaluator call per row, + 100 in the batch dtype."""
        dt = DTYPES[precision]
        pts = np.ascontiguousarray(X, dtype=dt)
        if not np.all(np.isfinite(pts)):
            raise NonFinite("batch contains NaN or infinity")
        f = self.evaluator(fn_id, precision)
        out = np.empty(pts.shape[0], dtype=dt)
        for i in range(pts.shape[0]):
            out[i] = f(pts[i]) + BIAS
        return out


def population(dim, n, seed=0, rows=None):
    """Synthetic U[-100,100]^{n x dim} population of SURVEY.md §8d (Philox
    keyed (seed, dim, n, 1001), bench.py:75-81 style)."""
    rng = np.random.Generator(np.random.Philox(np.random.SeedSequence((seed, dim, n, 1001))))
    x = rng.uniform(-100.0, 100.0, (n, dim))
    return x if rows is None else x[rows]
