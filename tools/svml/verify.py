"""Compare the CPU build of csrc/rb_svml_powf.cuh with np.power (float32)
bit for bit.  Usage: python tools/svml/verify.py [n_random]"""
import ctypes
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
lib = ctypes.CDLL(str(HERE / "libverify.so"))
lib.powf_np_batch.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_long]


def emu(x, y):
    x = np.ascontiguousarray(x, np.float32)
    y = np.ascontiguousarray(np.broadcast_to(y, x.shape), np.float32)
    out = np.empty_like(x)
    lib.powf_np_batch(x.ctypes.data, y.ctypes.data, out.ctypes.data, x.size)
    return out


def check(name, x, y):
    want = np.power(x.astype(np.float32), np.float32(y) if np.isscalar(y) else y.astype(np.float32))
    got = emu(x, y)
    bad = got.view(np.uint32) != want.view(np.uint32)
    # rare lanes are not emulated: exclude |y*log2 x| > 125 from the score
    print(f"{name:28s} n={x.size:9d} mismatches={int(bad.sum())}")
    if bad.any():
        i = np.flatnonzero(bad)[:5]
        print("   x", x.ravel()[i], "y", np.broadcast_to(y, x.shape).ravel()[i],
              "got", got.ravel()[i], "want", want.ravel()[i])
    return int(bad.sum())


n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
rng = np.random.default_rng(0)
bad = 0
for y in (0.2, -0.5, 0.25, 2.5, 6.0):   # (scalar 2.0 takes NumPy's x*x fast path)
    x = np.exp(rng.uniform(np.log(1e-6), np.log(1e6), n)).astype(np.float32)
    bad += check(f"y={y}", x, y)
# POWERS exponents 2 + 4 i / (d-1) for the suite dims, z in [-200, 200]
for d in (10, 30, 50, 100):
    e = (2.0 + 4.0 * np.arange(d, dtype=np.float32) / max(d - 1, 1)).astype(np.float32)
    x = np.abs(rng.uniform(-200, 200, (n // d, d))).astype(np.float32)
    bad += check(f"powers d={d}", x, np.broadcast_to(e, x.shape).copy())
# random bit patterns of positive normal floats with random exponents
xb = rng.integers(0x30000000, 0x4f000000, n, dtype=np.uint32).view(np.float32)
yy = rng.uniform(-3, 3, n).astype(np.float32)
q = np.abs(yy * np.log2(xb.astype(np.float64)))
keep = q < 120
bad += check("random x, y", xb[keep], yy[keep])
print("TOTAL mismatches", bad)
