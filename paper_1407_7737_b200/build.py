"""Compile the native library in-tree: csrc/*.cu -> librobench_b200.so.

nvcc for sm_100a only.  -fmad=false keeps every product individually
rounded (NumPy semantics; explicit fma()/mma are unaffected); no fast-math,
so division, square root and denormals are IEEE.  -lineinfo lets ncu's
source page map back to csrc/.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent
LIB = HERE / "librobench_b200.so"
SOURCES = [HERE / "csrc" / n for n in ("rb_capi.cu", "rb_kern_f64.cu", "rb_kern_f32.cu",
                                       "rb_kern_f64x.cu", "rb_kern_f32x.cu")]
DEPS = SOURCES + sorted((HERE / "csrc").glob("*.cuh")) + [ROOT / "include" / "robench_b200.h"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-fmad=false",
    "-Xcompiler", "-fPIC", "-Xptxas", "-v",
    "-I", str(ROOT / "include"),
]


def nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


def stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in DEPS)


def _compile(src: Path, extra=(), tag="") -> tuple[Path, str]:
    obj = HERE / "build" / (src.stem + tag + ".o")
    obj.parent.mkdir(exist_ok=True)
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-c", "-o", str(obj), str(src)]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src.name} ({proc.returncode}):\n{proc.stderr[-4000:]}")
    return obj, proc.stdout + proc.stderr


def build(force: bool = False, verbose: bool = False, extra=(), out: Path | None = None) -> Path:
    """Compile the translation units in parallel, then link the shared library.
    ``extra``/``out`` build tuning variants (tools/variants.sh) next to it."""
    lib = out or LIB
    if not force and not extra and not stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    tag = "" if out is None else "_" + Path(out).stem
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as pool:
        results = list(pool.map(lambda s: _compile(s, extra, tag), SOURCES))
    log = "".join(f"== {src.name}\n{out}" for src, (_, out) in zip(SOURCES, results))
    link = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(lib),
            *[str(o) for o, _ in results], "-lcudart"]
    proc = subprocess.run(link, capture_output=True, text=True)
    log += proc.stdout + proc.stderr
    (HERE / ("build.log" if out is None else f"build{tag}.log")).write_text(log)
    if proc.returncode != 0:
        raise RuntimeError(f"link failed ({proc.returncode}):\n{log[-4000:]}")
    if verbose:
        print(log)
    return lib


if __name__ == "__main__":
    # python build.py [--force] [--out PATH -DNAME=VAL ...]
    args = sys.argv[1:]
    out = Path(args[args.index("--out") + 1]) if "--out" in args else None
    extra = [a for a in args if a.startswith("-D")]
    build(force="--force" in args or out is not None, verbose=out is None, extra=extra, out=out)
