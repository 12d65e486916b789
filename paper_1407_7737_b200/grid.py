"""Landscape grid export on the GPU.

The reference's ``robench grid`` (cli.py:72-91) evaluates a K x K grid of
2-D points with ``scalar_evaluator`` (engine.py:121-138) in a Python double
loop -- 10 201 scalar calls for the default 101 x 101 grid.  Here the grid
is one batched evaluation of K^2 rows through the same kernels as every
other evaluation: row i fixes coordinate 1 at node i, column j fixes
coordinate 2 at node j, nodes ``np.linspace(lo, hi, K)``; the result is
written in the reference's grid format (fileio.write_grid).

As in the reference, functions that embed hybrids (ids 23-28, 35, 36)
cannot be evaluated at D = 2 (UnsupportedAtDim2); compositions of basic
members are built at D = 2 the way scalar_evaluator builds them.
"""

from __future__ import annotations

import numpy as np

from . import catalog
from .engine import Engine, EngineConfig
from .errors import UnsupportedAtDim2


def landscape(fn_id: int, seed: int = 0, lo: float = -100.0, hi: float = 100.0,
              steps: int = 101, precision: str = "double", device: int = 0) -> np.ndarray:
    """K x K values (bias included) of function ``fn_id`` at D = 2."""
    row = catalog.lookup(fn_id)
    if row.category == catalog.HYBRID or row.hybrid_ids:
        raise UnsupportedAtDim2(f"function {fn_id} ({row.name}) embeds hybrids and cannot be "
                                f"evaluated on a 2-D grid")
    if not lo < hi:
        raise ValueError("need lo < hi")
    nodes = np.linspace(lo, hi, steps)
    pts = np.empty((steps * steps, 2))
    pts[:, 0] = np.repeat(nodes, steps)          # row i: coordinate 1 = nodes[i]
    pts[:, 1] = np.tile(nodes, steps)            # column j: coordinate 2 = nodes[j]
    engine = Engine(EngineConfig(dim=2, max_concurrency=steps * steps, seed=seed, device=device),
                    enabled=(fn_id,))
    try:
        values = engine.evaluate(fn_id, pts, precision=precision).values
    finally:
        engine.dispose()
    return np.asarray(values, dtype=np.float64).reshape(steps, steps)


def export_grid(path, fn_id: int, seed: int = 0, lo: float = -100.0, hi: float = 100.0,
                steps: int = 101) -> np.ndarray:
    """``robench grid`` (cli.py:72-91): compute and write the grid file."""
    from .fileio import write_grid

    values = landscape(fn_id, seed, lo, hi, steps)
    write_grid(path, fn_id, seed, lo, hi, values)
    return values
