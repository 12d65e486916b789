"""On-device population source: the synthetic
population of the measurement protocol generated directly in device memory,
bit-identical to what the host would draw.

SURVEY.md §8d defines the workload population as

    X = numpy.random.Generator(numpy.random.Philox(
            numpy.random.SeedSequence((0, D, N, 1001)))).uniform(-100, 100, (N, D))

in the style of the reference's ``protocol_points`` (bench.py:75-81).  At
N = 10^7, D = 100 that is 8 GB: drawing it on the host and copying it over
PCIe would dwarf the evaluation.  ``uniform_population`` runs numpy's own
Philox4x64-10 stream on the device (``rb_uniform_population``): the key is
taken from the same SeedSequence on the host, element e of the stream comes
from counter block e // 4 + 1, word e % 4, so any row range -- a shard of a
multi-GPU run, or a sampled row for a parity check -- is produced
independently and equals the host draw bit for bit (tests/test_population.py).
"""

from __future__ import annotations

import numpy as np

from . import _lib, catalog

POINTS_STREAM = 1001           # purpose tag of the population stream (bench.py:34)


def philox_key(entropy) -> tuple[int, int]:
    """numpy.random.Philox's key for SeedSequence(entropy)."""
    state = np.random.Philox(np.random.SeedSequence(entropy)).state["state"]
    k = state["key"]
    assert not np.any(state["counter"]), "fresh Philox streams start at counter 0"
    return int(k[0]), int(k[1])


def workload_entropy(dim: int, n: int, seed: int = 0) -> tuple[int, ...]:
    """SeedSequence entropy of the §8d workload population."""
    return (int(seed), int(dim), int(n), POINTS_STREAM)


def uniform_population(dim: int, n_rows: int, entropy, first_row: int = 0, device=None,
                       dtypes=("double",)):
    """Rows [first_row, first_row + n_rows) of the (N, dim) population drawn
    from ``Generator(Philox(SeedSequence(entropy))).uniform(-100, 100)``, as
    CUDA tensors: {"double": float64 (n_rows, dim), "single": float32 copy
    rounded from it (the reference casts the float64 batch, engine.py:201)}."""
    import torch

    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    k0, k1 = philox_key(entropy)
    lo, hi = catalog.SEARCH_DOMAIN
    out = {}
    x64 = torch.empty((n_rows, dim), dtype=torch.float64, device=dev) if "double" in dtypes else None
    x32 = torch.empty((n_rows, dim), dtype=torch.float32, device=dev) if "single" in dtypes else None
    stream = torch.cuda.current_stream(dev).cuda_stream
    with torch.cuda.device(dev):
        _lib.check(_lib.load().rb_uniform_population(
            k0, k1, first_row * dim, n_rows * dim, lo, hi,
            x64.data_ptr() if x64 is not None else None,
            x32.data_ptr() if x32 is not None else None, stream))
    if x64 is not None:
        out["double"] = x64
    if x32 is not None:
        out["single"] = x32
    return out


def host_rows(dim: int, entropy, first_row: int, n_rows: int) -> np.ndarray:
    """The same rows drawn on the host with numpy (the checker), for row
    ranges that start on a 4-element boundary of the stream."""
    first = first_row * dim
    if first % 4:
        raise ValueError("host_rows needs first_row * dim to be a multiple of 4")
    bg = np.random.Philox(np.random.SeedSequence(entropy))
    bg.advance(first // 4)
    lo, hi = catalog.SEARCH_DOMAIN
    return np.random.Generator(bg).uniform(lo, hi, (n_rows, dim))
