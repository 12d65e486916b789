"""Host-side instance generation: shift vectors, grouped rotations, split
permutations, chunk rotations and composition member data.

The device pack must hold exactly the numbers the reference evaluates with,
so every datum here is drawn from the same counter-based stream the reference
uses and is post-processed with the same floating-point operations in the
same order.  Stream keys are ``SeedSequence((seed, fn, dim, *ns, tag[, k]))``
with purpose tags 1..6 (/root/reference/pkg/src/robench/transforms.py:21-39).
Bit-identity with the reference is asserted by tests/test_instances.py (live,
when /root/reference is mounted) and by the committed digests in
tests/golden/instances.json (everywhere).

This runs once per engine, on the host, in float64; the single-precision pack
is a cast of the same data (engine.py:88-94, hybrid.py:60-69,
composition.py:63-72).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from math import ceil

import numpy as np

from . import catalog
from .errors import DimensionTooSmall, RankDeficiency

TAG_SHIFT, TAG_GROUPING, TAG_BLOCK, TAG_SPLIT, TAG_CHUNK, TAG_MEMBER = 1, 2, 3, 4, 5, 6
_RANK_EPS = 1e-12      # transforms.py:27
_MAX_REDRAWS = 100     # transforms.py:32


def stream(seed: int, fn_id: int, dim: int, *tags: int) -> np.random.Generator:
    """Philox generator keyed like transforms._rng (transforms.py:37-39)."""
    key = tuple(int(t) for t in (seed, fn_id, dim, *tags))
    return np.random.Generator(np.random.Philox(np.random.SeedSequence(key)))


def shuffle_indices(rng: np.random.Generator, n: int) -> np.ndarray:
    """Descending Fisher-Yates over 0..n-1, one ``integers`` draw per step
    (transforms.py:85-91); the draw sequence fixes the permutation."""
    out = np.arange(n, dtype=np.int64)
    for top in range(n - 1, 0, -1):
        pick = int(rng.integers(0, top + 1))
        out[top], out[pick] = out[pick], out[top]
    return out


def orthonormalize(raw: np.ndarray) -> np.ndarray:
    """Columns of ``raw`` orthonormalised by modified Gram-Schmidt with one
    re-orthogonalisation sweep (transforms.py:51-72).

    The projections run on column views of a C-ordered matrix exactly as the
    reference does, because the BLAS dot kernel (and hence the rounding)
    differs between strided and contiguous operands.
    """
    q = np.array(raw, dtype=np.float64, copy=True)
    n = q.shape[0]
    for col in range(n):
        v = q[:, col]
        for _sweep in (0, 1):
            for prev in range(col):
                basis = q[:, prev]
                v -= (basis @ v) * basis
        length = np.linalg.norm(v)
        if length < _RANK_EPS:
            raise RankDeficiency(f"column {col} is numerically dependent")
        q[:, col] = v / length
    return q


def random_rotation(rng: np.random.Generator, n: int) -> np.ndarray:
    """Orthonormalised standard-normal n x n draw (transforms.py:75-82)."""
    for _ in range(_MAX_REDRAWS):
        try:
            return orthonormalize(rng.standard_normal((n, n)))
        except RankDeficiency:
            continue
    raise RankDeficiency(f"no full-rank draw in {_MAX_REDRAWS} attempts")


def group_sizes(dim: int) -> tuple[int, ...]:
    """Three near-equal coordinate groups, ceilings first (transforms.py:94-102)."""
    a = ceil(dim / 3)
    b = ceil((dim - a) / 2)
    return tuple(s for s in (a, b, dim - a - b) if s > 0)


def chunk_sizes(fractions: tuple[float, ...], dim: int) -> tuple[int, ...]:
    """Hybrid subcomponent sizes: ceil(p_i * dim) in exact integer tenths,
    remainder to the last, every chunk >= 1 (hybrid.py:19-39)."""
    tenths = [round(p * 10) for p in fractions]
    head = [(t * dim + 9) // 10 for t in tenths[:-1]]
    rest = dim - sum(head)
    while rest < 1:
        big = head.index(max(head))
        if head[big] <= 1:
            raise DimensionTooSmall(f"dimension {dim} cannot hold {len(fractions)} subcomponents")
        head[big] -= 1
        rest += 1
    return (*head, rest)


def shift(fn_id: int, dim: int, seed: int, ns: tuple[int, ...] = ()) -> np.ndarray:
    lo, hi = catalog.SHIFT_DOMAIN
    return stream(seed, fn_id, dim, *ns, TAG_SHIFT).uniform(lo, hi, dim)


@dataclass(frozen=True, eq=False)
class GroupedRotation:
    """R block-diagonal in a permuted basis: group g owns coordinates
    ``perm[off_g : off_g + n_g]`` (rows and columns) and rotates them by
    ``blocks[g]`` (transforms.py:110-128)."""

    perm: np.ndarray
    blocks: tuple[np.ndarray, ...]

    def groups(self):
        off = 0
        for blk in self.blocks:
            yield self.perm[off:off + blk.shape[0]], blk
            off += blk.shape[0]

    def dense(self) -> np.ndarray:
        dim = int(self.perm.shape[0])
        out = np.zeros((dim, dim))
        for idx, blk in self.groups():
            out[np.ix_(idx, idx)] = blk
        return out


def grouped_rotation(fn_id: int, dim: int, seed: int, ns: tuple[int, ...] = ()) -> GroupedRotation:
    perm = shuffle_indices(stream(seed, fn_id, dim, *ns, TAG_GROUPING), dim)
    blocks = tuple(random_rotation(stream(seed, fn_id, dim, *ns, TAG_BLOCK, g), n)
                   for g, n in enumerate(group_sizes(dim)))
    return GroupedRotation(perm, blocks)


@dataclass(frozen=True, eq=False)
class BasicInstance:
    fn_id: int
    kernel: str
    shift: np.ndarray
    rotation: GroupedRotation | None  # None for the shift-only ids 10, 15


@dataclass(frozen=True, eq=False)
class HybridInstance:
    fn_id: int                       # hybrid recipe id (23..28)
    kernels: tuple[str, ...]
    sizes: tuple[int, ...]
    shift: np.ndarray
    split_perm: np.ndarray
    chunk_rotations: tuple[np.ndarray, ...]


@dataclass(frozen=True, eq=False)
class Member:
    shift: np.ndarray
    kernel: str | None = None
    rotation: GroupedRotation | None = None
    hybrid: HybridInstance | None = None


@dataclass(frozen=True, eq=False)
class CompositionInstance:
    fn_id: int
    sigma: np.ndarray
    heights: np.ndarray
    biases: np.ndarray
    members: tuple[Member, ...] = field(default_factory=tuple)


def _hybrid(recipe_id: int, dim: int, seed: int, stream_fn: int,
            ns: tuple[int, ...], shift_vec: np.ndarray) -> HybridInstance:
    """hybrid._build (hybrid.py:83-95); compositions 35/36 pass their own
    stream id and member namespace."""
    row = catalog.lookup(recipe_id)
    sizes = chunk_sizes(row.fractions, dim)
    split = shuffle_indices(stream(seed, stream_fn, dim, *ns, TAG_SPLIT), dim)
    chunks = tuple(random_rotation(stream(seed, stream_fn, dim, *ns, TAG_CHUNK, k), n)
                   for k, n in enumerate(sizes))
    return HybridInstance(recipe_id, row.parts, sizes, shift_vec, split, chunks)


def member_shift(fn_id: int, dim: int, seed: int, k: int) -> np.ndarray:
    """Member optimum; member 2 sits at the origin (transforms.py:143-152)."""
    if k == 2:
        return np.zeros(dim)
    lo, hi = catalog.SHIFT_DOMAIN
    return stream(seed, fn_id, dim, TAG_MEMBER, k, TAG_SHIFT).uniform(lo, hi, dim)


def build(fn_id: int, dim: int, seed: int):
    """Instance of one function id; same data as engine._prepare
    (engine.py:107-118) builds for it."""
    row = catalog.lookup(fn_id)
    # basic-kernel compositions build from dim 2 (composition.py:75-91)
    least = catalog.MIN_DIMENSION if row.parts and row.category == catalog.COMPOSITION \
        else catalog.min_dimension(fn_id)
    if dim < least:
        raise DimensionTooSmall(f"{row.name} needs dimension >= {least}")
    if row.category in (catalog.UNIMODAL, catalog.BASIC_MULTIMODAL):
        rot = grouped_rotation(fn_id, dim, seed) if row.rotate else None
        return BasicInstance(fn_id, row.kernel, shift(fn_id, dim, seed), rot)
    if row.category == catalog.HYBRID:
        return _hybrid(fn_id, dim, seed, fn_id, (), shift(fn_id, dim, seed))
    members = []
    for k in range(row.n_members):
        o = member_shift(fn_id, dim, seed, k)
        if row.hybrid_ids:
            members.append(Member(o, hybrid=_hybrid(row.hybrid_ids[k], dim, seed, fn_id, (k,), o)))
        else:
            members.append(Member(o, kernel=row.parts[k],
                                  rotation=grouped_rotation(fn_id, dim, seed, (k,))))
    return CompositionInstance(fn_id, np.asarray(row.sigma, dtype=np.float64),
                               np.asarray(row.heights, dtype=np.float64),
                               np.asarray(row.biases, dtype=np.float64), tuple(members))
