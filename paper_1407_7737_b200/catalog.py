"""The 37-function table of the suite, as data the device pack is built from.

Restates the reference catalog (/root/reference/pkg/src/robench/catalog.py):
suite constants (catalog.py:16-22), the per-kernel input pipeline
``z = R(scale*(x - o) + pre) + post`` (catalog.py:84-106), the 37 function
rows (catalog.py:124-212) and the id -> kernel map (catalog.py:215-221).

Kernels are numbered 0..20 (``KERNEL_IDS``); the same numbering is the
``rb_kernel`` enum of the CUDA side (csrc/rb_kernels.cuh).
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import UnknownFunction

SEARCH_DOMAIN = (-100.0, 100.0)
SHIFT_DOMAIN = (-70.0, 70.0)
VALUE_BIAS = 100.0
FUNCTION_COUNT = 37
MIN_DIMENSION = 2
MIN_CONSTRUCTED_DIMENSION = 10

UNIMODAL, BASIC_MULTIMODAL, HYBRID, COMPOSITION = (
    "unimodal", "basic-multimodal", "hybrid", "composition")

# kernel name -> (scale, pre_offset, post_offset); every kernel is rotated
# unless the function row says otherwise (catalog.py:84-106).
KERNEL_PIPELINE: dict[str, tuple[float, float, float]] = {
    "sphere": (1.0, 0.0, 0.0),
    "ellipsoid": (1.0, 0.0, 0.0),
    "elliptic": (1.0, 0.0, 0.0),
    "discus": (1.0, 0.0, 0.0),
    "cigar": (1.0, 0.0, 0.0),
    "powers": (0.01, 0.0, 0.0),
    "sharp_valley": (1.0, 0.0, 0.0),
    "step": (1.0, 0.0, 0.0),
    "weierstrass": (0.005, 0.0, 0.0),
    "griewank": (6.0, 0.0, 0.0),
    "rastrigin": (0.0512, 0.0, 0.0),
    "schaffers_f7": (1.0, 0.0, 0.0),
    "grie_rosen": (0.05, 0.0, 1.0),
    "rosenbrock": (0.02048, 0.0, 1.0),
    "schwefel": (10.0, 0.0, 0.0),
    "katsuura": (0.05, 0.0, 0.0),
    "lunacek": (0.1, 2.5, 0.0),
    "ackley": (1.0, 0.0, 0.0),
    "happycat": (0.05, 0.0, -1.0),
    "hgbat": (0.05, 0.0, -1.0),
    "schaffers_f6": (1.0, 0.0, 0.0),
}
KERNEL_NAMES: tuple[str, ...] = tuple(KERNEL_PIPELINE)
KERNEL_IDS: dict[str, int] = {name: i for i, name in enumerate(KERNEL_NAMES)}


@dataclass(frozen=True)
class FunctionRow:
    fn_id: int
    name: str
    category: str
    kernel: str | None = None          # basic functions
    rotate: bool = True                # basic functions
    fractions: tuple[float, ...] = ()  # hybrids
    parts: tuple[str, ...] = ()        # hybrid chunk kernels / composition basic members
    sigma: tuple[float, ...] = ()      # compositions
    heights: tuple[float, ...] = ()
    biases: tuple[float, ...] = ()
    hybrid_ids: tuple[int, ...] = ()   # compositions of hybrids (35, 36)

    @property
    def n_members(self) -> int:
        return len(self.hybrid_ids) or len(self.parts)


_BASIC = (
    ("SPHERE", UNIMODAL, "sphere"), ("ELLIPSOID", UNIMODAL, "ellipsoid"),
    ("ELLIPTIC", UNIMODAL, "elliptic"), ("DISCUS", UNIMODAL, "discus"),
    ("CIGAR", UNIMODAL, "cigar"), ("POWERS", UNIMODAL, "powers"),
    ("SHARPV", UNIMODAL, "sharp_valley"), ("STEP", BASIC_MULTIMODAL, "step"),
    ("WEIERSTRASS", BASIC_MULTIMODAL, "weierstrass"),
    ("GRIEWANK", BASIC_MULTIMODAL, "griewank"),
    ("RARSTRIGIN_U", BASIC_MULTIMODAL, "rastrigin"),
    ("RARSTRIGIN", BASIC_MULTIMODAL, "rastrigin"),
    ("SCHAFFERSF7", BASIC_MULTIMODAL, "schaffers_f7"),
    ("GRIE_ROSEN", BASIC_MULTIMODAL, "grie_rosen"),
    ("ROSENBROCK", BASIC_MULTIMODAL, "rosenbrock"),
    ("SCHWEFEL_U", BASIC_MULTIMODAL, "schwefel"),
    ("SCHWEFEL", BASIC_MULTIMODAL, "schwefel"),
    ("KATSUURA", BASIC_MULTIMODAL, "katsuura"),
    ("LUNACEK", BASIC_MULTIMODAL, "lunacek"), ("ACKLEY", BASIC_MULTIMODAL, "ackley"),
    ("HAPPYCAT", BASIC_MULTIMODAL, "happycat"), ("HGBAT", BASIC_MULTIMODAL, "hgbat"),
    ("SCHAFFERSF6", BASIC_MULTIMODAL, "schaffers_f6"),
)
_UNROTATED = {10, 15}

_HYBRIDS = (  # catalog.py:147-164
    ((0.3, 0.3, 0.4), ("schwefel", "rastrigin", "elliptic")),
    ((0.3, 0.3, 0.4), ("cigar", "hgbat", "rastrigin")),
    ((0.2, 0.2, 0.3, 0.3), ("griewank", "weierstrass", "rosenbrock", "schaffers_f6")),
    ((0.2, 0.2, 0.3, 0.3), ("hgbat", "discus", "grie_rosen", "rastrigin")),
    ((0.1, 0.2, 0.2, 0.2, 0.3), ("schaffers_f6", "hgbat", "rosenbrock", "schwefel", "elliptic")),
    ((0.1, 0.2, 0.2, 0.2, 0.3), ("katsuura", "happycat", "grie_rosen", "schwefel", "ackley")),
)

_B5 = (0.0, 100.0, 200.0, 300.0, 400.0)
_B3 = (0.0, 100.0, 200.0)
_COMPOSITIONS = (  # catalog.py:165-211: (sigma, heights, biases, members)
    ((10.0, 20.0, 30.0, 40.0, 50.0), (1e-10, 1e-6, 1e-26, 1e-6, 1e-6), _B5,
     ("rosenbrock", "elliptic", "cigar", "discus", "elliptic")),
    ((15.0, 15.0, 15.0), (1.0, 1.0, 1.0), _B3, ("schwefel", "rastrigin", "hgbat")),
    ((20.0, 50.0, 40.0), (0.25, 1.0, 1e-7), _B3, ("schwefel", "rastrigin", "elliptic")),
    ((20.0, 15.0, 10.0, 10.0, 40.0), (2.5e-2, 0.1, 1e-8, 0.25, 1.0), _B5,
     ("schwefel", "happycat", "elliptic", "weierstrass", "griewank")),
    ((15.0, 15.0, 15.0, 15.0, 15.0), (10.0, 10.0, 2.5, 2.5, 1e-6), _B5,
     ("hgbat", "rastrigin", "elliptic", "weierstrass", "schwefel")),
    ((10.0, 20.0, 30.0, 40.0, 50.0), (2.5, 10.0, 2.5, 5e-4, 1e-6), _B5,
     ("grie_rosen", "happycat", "schwefel", "schaffers_f6", "elliptic")),
    ((10.0, 30.0, 50.0), (1.0, 1.0, 1.0), _B3, (23, 24, 25)),
    ((10.0, 30.0, 50.0), (1.0, 1.0, 1.0), _B3, (26, 27, 28)),
)


def _rows() -> tuple[FunctionRow, ...]:
    rows = [FunctionRow(i, name, cat, kernel=k, rotate=i not in _UNROTATED)
            for i, (name, cat, k) in enumerate(_BASIC)]
    for h, (fractions, parts) in enumerate(_HYBRIDS):
        fn = 23 + h
        rows.append(FunctionRow(fn, f"HYBRID{h + 1}", HYBRID,
                                fractions=fractions, parts=parts))
    for c, (sigma, heights, biases, members) in enumerate(_COMPOSITIONS):
        fn = 29 + c
        hybrid = isinstance(members[0], int)
        rows.append(FunctionRow(
            fn, f"COMPOSITION{c + 1}", COMPOSITION, sigma=sigma, heights=heights,
            biases=biases, parts=() if hybrid else members,
            hybrid_ids=members if hybrid else ()))
    return tuple(rows)


FUNCTIONS: tuple[FunctionRow, ...] = _rows()
BASIC_KERNELS: dict[int, str] = {r.fn_id: r.kernel for r in FUNCTIONS if r.kernel}


def lookup(fn_id) -> FunctionRow:
    """Catalog row for ``fn_id``; UnknownFunction outside 0..36 (catalog.py:224-229)."""
    fn_id = int(fn_id)
    if not 0 <= fn_id < FUNCTION_COUNT:
        raise UnknownFunction(f"function id {fn_id} is not in 0..{FUNCTION_COUNT - 1}")
    return FUNCTIONS[fn_id]


def min_dimension(fn_id) -> int:
    row = lookup(fn_id)
    return MIN_CONSTRUCTED_DIMENSION if row.category in (HYBRID, COMPOSITION) else MIN_DIMENSION
