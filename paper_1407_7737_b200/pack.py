"""Flatten the host-built instances of one (dim, seed) into the device pack.

The pack is the ``rb_pack`` of include/robench_b200.h: four descriptor
tables (functions, members, segments, groups), one int32 index table and two
value tables of equal length (float64 and float32).  rb_initialize copies it
to the device once; evaluation never touches the host copy again.

Layout decisions:

* Rotations are stored per diagonal block, never dense: R is block-diagonal
  in a permuted basis (transforms.py:110-128), so only sum(n_b^2) of the
  D^2 entries exist (3 334 of 10 000 at D=100).
* Block columns are stored in *q-order*: grouped by the accumulator slot the
  column occupies in NumPy's pairwise row sum (slot = column % 8 below the
  last multiple of 8, then the sequential tail), ascending within a slot.
  The exact-order float32 rotate walks q-order and reproduces the rounding of
  ``(R * v).sum(axis=1)`` (transforms.py:42-48) bit for bit; structural zeros
  of the dense row are exact no-ops and are skipped.
* Per-(kernel, d) constant arrays that the reference builds with NumPy in the
  working dtype (elliptic weights kernels.py:66-67, powers exponents :83,
  Weierstrass series :100-106, Katsuura scalars :177-184) are computed here
  with the very same NumPy expressions in each dtype, so both sides see the
  same bits on the machine that runs them.
"""

from __future__ import annotations

import numpy as np

from . import catalog, instances

GROUP_DT = np.dtype([("m", "<i4"), ("qb", "<i4", (10,)), ("col", "<i4"),
                     ("row", "<i4"), ("mat", "<i4"), ("frag", "<i4"), ("cz", "<i4"),
                     ("col64", "<i4"), ("leaf", "<i4")])
SEGMENT_DT = np.dtype({
    "names": ["kernel", "d", "src", "n_groups", "group0", "ctab", "scale", "pre", "post"],
    "formats": ["<i4"] * 6 + ["<f8"] * 3,
    "offsets": [0, 4, 8, 12, 16, 20, 24, 32, 40], "itemsize": 48})
MEMBER_DT = np.dtype({
    "names": ["n_segments", "segment0", "shift", "perm", "sigma", "height", "bias"],
    "formats": ["<i4"] * 4 + ["<f8"] * 3,
    "offsets": [0, 4, 8, 12, 16, 24, 32], "itemsize": 40})
FUNCTION_DT = np.dtype([("category", "<i4"), ("n_members", "<i4"), ("member0", "<i4"),
                        ("reserved", "<i4")])

CATEGORY = {catalog.UNIMODAL: 0, catalog.BASIC_MULTIMODAL: 0,
            catalog.HYBRID: 1, catalog.COMPOSITION: 2}
DISABLED = -1
EXACT_ORDER_LEAF = 128  # NumPy's pairwise-sum leaf
EXACT_ORDER_STACK = 4   # device stack of pending subtree sums (every row length <= 968)


def pairwise_leaves(n: int, a: int = 0) -> list[tuple[int, int]]:
    """The leaves [a, b) of NumPy's pairwise sum of a length-n row
    (SURVEY.md Appendix A): n <= 128 is one leaf, else the row splits at
    m = n/2 rounded down to a multiple of 8."""
    if n <= EXACT_ORDER_LEAF:
        return [(a, a + n)]
    m = n // 2 - (n // 2) % 8
    return pairwise_leaves(m, a) + pairwise_leaves(n - m, a + m)


def store_row_order(pos) -> list[int]:
    """Order of a block's rows for the float32 rotate's z stores: row r is
    computed by item row-quad r // 4 (element r % 4), and a warp stores the
    same element of 4 consecutive row-quads at once (rb_device.cuh, rotate
    float), so rows 4 rq + j, 4 (rq+1) + j, ... should differ in position
    mod 8 (distinct shared-memory banks at ldz = 8 mod 32).  Greedy: avoid
    the residues of the previous 3 row-quads' row j, prefer (rq + 2j) mod 8."""
    pos = [int(p) for p in pos]
    remaining = list(range(len(pos)))
    out: list[int] = []
    for r in range(len(pos)):
        rq, j = divmod(r, 4)
        taken = {pos[out[4 * (rq - k) + j]] % 8 for k in (1, 2, 3) if rq - k >= 0}
        want = (rq + 2 * j) % 8
        cands = [i for i in remaining if pos[i] % 8 not in taken] or remaining
        pick = min(cands, key=lambda i: ((pos[i] % 8 - want) % 8, pos[i]))
        out.append(pick)
        remaining.remove(pick)
    return out


def pairwise_program(n: int) -> list[int]:
    """Post-order schedule of NumPy's pairwise tree over the leaves of a
    length-n row: entry i = how many additions follow leaf i (the ancestors
    whose last leaf is leaf i), each adding the top two pending sums
    (left + right).  Evaluated with a stack of pending sums."""
    def walk(n: int, out: list[int]) -> None:
        if n <= EXACT_ORDER_LEAF:
            out.append(0)
            return
        m = n // 2 - (n // 2) % 8
        walk(m, out)
        walk(n - m, out)
        out[-1] += 1
    out: list[int] = []
    walk(n, out)
    return out


def program_depth(prog) -> int:
    """Largest number of pending sums the schedule holds."""
    sp = best = 0
    for adds in prog:
        sp += 1
        best = max(best, sp)
        sp -= adds
    return best


def slot_of(pos: int, n: int) -> int:
    """Accumulator slot of element ``pos`` in NumPy's pairwise sum of a
    contiguous length-n row: 0..7, or 8 for the tail."""
    main = 0 if n < 8 else n - n % 8
    return pos % 8 if pos < main else 8


def kernel_constants(kernel: str, d: int, dt) -> np.ndarray:
    """Constant table of one kernel at length d, computed with the
    reference's own NumPy expressions in dtype ``dt``."""
    if kernel == "elliptic":                                   # kernels.py:66-67
        e = np.arange(d, dtype=dt) / max(d - 1, 1)
        return np.asarray(1.0e6**e, dtype=dt)
    if kernel == "powers":                                     # kernels.py:83
        return np.asarray(2.0 + 4.0 * np.arange(d, dtype=dt) / max(d - 1, 1), dtype=dt)
    if kernel == "weierstrass":                                # kernels.py:100-106
        k = np.arange(21, dtype=dt)
        ak, bk = 0.5**k, 3.0**k
        arg = 2.0 * np.pi * bk        # left operand of "* (z[:, None] + 0.5)"
        base = np.sum(ak * np.cos(np.pi * bk))
        return np.concatenate([ak, arg, np.asarray([d * base], dtype=dt)]).astype(dt)
    if kernel == "griewank":                                   # kernels.py:111-112
        root = np.sqrt(np.arange(1, d + 1, dtype=dt))
        # float32 divides by NumPy's sqrt like the reference; float64
        # multiplies by the reciprocal (parity to tolerance)
        return root if dt == np.float32 else 1.0 / root
    if kernel == "katsuura":                                   # kernels.py:183-184
        return np.asarray([10.0 / d**1.2, 10.0 / (d * d)], dtype=dt)
    return np.zeros(0, dtype=dt)


def fp64_column_order(x_col, dim: int) -> list[int]:
    """Order of a block's columns for the float64 DMMA A fragments: each
    k-step gathers 4 columns for 8 points whose X rows are ``dim`` doubles
    apart; a half-warp (4 points x 4 columns) reads shared memory without
    bank conflicts when the 16 double-banks (row_offset + column) mod 16
    are distinct.  Greedy: fill every k-step with mutually conflict-free
    columns first."""
    offs = [(g * dim) % 16 for g in range(4)]
    banks = [frozenset((o + int(c)) % 16 for o in offs) for c in x_col]
    rem = list(range(len(x_col)))
    order: list[int] = []
    while rem:
        used: set = set()
        pick: list[int] = []
        for k in rem:
            if not (banks[k] & used):
                pick.append(k)
                used |= banks[k]
                if len(pick) == 4:
                    break
        for k in rem:                     # no conflict-free 4th column: take any
            if len(pick) == 4:
                break
            if k not in pick:
                pick.append(k)
        order += pick
        rem = [k for k in rem if k not in pick]
    return order


class _Builder:
    def __init__(self, dim: int):
        self.dim = dim
        self.functions = np.zeros(catalog.FUNCTION_COUNT, dtype=FUNCTION_DT)
        self.members, self.segments, self.groups = [], [], []
        self.index: list[np.ndarray] = []
        self.n_index = 0
        self.v64: list[np.ndarray] = []
        self.v32: list[np.ndarray] = []
        self.n_values = 0
        self.max_exact_len = 0   # longest rotated segment (exact-order fp32 bound)
        self.max_q = 0           # widest per-segment sum of 4-padded group sizes
        self.max_d = 0
        self.group_src: list = []   # (block, segment positions, scale) per group

    # -- tables
    def values(self, a64, a32=None) -> int:
        """Append to both value tables; every block starts 32-byte aligned."""
        a64 = np.ascontiguousarray(a64, dtype=np.float64).ravel()
        a32 = (a64.astype(np.float32) if a32 is None
               else np.ascontiguousarray(a32, dtype=np.float32).ravel())
        assert a64.shape == a32.shape
        if self.n_values % 4:
            pad = 4 - self.n_values % 4
            self.v64.append(np.zeros(pad))
            self.v32.append(np.zeros(pad, np.float32))
            self.n_values += pad
        off = self.n_values
        self.v64.append(a64)
        self.v32.append(a32)
        self.n_values += a64.size
        return off

    def ints(self, a) -> int:
        a = np.ascontiguousarray(a, dtype=np.int32).ravel()
        off = self.n_index
        self.index.append(a)
        self.n_index += a.size
        return off

    # -- descriptors
    def group(self, block: np.ndarray, cols, rows, n: int, scale: float, pre: float,
              post: float) -> int:
        """One rotation block acting on positions ``cols`` of a length-n
        segment vector and writing positions ``rows`` of z.

        float64 rotate algebra: z = R(scale (x - o) + pre) + post
        = (scale R)(x - o) - cz with cz_r = -pre sum_q R[r, q] - post, so the
        DMMA fragments hold scale * block and x - o stays an exact zero at
        the optimum (z is then exactly post, as in the reference)."""
        m = block.shape[0]
        cols = [int(c) for c in cols]
        rorder = store_row_order(rows)             # row order is free: rows are independent
        block = block[rorder]
        rows = [int(rows[i]) for i in rorder]
        leaves = pairwise_leaves(n)
        leaf_of = [next(i for i, (a, b) in enumerate(leaves) if a <= c < b) for c in cols]

        def key(k):                      # (leaf, slot inside the leaf, position)
            a, b = leaves[leaf_of[k]]
            return (leaf_of[k], slot_of(cols[k] - a, b - a), cols[k])
        order = sorted(range(m), key=key)
        # per leaf: slot s spans q in [qb[s], qb[s+1]) (s < 8), tail [qb[8], qb[9])
        leaf_qb = []
        q0 = 0
        for li, (a, b) in enumerate(leaves):
            ks = [k for k in order if leaf_of[k] == li]
            slots = [slot_of(cols[k] - a, b - a) for k in ks]
            qb_l = q0 + np.searchsorted(np.asarray(slots, dtype=np.int64), np.arange(10), side="left")
            qb_l[9] = q0 + len(ks)
            leaf_qb.append(qb_l.astype(np.int32))
            q0 += len(ks)
        qb = leaf_qb[0] if len(leaves) == 1 else np.zeros(10, np.int32)
        mat = np.ascontiguousarray(block[:, order].T)          # mat[q, r] = block[r, order[q]]
        m4, nt, nk = (m + 3) // 4 * 4, (m + 7) // 8, (m + 3) // 4
        padded = np.zeros((nk * 4, nt * 8))
        padded[:m, :m] = mat
        rec = np.zeros((), dtype=GROUP_DT)
        rec["m"] = m
        rec["qb"] = qb
        rec["col"] = self.ints([cols[k] for k in order])
        rec["row"] = self.ints(rows)
        rec["mat"] = self.values(padded[:m, :m4])
        cz = -np.longdouble(pre) * mat.astype(np.longdouble).sum(axis=0) - np.longdouble(post)
        rec["cz"] = self.values(cz.astype(np.float64))
        rec["frag"] = rec["col64"] = -1                  # member(): needs the x columns
        # float32 rows longer than a pairwise leaf: leaf table [n_leaf, then
        # per leaf its qb (10 ints) and the additions that follow it
        # (pairwise_program)] in the index table; -1 = one leaf (qb above),
        # -2 = the tree needs more than EXACT_ORDER_STACK pending sums
        if len(leaves) == 1:
            rec["leaf"] = -1
        else:
            prog = pairwise_program(n)
            if program_depth(prog) > EXACT_ORDER_STACK:
                rec["leaf"] = -2
            else:
                table = [len(leaves)]
                for qb_l, adds in zip(leaf_qb, prog):
                    table += [int(v) for v in qb_l] + [adds]
                rec["leaf"] = self.ints(np.asarray(table, dtype=np.int32))
        self.groups.append(rec)
        self.group_src.append((block, cols, scale))
        return len(self.groups) - 1

    def fp64_layout(self, gi: int, x_col) -> None:
        """float64 DMMA operands of group gi: its own column order (the
        float64 sum order is free) and the B fragments in that order.
        ``x_col[k]``: X column feeding block column k."""
        block, cols, scale = self.group_src[gi]
        order = fp64_column_order(x_col, self.dim)
        m = block.shape[0]
        nt, nk = (m + 7) // 8, (m + 3) // 4
        padded = np.zeros((nk * 4, nt * 8))
        padded[:m, :m] = block[:, order].T                     # [q, r] = block[r, order[q]]
        lane = np.arange(32)
        # frag[nt][ks][lane] = padded[4ks + lane%4, 8nt + lane/4]
        frag = padded[(4 * np.arange(nk)[None, :, None] + lane % 4)[..., :],
                      (8 * np.arange(nt)[:, None, None] + lane // 4)]
        self.groups[gi]["frag"] = self.values(scale * frag, frag.astype(np.float32))
        self.groups[gi]["col64"] = self.ints([cols[k] for k in order])

    def segment(self, kernel: str, d: int, src: int, blocks) -> int:
        """blocks: list of (block, cols, rows) or [] when not rotated."""
        scale, pre, post = catalog.KERNEL_PIPELINE[kernel]
        g0 = len(self.groups)
        for blk, cols, rows in blocks:
            self.group(blk, cols, rows, d, scale, pre, post)
        if blocks:
            self.max_exact_len = max(self.max_exact_len, d)
            self.max_q = max(self.max_q, sum((b.shape[0] + 3) // 4 * 4 for b, _, _ in blocks))
        self.max_d = max(self.max_d, d)
        c64, c32 = kernel_constants(kernel, d, np.float64), kernel_constants(kernel, d, np.float32)
        rec = np.zeros((), dtype=SEGMENT_DT)
        rec["kernel"] = catalog.KERNEL_IDS[kernel]
        rec["d"] = d
        rec["src"] = src
        rec["n_groups"] = len(blocks)
        rec["group0"] = g0
        rec["ctab"] = self.values(c64, c32) if c64.size else 0
        rec["scale"], rec["pre"], rec["post"] = scale, pre, post
        self.segments.append(rec)
        return len(self.segments) - 1

    def member(self, shift, segs: list[int], perm=None, sigma=0.0, height=0.0, bias=0.0) -> int:
        for si in segs:
            seg = self.segments[si]
            for gi in range(int(seg["group0"]), int(seg["group0"]) + int(seg["n_groups"])):
                pos = np.asarray(self.group_src[gi][1], dtype=np.int64) + int(seg["src"])
                self.fp64_layout(gi, np.asarray(perm)[pos] if perm is not None else pos)
        rec = np.zeros((), dtype=MEMBER_DT)
        rec["n_segments"] = len(segs)
        rec["segment0"] = segs[0]
        rec["shift"] = self.values(shift)
        rec["perm"] = -1 if perm is None else self.ints(perm)
        rec["sigma"], rec["height"], rec["bias"] = sigma, height, bias
        self.members.append(rec)
        return len(self.members) - 1

    def rotated_segment(self, kernel: str, rot: instances.GroupedRotation) -> int:
        return self.segment(kernel, self.dim, 0, [(blk, idx, idx) for idx, blk in rot.groups()])

    def hybrid_segments(self, h: instances.HybridInstance) -> list[int]:
        segs, off = [], 0
        for name, n, mat in zip(h.kernels, h.sizes, h.chunk_rotations):
            ar = np.arange(n)
            segs.append(self.segment(name, n, off, [(mat, ar, ar)]))
            off += n
        return segs


class Pack:
    """Host copy of an ``rb_pack`` (numpy arrays kept alive for the FFI)."""

    def __init__(self, dim: int, seed: int, disabled=frozenset(), overrides=None):
        """``overrides``: {fn: instance} used instead of regenerating that
        function's instance from the seed (instances loaded from files)."""
        b = _Builder(dim)
        overrides = overrides or {}
        for fn in range(catalog.FUNCTION_COUNT):
            rec = b.functions[fn]
            if fn in disabled:
                rec["category"] = DISABLED
                continue
            inst = overrides[fn] if fn in overrides else instances.build(fn, dim, seed)
            row = catalog.lookup(fn)
            rec["category"] = CATEGORY[row.category]
            rec["member0"] = len(b.members)
            if isinstance(inst, instances.BasicInstance):
                if inst.rotation is None:
                    seg = b.segment(inst.kernel, dim, 0, [])
                else:
                    seg = b.rotated_segment(inst.kernel, inst.rotation)
                b.member(inst.shift, [seg])
                rec["n_members"] = 1
            elif isinstance(inst, instances.HybridInstance):
                b.member(inst.shift, b.hybrid_segments(inst), perm=inst.split_perm)
                rec["n_members"] = 1
            else:
                for k, m in enumerate(inst.members):
                    blend = dict(sigma=inst.sigma[k], height=inst.heights[k], bias=inst.biases[k])
                    if m.hybrid is not None:
                        b.member(m.shift, b.hybrid_segments(m.hybrid), perm=m.hybrid.split_perm, **blend)
                    else:
                        b.member(m.shift, [b.rotated_segment(m.kernel, m.rotation)], **blend)
                rec["n_members"] = len(inst.members)
        self.dim, self.seed = dim, seed
        self.functions = b.functions
        self.members = np.array(b.members, dtype=MEMBER_DT) if b.members else np.zeros(0, MEMBER_DT)
        self.segments = np.array(b.segments, dtype=SEGMENT_DT) if b.segments else np.zeros(0, SEGMENT_DT)
        self.groups = np.array(b.groups, dtype=GROUP_DT) if b.groups else np.zeros(1, GROUP_DT)
        self.index = np.concatenate(b.index) if b.index else np.zeros(1, np.int32)
        self.values_f64 = np.concatenate(b.v64) if b.v64 else np.zeros(1)
        self.values_f32 = np.concatenate(b.v32) if b.v32 else np.zeros(1, np.float32)
        self.max_exact_len = b.max_exact_len
        self.max_q, self.max_d = b.max_q, b.max_d
