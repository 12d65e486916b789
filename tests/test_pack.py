"""Pack invariants and the exact-order rotate schedule: walking a group's
columns in q-order with the 8-slot fold reproduces NumPy's float32
``(R * v).sum(axis=1)`` (transforms.py:42-48) bit for bit — the schedule the
float32 CUDA rotate executes."""

import numpy as np
import pytest

from paper_1407_7737_b200 import catalog, instances, pack as P

F32 = np.float32


def _leaf_sum(v, cols, mat, qb, r):
    t0 = t1 = t2 = F32(0)
    for s in range(8):
        acc = F32(0)
        for q in range(qb[s], qb[s + 1]):
            acc = F32(acc + F32(v[cols[q]] * mat[q, r]))
        if s == 0:
            t0 = acc
        elif s == 1:
            t0 = F32(t0 + acc)
        elif s in (2, 4):
            t1 = acc
        elif s == 3:
            t1 = F32(t1 + acc)
            t0 = F32(t0 + t1)
        elif s == 5:
            t1 = F32(t1 + acc)
        elif s == 6:
            t2 = acc
        else:
            t2 = F32(t2 + acc)
            t1 = F32(t1 + t2)
            t0 = F32(t0 + t1)
    for q in range(qb[8], qb[9]):
        t0 = F32(t0 + F32(v[cols[q]] * mat[q, r]))
    return t0


def exact_order_rotate(pk, group, v):
    m = int(group["m"])
    cols = pk.index[group["col"]:group["col"] + m]
    rows = pk.index[group["row"]:group["row"] + m]
    m4 = (m + 3) // 4 * 4                      # rows 4-padded (float4 loads)
    mat = pk.values_f32[group["mat"]:group["mat"] + m * m4].reshape(m, m4)
    leaf = int(group["leaf"])
    assert leaf != -2
    if leaf < 0:
        qbs, prog = [group["qb"]], [0]
    else:                                      # [n_leaf, (qb[10], additions) per leaf]
        nl = int(pk.index[leaf])
        ents = [pk.index[leaf + 1 + 11 * i:leaf + 12 + 11 * i] for i in range(nl)]
        qbs, prog = [e[:10] for e in ents], [int(e[10]) for e in ents]
    out = {}
    for r in range(m):
        stack = []
        for qb, adds in zip(qbs, prog):        # post-order: leaf, then (left + right)s
            stack.append(_leaf_sum(v, cols, mat, qb, r))
            for _ in range(adds):
                right = stack.pop()
                stack[-1] = F32(stack[-1] + right)
        assert len(stack) == 1
        z = stack[0]
        out[int(rows[r])] = z
    return out


def dense_for(fn, dim, seed):
    inst = instances.build(fn, dim, seed)
    if isinstance(inst, instances.BasicInstance):
        return inst.rotation.dense()
    if isinstance(inst, instances.HybridInstance):
        return inst.chunk_rotations[0]
    m = inst.members[0]
    return m.rotation.dense() if m.rotation is not None else m.hybrid.chunk_rotations[0]


@pytest.mark.parametrize("dim", [2, 5, 8, 9, 10, 13, 30, 50, 100, 128, 129, 200, 250, 300, 520])
def test_exact_order_schedule_reproduces_numpy(dim):
    disabled = frozenset(range(23, 37)) if dim < 10 else frozenset()
    pk = P.Pack(dim, 1, disabled)
    rng = np.random.default_rng(dim)
    for fn in (0, 11, 23, 27, 29, 35):
        if fn in disabled:
            continue
        rec = pk.functions[fn]
        seg = pk.segments[pk.members[rec["member0"]]["segment0"]]
        R = dense_for(fn, dim, 1).astype(F32)
        for _ in range(3):
            v = rng.uniform(-100, 100, int(seg["d"])).astype(F32)
            want = (R * v).sum(axis=1)
            got = np.zeros_like(want)
            for g in range(seg["n_groups"]):
                for r, z in exact_order_rotate(pk, pk.groups[seg["group0"] + g], v).items():
                    got[r] = z
            assert np.array_equal(got, want)


def test_pack_shapes_and_disabled():
    pk = P.Pack(10, 0)
    assert len(pk.functions) == 37
    assert (pk.functions["category"] >= 0).all()
    pk2 = P.Pack(2, 0, frozenset(range(23, 37)))
    assert (pk2.functions["category"][23:] == P.DISABLED).all()
    # block-sparse storage: sum of squared group sizes, never D^2
    pk100 = P.Pack(100, 0)
    seg = pk100.segments[pk100.members[pk100.functions[0]["member0"]]["segment0"]]
    sizes = [int(pk100.groups[seg["group0"] + g]["m"]) for g in range(seg["n_groups"])]
    assert sizes == [34, 33, 33]
    assert pk100.max_exact_len == 100


def _segment_of_group(pk, gi):
    for seg in pk.segments:
        if seg["group0"] <= gi < seg["group0"] + seg["n_groups"]:
            return seg
    raise AssertionError(gi)


def test_dmma_fragments_match_q_ordered_block():
    pk = P.Pack(100, 0)
    for gi, g in enumerate(pk.groups[:12]):
        scale = float(_segment_of_group(pk, gi)["scale"])
        m = int(g["m"])
        nt, nk, m4 = (m + 7) // 8, (m + 3) // 4, (m + 3) // 4 * 4
        mat = pk.values_f64[g["mat"]:g["mat"] + m * m4].reshape(m, m4)
        col = pk.index[g["col"]:g["col"] + m]
        col64 = pk.index[g["col64"]:g["col64"] + m]
        assert sorted(col) == sorted(col64)
        qpos = {int(c): q for q, c in enumerate(col)}           # q-order row of mat per column
        frag = pk.values_f64[g["frag"]:g["frag"] + nt * nk * 32].reshape(nt, nk, 32)
        for a in range(nt):
            for ks in range(nk):
                for lane in range(32):
                    q, r = 4 * ks + lane % 4, 8 * a + lane // 4
                    want = scale * mat[qpos[int(col64[q])], r] if (q < m and r < m) else 0.0
                    assert frag[a, ks, lane] == want
        assert g["mat"] % 4 == 0 and g["frag"] % 4 == 0


@pytest.mark.parametrize("dim", [2, 3, 10, 13, 50, 100])
def test_fp64_offsets_restate_the_transform(dim):
    """(scale B)(x - o)[src] - cz == R(scale (x - o)[src] + pre) + post for
    every rotated segment of every member (the float64 rotate's algebra),
    and exactly post at the optimum."""
    pk = P.Pack(dim, 0, disabled=frozenset(range(23, 37)) if dim < 10 else frozenset())
    rng = np.random.default_rng(7)
    x = rng.uniform(-100, 100, dim)
    for mem in pk.members:
        o = pk.values_f64[mem["shift"]:mem["shift"] + dim]
        perm = (pk.index[mem["perm"]:mem["perm"] + dim] if mem["perm"] >= 0 else None)
        for si in range(mem["segment0"], mem["segment0"] + mem["n_segments"]):
            seg = pk.segments[si]
            for gi in range(seg["group0"], seg["group0"] + seg["n_groups"]):
                g = pk.groups[gi]
                m = int(g["m"])
                m4 = (m + 3) // 4 * 4
                mat = pk.values_f64[g["mat"]:g["mat"] + m * m4].reshape(m, m4)[:, :m]
                pos = pk.index[g["col"]:g["col"] + m] + seg["src"]
                src = perm[pos] if perm is not None else pos
                v = seg["scale"] * (x[src] - o[src]) + seg["pre"]
                want = mat.T @ v + seg["post"]
                cz = pk.values_f64[g["cz"]:g["cz"] + m]
                got = (seg["scale"] * mat).T @ (x[src] - o[src]) - cz
                # the float64 column order feeds the same columns
                pos64 = pk.index[g["col64"]:g["col64"] + m] + seg["src"]
                assert sorted(pos64) == sorted(pos)
                assert np.allclose(got, want, rtol=1e-12, atol=1e-10 * max(1.0, np.abs(want).max()))
                if seg["pre"] == 0.0:
                    assert np.all(-cz == seg["post"])


def test_fp64_column_order_avoids_bank_conflicts():
    # D=100: X rows are 100 doubles apart (4 mod 16 banks): a k-step is
    # conflict-free iff its 4 columns differ mod 4; the greedy order achieves
    # it wherever the residue counts allow
    cols = list(range(0, 100, 3))[:34]
    order = P.fp64_column_order(cols, 100)
    assert sorted(order) == list(range(34))
    full = [order[i:i + 4] for i in range(0, 32, 4)]
    good = sum(len({cols[k] % 4 for k in ks}) == 4 for ks in full)
    assert good >= 6


def test_kernel_constants_follow_numpy():
    c = P.kernel_constants("weierstrass", 30, np.float32)
    k = np.arange(21, dtype=np.float32)
    assert np.array_equal(c[:21], 0.5**k)
    assert np.array_equal(c[21:42], 2.0 * np.pi * 3.0**k)
    assert c.dtype == np.float32
    e = P.kernel_constants("elliptic", 7, np.float64)
    assert e[0] == 1.0 and e[-1] == 1e6


def test_pairwise_leaves():
    assert P.pairwise_leaves(100) == [(0, 100)]
    assert P.pairwise_leaves(200) == [(0, 96), (96, 200)]
    assert P.pairwise_leaves(250) == [(0, 120), (120, 184), (184, 250)]
    assert P.pairwise_leaves(256) == [(0, 128), (128, 256)]
    for n in range(129, 969):                  # the device stack holds the whole tree
        prog = P.pairwise_program(n)
        assert len(prog) == len(P.pairwise_leaves(n)) and sum(prog) == len(prog) - 1
        assert P.program_depth(prog) <= P.EXACT_ORDER_STACK
    assert P.pairwise_program(250) == [0, 0, 2]              # l0 + (l1 + l2)
    assert P.pairwise_program(512) == [0, 1, 0, 2]           # (l0 + l1) + (l2 + l3)


def test_slot_of():
    assert [P.slot_of(i, 5) for i in range(5)] == [8] * 5
    assert [P.slot_of(i, 10) for i in range(10)] == [0, 1, 2, 3, 4, 5, 6, 7, 8, 8]
    assert P.slot_of(17, 100) == 1 and P.slot_of(96, 100) == 8
