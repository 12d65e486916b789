"""The C-ABI library loads without a GPU and exports every entry point the
header declares, with the struct layout the Python pack uses."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from paper_1407_7737_b200 import _lib, pack

HEADER = Path(__file__).resolve().parent.parent / "include" / "robench_b200.h"


def declared():
    text = HEADER.read_text()
    decl = r"^(?:rb_status|int32_t|int64_t|void|const char\*)\s+(rb_[a-z0-9_]+)\s*\("
    return sorted(set(re.findall(decl, text, flags=re.M)))


def test_header_declares_the_paper_api():
    names = declared()
    for want in ("rb_initialize", "rb_func_evaluate", "rb_func_evaluatef",
                 "rb_h_func_evaluate", "rb_h_func_evaluatef", "rb_dispose"):
        assert want in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    for name in declared():
        assert hasattr(lib, name), name
    assert set(_lib.EXPORTS) <= set(declared())


def test_struct_layout_matches_python():
    lib = _lib.load()
    sizes = (ctypes.c_int64 * 5)()
    lib.rb_struct_sizes(sizes)
    assert tuple(sizes) == (pack.GROUP_DT.itemsize, pack.SEGMENT_DT.itemsize,
                            pack.MEMBER_DT.itemsize, pack.FUNCTION_DT.itemsize,
                            ctypes.sizeof(_lib.RbPack))
    assert lib.rb_abi_version() == 1


def test_null_and_disposed_handles_map_to_reference_errors():
    lib = _lib.load()
    x = np.zeros(10)
    f = np.zeros(1)
    st = lib.rb_h_func_evaluate(None, 0, x.ctypes.data, 1, f.ctypes.data)
    assert _lib._STATUS[st].__name__ == "UseAfterDispose"
    handle = ctypes.c_void_p()
    assert lib.rb_dispose(ctypes.byref(handle)) == 0      # idempotent on NULL
    assert lib.rb_initialize(None, 1, 0, ctypes.byref(handle)) == 7


def _corrupt(p, table, idx, field, value):
    arr = getattr(p, table)
    arr[idx][field] = value


@pytest.mark.parametrize("table,field,value", [
    ("members", "segment0", 10 ** 6),
    ("members", "shift", -5),
    ("members", "perm", 10 ** 8),
    ("segments", "ctab", 10 ** 9),
    ("segments", "src", 7),
    ("groups", "col", 10 ** 9),
    ("groups", "mat", -100),
    ("groups", "frag", 10 ** 9),
    ("groups", "cz", 10 ** 9),
    ("groups", "leaf", 10 ** 9),
    ("groups", "m", 0),
])
def test_malformed_pack_offsets_are_rejected_before_any_read(table, field, value):
    # rb_initialize bounds-checks every offset with its extent (a public C ABI:
    # non-Python hosts build packs too); the check precedes any CUDA call, so
    # it runs without a GPU
    p = pack.Pack(10, 0)
    idx = {"members": 3, "segments": 5, "groups": 4}[table]
    if table == "members" and field == "perm":
        idx = int(p.functions[23]["member0"])          # a hybrid: has a permutation
    _corrupt(p, table, idx, field, value)
    handle = ctypes.c_void_p()
    st = _lib.load().rb_initialize(ctypes.byref(_lib.make_pack(p)), 8, 0, ctypes.byref(handle))
    assert st == 7, (table, field, st)
    assert b"out of range" in _lib.load().rb_last_error()


def test_malformed_index_entries_are_rejected():
    p = pack.Pack(10, 0)
    g = p.groups[0]
    p.index[int(g["col"])] = 10 ** 6                    # a column outside the segment
    handle = ctypes.c_void_p()
    assert _lib.load().rb_initialize(ctypes.byref(_lib.make_pack(p)), 8, 0, ctypes.byref(handle)) == 7


@pytest.mark.parametrize("dim", [10, 13, 30, 100, 300])
def test_well_formed_packs_pass_validation(dim):
    # without a GPU the call gets past validation and fails at the device
    # query (RB_E_CUDA); with one it succeeds
    p = pack.Pack(dim, 0)
    handle = ctypes.c_void_p()
    st = _lib.load().rb_initialize(ctypes.byref(_lib.make_pack(p)), 8, 0, ctypes.byref(handle))
    assert st in (0, 9), _lib.load().rb_last_error()
    if st == 0:
        _lib.load().rb_dispose(ctypes.byref(handle))
