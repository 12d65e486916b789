"""The C-ABI library loads without a GPU and exports every entry point the
header declares, with the struct layout the Python pack uses."""

import ctypes
import re
from pathlib import Path

import numpy as np

from paper_1407_7737_b200 import _lib, pack

HEADER = Path(__file__).resolve().parent.parent / "include" / "robench_b200.h"


def declared():
    text = HEADER.read_text()
    decl = r"^(?:rb_status|int32_t|int64_t|void|const char\*)\s+(rb_[a-z_]+)\s*\("
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
