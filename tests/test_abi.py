"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/onmt.h
declares, and rejects bad arguments without touching a GPU."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "onmt.h")).read()
    return sorted(set(re.findall(r"ONMT_API\s+[\w\s\*]+?\b(onmt_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ["onmt_load_weights", "onmt_encode", "onmt_translate", "onmt_free", "onmt_last_error"]:
        assert s in syms


def test_library_exports_every_declared_symbol():
    import paper_1805_11462_b200 as ob
    if not os.path.exists(ob.LIB_PATH):
        pytest.skip("library not built (run __graft_entry__.build())")
    L = ob.lib()
    for s in declared_symbols():
        assert hasattr(L, s), s
    assert sorted(ob.EXPORTS) == declared_symbols()


def test_null_arguments_rejected_without_gpu():
    import paper_1805_11462_b200 as ob
    if not os.path.exists(ob.LIB_PATH):
        pytest.skip("library not built")
    L = ob.lib()
    h = ctypes.c_void_p()
    assert L.onmt_load_weights(None, 0, 0, ctypes.byref(h)) == -1
    assert L.onmt_load_weights(b"/x", 0, 7, ctypes.byref(h)) == -1
    assert L.onmt_translate(None, None, None, 0, 1, 1, 1, 0.0, None, None, None, None, None) == -1
    assert L.onmt_last_error() != b""
    L.onmt_free(None)


def test_sm100a_code_in_library():
    import shutil
    import subprocess
    import paper_1805_11462_b200 as ob
    if not os.path.exists(ob.LIB_PATH) or not shutil.which("cuobjdump"):
        pytest.skip("library or cuobjdump missing")
    out = subprocess.run(["cuobjdump", "-sass", ob.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "UTCHMMA" in out and "UTMALDG" in out and "LDTM" in out   # tcgen05.mma, TMA, tcgen05.ld
