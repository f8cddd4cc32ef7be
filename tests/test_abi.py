"""The C ABI library loads without a GPU and exports every entry point that
include/emm.h declares (no compute calls)."""
import ctypes
import os
import re

from paper_2507_10069_b200 import _lib

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                   "emm.h")


def declared():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(emm_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_entry_points():
    names = declared()
    assert len(names) > 40
    assert "emm_cache_match_prefix" in names and "emm_gemm_bf16" in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_version_and_error_plumbing():
    assert _lib.lib.emm_version() == 1
    h = ctypes.c_void_p()
    assert _lib.lib.emm_tree_create(10, ctypes.byref(h)) == 0
    assert _lib.lib.emm_tree_release(h, 123456789) == 2  # EMM_E_RELEASE_WITHOUT_MATCH
    assert b"released or unknown" in _lib.lib.emm_last_error()
    assert _lib.lib.emm_tree_destroy(h) == 0
