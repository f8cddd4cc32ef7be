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


def test_gemm_epilogue_struct_layout_matches_header(tmp_path):
    """ops.GemmEpilogue (ctypes) has the size and field offsets of
    emm_gemm_epilogue as gcc lays it out from include/emm.h."""
    import subprocess

    from paper_2507_10069_b200.ops import GemmEpilogue
    fields = [f[0] for f in GemmEpilogue._fields_]
    src = tmp_path / "layout.c"
    body = "".join(f'  printf("{f} %zu\\n", offsetof(emm_gemm_epilogue, {f}));\n' for f in fields)
    src.write_text('#include <stddef.h>\n#include <stdio.h>\n#include "emm.h"\nint main(void) {\n'
                   '  printf("sizeof %zu\\n", sizeof(emm_gemm_epilogue));\n' + body + "  return 0;\n}\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.dirname(HDR), str(src), "-o", str(exe)], check=True)
    got = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True,
                                                        check=True).stdout.splitlines())
    assert int(got["sizeof"]) == ctypes.sizeof(GemmEpilogue)
    for f in fields:
        assert int(got[f]) == getattr(GemmEpilogue, f).offset, f
