"""The C ABI library (no compute without a GPU): it loads, exports every
function include/hprlp_b200.h declares, the Python binding covers them, and
the product refuses to run without CUDA (no CPU fallback)."""

import ctypes
import os
import re

import pytest

from conftest import ROOT, has_gpu

HEADER = os.path.join(ROOT, "include", "hprlp_b200.h")


def declared_functions():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*)\s*(hpr_\w+)\s*\(", txt, re.M)))


def test_library_builds_and_exports_header_symbols():
    from paper_2408_12179_b200 import _native as N
    from paper_2408_12179_b200.build import build
    build()
    lib = ctypes.CDLL(N.LIB_PATH)
    names = declared_functions()
    assert len(names) >= 18
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(N.EXPORTED_SYMBOLS)
    assert N.load_library().hpr_abi_version() == 1


def test_error_path_without_device():
    """Argument validation returns codes, never aborts."""
    from paper_2408_12179_b200 import _native as N
    lib = N.load_library()
    rc = lib.hpr_workspace_bytes(None, None)
    assert rc == -1
    assert b"null" in lib.hpr_last_error()
    bad = N.HprDims(0, 0, 0, 0)
    sz = ctypes.c_size_t(0)
    assert lib.hpr_workspace_bytes(ctypes.byref(bad), ctypes.byref(sz)) == -1
    assert lib.hpr_ctx_create(None, None, 0, None) == -1
    assert lib.hpr_launch_count(None, None) == -1


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU behaviour")
def test_solve_fails_loudly_without_cuda():
    import paper_2408_12179_b200 as P
    from paper_2408_12179_b200._native import NativeUnavailableError
    p = P.LpProblem.from_dense([[1.0]], [1.0], None, None, [1.0])
    with pytest.raises(NativeUnavailableError):
        P.solve(p)
    with pytest.raises(NativeUnavailableError):
        P.solve_batch([p, p])


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2408_12179_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
