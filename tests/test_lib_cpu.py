"""CPU-side checks of the C ABI: the library loads, exports every symbol that
include/wmh.h declares, and rejects invalid arguments before touching a GPU."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1602_08393_b200 import build, _lib
    build.build()
    return _lib.load()


def _header_functions():
    src = open(os.path.join(ROOT, "include", "wmh.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(wmh_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    from paper_1602_08393_b200 import _lib
    names = _header_functions()
    assert set(names) == set(_lib.EXPORTS)
    for n in names:
        assert hasattr(lib, n), n


def test_so_is_sm100a_only():
    """The fatbin carries sm_100a SASS (no PTX JIT fallback for other arches)."""
    import subprocess
    from paper_1602_08393_b200 import build
    out = subprocess.run(["cuobjdump", "--list-elf", build.SO], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_version_and_last_error(lib):
    assert b"sm_100a" in lib.wmh_version()
    assert isinstance(lib.wmh_last_error(), bytes)


def test_invalid_arguments_rejected_without_gpu(lib):
    from paper_1602_08393_b200 import _lib
    rows = _lib.WmhRows(0, 4, 8, None, None, None, None, 0)
    # NULL layout
    st = lib.wmh_hash(None, ctypes.byref(rows), 1, 4, 10, 1, None, None, None)
    assert st == _lib.WMH_EINVAL and b"layout" in lib.wmh_last_error()
    # NULL out pointer for prepare
    st = lib.wmh_prepare(None, 8, None, None, None)
    assert st == _lib.WMH_EINVAL
    # bad sig width / cap in collide
    st = lib.wmh_collide(None, 3, 4, 1, None, 1, None, None, 0, None)
    assert st == _lib.WMH_EINVAL and b"sig_bytes" in lib.wmh_last_error()
    st = lib.wmh_collide(None, 2, 0, 1, None, 1, None, None, 0, None)
    assert st == _lib.WMH_EINVAL
    # colmax with NULL rows
    assert lib.wmh_colmax(None, None, None) == _lib.WMH_EINVAL
    # unknown rows kind
    bad = _lib.WmhRows(7, 4, 8, None, None, None, None, 0)
    assert lib.wmh_colmax(ctypes.byref(bad), None, None) == _lib.WMH_EINVAL


def test_binding_has_no_cpu_fallback():
    """The product path imports no oracle and refuses CPU tensors."""
    import torch
    import paper_1602_08393_b200 as wmh
    src = open(wmh.__file__).read() + open(os.path.join(os.path.dirname(wmh.__file__), "_lib.py")).read()
    assert "oracle" not in src.replace("oracle/", "")
    rows = wmh.Rows.from_dense(torch.zeros((2, 8), dtype=torch.uint8))
    with pytest.raises(ValueError):
        wmh.colmax(rows)
