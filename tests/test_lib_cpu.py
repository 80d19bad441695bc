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
    return sorted(set(re.findall(r"\b(wmh_[a-z0-9_]+)\s*\(", src)))


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


def test_new_entry_points_validate_without_gpu(lib):
    """f1 / f3 / hasher / timing entry points reject bad arguments before any
    CUDA call (so these run on a CPU-only host)."""
    from paper_1602_08393_b200 import _lib
    E = _lib.WMH_EINVAL
    out = ctypes.c_void_p()
    # LSH: K*L > k, bad width, NULL signatures, NULL index
    assert lib.wmh_lsh_build(ctypes.c_void_p(1), 2, 10, 5, 4, 3, ctypes.byref(out), None) == E
    assert b"K*L" in lib.wmh_last_error()
    assert lib.wmh_lsh_build(ctypes.c_void_p(1), 4, 10, 5, 2, 2, ctypes.byref(out), None) == E
    assert lib.wmh_lsh_build(None, 2, 10, 5, 2, 2, ctypes.byref(out), None) == E
    cnt = ctypes.c_void_p(1)
    assert lib.wmh_lsh_query(None, None, 1, 1, None, cnt, None) == E
    # hasher: NULL layout, k out of range
    assert lib.wmh_hasher_create(None, 1, 8, 10, 0, ctypes.byref(out), None) == E
    assert lib.wmh_hasher_create(ctypes.c_void_p(1), 1, 0, 10, 0, ctypes.byref(out), None) == E
    assert lib.wmh_hasher_run(None, None, 2, None, None, None) == E
    # quantiser and scale objective: bad scale, n < 0, empty grid
    assert lib.wmh_quantize(None, 4, ctypes.c_float(0.0), None, None) == E
    assert lib.wmh_quantize(None, -1, ctypes.c_float(2.0), None, None) == E
    rows = _lib.WmhRows(0, 4, 8, None, None, None, None, 0, 0)
    sc = (ctypes.c_float * 1)(1.0)
    o3 = (ctypes.c_uint64 * 3)()
    assert lib.wmh_scale_objective(ctypes.byref(rows), sc, 0, o3, None) == E
    # a weight width other than 1 / 2
    bad = _lib.WmhRows(0, 4, 8, None, None, None, None, 0, 3)
    assert lib.wmh_colmax(ctypes.byref(bad), None, None) == E
    assert b"weight_bytes" in lib.wmh_last_error()
    # no timed hash call on this thread yet
    ms = ctypes.c_float()
    assert lib.wmh_last_kernel_ms(ctypes.byref(ms)) == E


def test_tile_option_validated_before_any_call():
    """hash(tile=...) accepts only auto / bytes / bitplanes (WMH_OPT_TILE_* flags)."""
    import torch
    import paper_1602_08393_b200 as wmh
    from paper_1602_08393_b200 import _lib
    assert (_lib.WMH_OPT_TILE_BYTES, _lib.WMH_OPT_TILE_BITPLANES) == (2, 4)
    rows = wmh.Rows.from_dense(torch.zeros((2, 8), dtype=torch.uint8))
    with pytest.raises(ValueError, match="tile"):
        wmh.hash(None, rows, 1, 4, 10, tile="diagonal")


def test_sketches_refuse_mismatched_metadata():
    """collide_sketches checks (seed, k, cap, layout digest) before any call."""
    import torch
    import paper_1602_08393_b200 as wmh
    s = torch.zeros((2, 4), dtype=torch.uint16)
    a = wmh.Sketch(s, 1, 4, 100, 7)
    i = torch.zeros(1, dtype=torch.int64)
    for b, what in [(wmh.Sketch(s, 2, 4, 100, 7), "seed"), (wmh.Sketch(s, 1, 4, 99, 7), "cap"),
                    (wmh.Sketch(s, 1, 4, 100, 8), "layout digest")]:
        with pytest.raises(ValueError, match=what):
            wmh.collide_sketches(a, b, i, i)
