"""CPU oracle for rejection-sampling weighted minwise hashing (arXiv 1602.08393).

TEST INFRASTRUCTURE -- not the product.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It shares no code with ``paper_1602_08393_b200`` (the CUDA path) and
neither side imports the other.

This module is argument marshalling (numpy <-> ctypes) around ``wmh_oracle.c``,
which holds every step of the arithmetic (see that file's header for the paper
citations).  The shared library is compiled with plain ``gcc`` on first use.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from fractions import Fraction

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "wmh_oracle.c")
_SO = os.path.join(_HERE, "libwmh_oracle.so")
_lock = threading.Lock()
_lib = None

OK, EINVAL, EEMPTY, EOVERFLOW, EBOUND, ENOMEM = 0, -1, -2, -3, -4, -5


# WMH_ORACLE_SANITIZE=1: load an AddressSanitizer + UndefinedBehaviorSanitizer
# build instead (run python with LD_PRELOAD=$(gcc -print-file-name=libasan.so)
# and ASAN_OPTIONS=detect_leaks=0; scripts/sanitize_oracle.sh)
_SAN = os.environ.get("WMH_ORACLE_SANITIZE") == "1"
if _SAN:
    _SO = os.path.join(_HERE, "libwmh_oracle_san.so")


def build(force: bool = False) -> str:
    """Compile wmh_oracle.c into libwmh_oracle.so (plain gcc -O2, no fast-math)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        flags = ["-O1", "-g", "-fsanitize=address,undefined", "-fno-sanitize-recover=undefined",
                 "-fno-omit-frame-pointer"] if _SAN else ["-O2"]
        subprocess.check_call(["gcc", *flags, "-std=gnu11", "-fPIC", "-shared", "-pthread",
                               "-o", tmp, _SRC])
        os.replace(tmp, _SO)
    return _SO


def lib() -> ctypes.CDLL:
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_SO)
            u8p = ctypes.POINTER(ctypes.c_uint8)
            u16p = ctypes.POINTER(ctypes.c_uint16)
            u32p = ctypes.POINTER(ctypes.c_uint32)
            i32p = ctypes.POINTER(ctypes.c_int32)
            i64p = ctypes.POINTER(ctypes.c_int64)
            u64p = ctypes.POINTER(ctypes.c_uint64)
            i64, u64, u32, c_int = ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int
            sig = {
                "oracle_splitmix64": (u64, [u64]),
                "oracle_draw": (u32, [u64, u32, u32, u32]),
                "oracle_colmax_dense": (None, [u8p, i64, i64, u32p]),
                "oracle_colmax_csr": (None, [i64p, i32p, u8p, i64, i64, u32p]),
                "oracle_total_M": (c_int, [u32p, i64, u64p]),
                "oracle_build_layout": (c_int, [u32p, i64, u32p, u32p]),
                "oracle_check_bounds_dense": (c_int, [u8p, i64, i64, u32p, i64p, i64p]),
                "oracle_check_bounds_csr": (c_int, [i64p, i32p, u8p, i64, i64, i64, u32p, i64p,
                                                    ctypes.POINTER(c_int)]),
                "oracle_is_green_o1": (c_int, [u32p, u32p, u8p, u32]),
                "oracle_is_green_binsearch": (c_int, [u32p, i32p, u8p, i64, u32]),
                "oracle_is_green_direct": (c_int, [u32p, u8p, i64, u32]),
                "oracle_hash_from_draws": (u32, [u32p, u32p, u8p, u32p, u32]),
                "oracle_hash_one": (u32, [u32p, u32p, u32, u8p, u64, u32, u32]),
                "oracle_hash_dense": (c_int, [u8p, i64, i64, u32p, u32p, u32, u64, u32, u32, u32p, c_int]),
                "oracle_hash_csr": (c_int, [i64p, i32p, u8p, i64, i64, u32p, u32p, u32, u64, u32, u32,
                                            u32p, c_int]),
                "oracle_collide": (None, [u32p, u32, i64p, i64, u32p]),
                "oracle_jaccard_dense": (None, [u8p, u8p, i64, u64p, u64p]),
                "oracle_jaccard_csr": (None, [i64p, i32p, u8p, i64, i64, u64p, u64p]),
                "oracle_colmax_dense16": (None, [u16p, i64, i64, u32p]),
                "oracle_colmax_csr16": (None, [i64p, i32p, u16p, i64, i64, u32p]),
                "oracle_hash_one16": (u32, [u32p, u32p, u32, u16p, u64, u32, u32]),
                "oracle_hash_dense16": (c_int, [u16p, i64, i64, u32p, u32p, u32, u64, u32, u32, u32p, c_int]),
                "oracle_hash_csr16": (c_int, [i64p, i32p, u16p, i64, i64, u32p, u32p, u32, u64, u32, u32,
                                              u32p, c_int]),
            }
            for name, (res, args) in sig.items():
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            _lib = L
    return _lib


def _p(a: np.ndarray, ct):
    assert a.flags["C_CONTIGUOUS"], "oracle inputs must be C-contiguous"
    return a.ctypes.data_as(ctypes.POINTER(ct))


def _u8(a):
    a = np.asarray(a)
    if a.dtype == np.uint16:
        raise TypeError("uint16 weights go through the *16 oracle functions")
    return np.ascontiguousarray(a, dtype=np.uint8)


def _is16(a) -> bool:
    return np.asarray(a).dtype == np.uint16


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


# --------------------------------------------------------------------------- RNG
def splitmix64(v: int) -> int:
    return int(lib().oracle_splitmix64(ctypes.c_uint64(v & (2**64 - 1))))


def draw(seed: int, j: int, t: int, M: int) -> int:
    """r_t of hash j (readings R6-R8)."""
    return int(lib().oracle_draw(seed & (2**64 - 1), j, t, M))


# ----------------------------------------------------------------- preprocessing
def colmax_dense(x: np.ndarray) -> np.ndarray:
    if _is16(x):
        x = np.ascontiguousarray(x)
        m = np.zeros(x.shape[1], np.uint32)
        lib().oracle_colmax_dense16(_p(x, ctypes.c_uint16), x.shape[0], x.shape[1], _p(m, ctypes.c_uint32))
        return m
    x = _u8(x)
    n, d = x.shape
    m = np.zeros(d, np.uint32)
    lib().oracle_colmax_dense(_p(x, ctypes.c_uint8), n, d, _p(m, ctypes.c_uint32))
    return m


def colmax_csr(row_ptr, col, val, dim) -> np.ndarray:
    row_ptr = np.ascontiguousarray(row_ptr, np.int64)
    col = np.ascontiguousarray(col, np.int32)
    m = np.zeros(dim, np.uint32)
    if _is16(val):
        val = np.ascontiguousarray(val)
        lib().oracle_colmax_csr16(_p(row_ptr, ctypes.c_int64), _p(col, ctypes.c_int32), _p(val, ctypes.c_uint16),
                                  len(row_ptr) - 1, dim, _p(m, ctypes.c_uint32))
        return m
    val = _u8(val)
    lib().oracle_colmax_csr(_p(row_ptr, ctypes.c_int64), _p(col, ctypes.c_int32), _p(val, ctypes.c_uint8),
                            len(row_ptr) - 1, dim, _p(m, ctypes.c_uint32))
    return m


class Layout:
    """CompToM (D+1 entries, exclusive prefix) and IntToComp (M entries) from Alg. 4."""

    def __init__(self, m):
        m = _u32(m)
        self.m = m
        self.dim = len(m)
        M = ctypes.c_uint64(0)
        rc = lib().oracle_total_M(_p(m, ctypes.c_uint32), self.dim, ctypes.byref(M))
        if rc != OK:
            raise ValueError({EEMPTY: "M = 0 (all bounds zero)", EOVERFLOW: "M >= 2^32"}.get(rc, rc))
        self.M = int(M.value)
        self.comp_to_m = np.zeros(self.dim + 1, np.uint32)
        self.int_to_comp = np.zeros(self.M, np.uint32)
        rc = lib().oracle_build_layout(_p(m, ctypes.c_uint32), self.dim, _p(self.comp_to_m, ctypes.c_uint32),
                                       _p(self.int_to_comp, ctypes.c_uint32))
        assert rc == OK

    def _t(self):
        return _p(self.int_to_comp, ctypes.c_uint32), _p(self.comp_to_m, ctypes.c_uint32)

    def check_bounds_dense(self, x):
        x = _u8(x)
        br, bc = ctypes.c_int64(-1), ctypes.c_int64(-1)
        rc = lib().oracle_check_bounds_dense(_p(x, ctypes.c_uint8), x.shape[0], x.shape[1],
                                             _p(self.m, ctypes.c_uint32), ctypes.byref(br), ctypes.byref(bc))
        return None if rc == OK else (br.value, bc.value)

    def check_bounds_csr(self, row_ptr, col, val):
        """None, or (index of the first offending nonzero -- of the row for a
        malformed row_ptr --, reason 1 column range, 2 order, 3 bound, 4 row_ptr)."""
        rp = np.ascontiguousarray(row_ptr, np.int64)
        c = np.ascontiguousarray(col, np.int32)
        v = _u8(val)
        bi, why = ctypes.c_int64(-1), ctypes.c_int(0)
        rc = lib().oracle_check_bounds_csr(_p(rp, ctypes.c_int64), _p(c, ctypes.c_int32), _p(v, ctypes.c_uint8),
                                           len(rp) - 1, self.dim, len(c), _p(self.m, ctypes.c_uint32),
                                           ctypes.byref(bi), ctypes.byref(why))
        return None if rc == OK else (bi.value, why.value)

    # ISGREEN variants
    def is_green_o1(self, x_dense, r: int) -> bool:
        x = _u8(x_dense)
        i2c, c2m = self._t()
        return bool(lib().oracle_is_green_o1(i2c, c2m, _p(x, ctypes.c_uint8), r))

    def is_green_binsearch(self, cols, vals, r: int) -> bool:
        cols = np.ascontiguousarray(cols, np.int32)
        vals = _u8(vals)
        return bool(lib().oracle_is_green_binsearch(_p(self.comp_to_m, ctypes.c_uint32), _p(cols, ctypes.c_int32),
                                                    _p(vals, ctypes.c_uint8), len(cols), r))

    def is_green_direct(self, x_dense, r: int) -> bool:
        x = _u8(x_dense)
        return bool(lib().oracle_is_green_direct(_p(self.comp_to_m, ctypes.c_uint32), _p(x, ctypes.c_uint8),
                                                 self.dim, r))

    # hashing
    def hash_from_draws(self, x_dense, draws, cap: int) -> int:
        x = _u8(x_dense)
        d = _u32(draws)
        assert len(d) >= cap
        i2c, c2m = self._t()
        return int(lib().oracle_hash_from_draws(i2c, c2m, _p(x, ctypes.c_uint8), _p(d, ctypes.c_uint32), cap))

    def hash_one(self, x_dense, seed: int, j: int, cap: int) -> int:
        x = _u8(x_dense)
        i2c, c2m = self._t()
        return int(lib().oracle_hash_one(i2c, c2m, self.M, _p(x, ctypes.c_uint8), seed & (2**64 - 1), j, cap))

    def hash_dense(self, x, seed: int, k: int, cap: int, threads: int | None = None) -> np.ndarray:
        """uint8 weights, or uint16 (f1: fixed-point real data) through the *16 functions."""
        if _is16(x):
            x = np.ascontiguousarray(x)
            if x.ndim == 1:
                x = x[None, :]
            assert x.shape[1] == self.dim
            sig = np.zeros((x.shape[0], k), np.uint32)
            i2c, c2m = self._t()
            rc = lib().oracle_hash_dense16(_p(x, ctypes.c_uint16), x.shape[0], self.dim, i2c, c2m, self.M,
                                           seed & (2**64 - 1), k, cap, _p(sig, ctypes.c_uint32),
                                           threads or os.cpu_count() or 1)
            if rc != OK:
                raise ValueError(f"oracle_hash_dense16 failed: {rc}")
            return sig
        x = _u8(x)
        if x.ndim == 1:
            x = x[None, :]
        assert x.shape[1] == self.dim
        sig = np.zeros((x.shape[0], k), np.uint32)
        i2c, c2m = self._t()
        rc = lib().oracle_hash_dense(_p(x, ctypes.c_uint8), x.shape[0], self.dim, i2c, c2m, self.M,
                                     seed & (2**64 - 1), k, cap, _p(sig, ctypes.c_uint32),
                                     threads or os.cpu_count() or 1)
        if rc != OK:
            raise ValueError(f"oracle_hash_dense failed: {rc}")
        return sig

    def hash_csr(self, row_ptr, col, val, seed: int, k: int, cap: int, threads: int | None = None) -> np.ndarray:
        row_ptr = np.ascontiguousarray(row_ptr, np.int64)
        col = np.ascontiguousarray(col, np.int32)
        n = len(row_ptr) - 1
        sig = np.zeros((n, k), np.uint32)
        i2c, c2m = self._t()
        if _is16(val):
            val = np.ascontiguousarray(val)
            rc = lib().oracle_hash_csr16(_p(row_ptr, ctypes.c_int64), _p(col, ctypes.c_int32),
                                         _p(val, ctypes.c_uint16), n, self.dim, i2c, c2m, self.M,
                                         seed & (2**64 - 1), k, cap, _p(sig, ctypes.c_uint32),
                                         threads or os.cpu_count() or 1)
            if rc != OK:
                raise ValueError(f"oracle_hash_csr16 failed: {rc}")
            return sig
        val = _u8(val)
        rc = lib().oracle_hash_csr(_p(row_ptr, ctypes.c_int64), _p(col, ctypes.c_int32), _p(val, ctypes.c_uint8),
                                   n, self.dim, i2c, c2m, self.M, seed & (2**64 - 1), k, cap,
                                   _p(sig, ctypes.c_uint32), threads or os.cpu_count() or 1)
        if rc != OK:
            raise ValueError(f"oracle_hash_csr failed: {rc}")
        return sig


# ------------------------------------------------------------------- estimation
def collide(sig: np.ndarray, pairs: np.ndarray) -> np.ndarray:
    sig = _u32(sig)
    pairs = np.ascontiguousarray(pairs, np.int64).reshape(-1, 2)
    out = np.zeros(len(pairs), np.uint32)
    lib().oracle_collide(_p(sig, ctypes.c_uint32), sig.shape[1], _p(pairs, ctypes.c_int64), len(pairs),
                         _p(out, ctypes.c_uint32))
    return out


def jaccard_dense(x, y) -> Fraction | None:
    """Eq. 1 as an exact fraction (None for 0/0)."""
    x, y = _u8(x), _u8(y)
    num, den = ctypes.c_uint64(), ctypes.c_uint64()
    lib().oracle_jaccard_dense(_p(x, ctypes.c_uint8), _p(y, ctypes.c_uint8), len(x), ctypes.byref(num),
                               ctypes.byref(den))
    return None if den.value == 0 else Fraction(num.value, den.value)


def jaccard_csr(row_ptr, col, val, a: int, b: int) -> Fraction | None:
    row_ptr = np.ascontiguousarray(row_ptr, np.int64)
    col = np.ascontiguousarray(col, np.int32)
    val = _u8(val)
    num, den = ctypes.c_uint64(), ctypes.c_uint64()
    lib().oracle_jaccard_csr(_p(row_ptr, ctypes.c_int64), _p(col, ctypes.c_int32), _p(val, ctypes.c_uint8),
                             a, b, ctypes.byref(num), ctypes.byref(den))
    return None if den.value == 0 else Fraction(num.value, den.value)


# ----------------------------------------------- f1: real-valued weights (Sec. 4)
def quantize(x, scale: float) -> np.ndarray:
    """w = min(65535, floor(x * scale)) with the product rounded to nearest in
    float32 (IEEE, numpy) -- the fixed-point reading of P:137's ceil bound and
    Sec. 4's scaling (R18).  x >= 0."""
    x = np.asarray(x, np.float32)
    if np.any(~(x >= 0)):
        raise ValueError("weights must be >= 0")
    q = np.floor(x * np.float32(scale))
    return np.minimum(q, 65535).astype(np.uint16)


def scale_objective(x_rows, scales):
    """Sec. 4 for fixed point: per scale s, (sum_n sum_c floor(x s),
    n_rows * sum_c max_n floor(x s), #weights with floor(x s) >= 65536) -- the
    numerator and denominator of the mean effective sparsity (Eq. 17) of the
    quantised rows and the count the uint16 quantiser saturates.  x_rows: dense
    float32 (n_rows, D)."""
    x = np.asarray(x_rows, np.float32)
    out = []
    for s in scales:
        q = quantize(x, s).astype(np.int64)
        clipped = int((np.floor(x * np.float32(s)) >= 65536).sum())
        out.append((int(q.sum()), int(x.shape[0]) * int(q.max(axis=0).sum()), clipped))
    return out


def choose_scale(x_rows, scales) -> float:
    """argmax of the mean effective sparsity over the scales that saturate no
    weight; ties go to the smaller scale (SPEC optimize_alpha)."""
    best = None
    for s, (num, den, clipped) in sorted(zip(scales, scale_objective(x_rows, scales)), key=lambda t: t[0]):
        if den == 0 or clipped:
            continue
        if best is None or Fraction(num, den) > best[1]:
            best = (s, Fraction(num, den))
    return None if best is None else float(best[0])


# ------------------------------------------------ f3: (K, L) banding LSH
def lsh_candidates(sig, K: int, L: int, qsig):
    """For every query row, the sorted rows of `sig` equal to it in at least one
    band b (hashes [bK, (b+1)K)).  Plain dictionaries of band tuples."""
    sig = np.asarray(sig)
    qsig = np.asarray(qsig)
    index = [dict() for _ in range(L)]
    for n in range(sig.shape[0]):
        for b in range(L):
            index[b].setdefault(sig[n, b * K:(b + 1) * K].tobytes(), []).append(n)
    out = []
    for q in qsig:
        s = set()
        for b in range(L):
            s.update(index[b].get(q[b * K:(b + 1) * K].tobytes(), ()))
        out.append(np.array(sorted(s), np.int64))
    return out
