"""Seeded synthetic input generators shared by the oracle side and the CUDA side.

Holds NONE of the method's arithmetic (no draws, no layout, no hashing, no
maxima): it only produces rows shaped like the paper's workloads (DESIGN.md §4,
the input recipe) for the five configurations of BASELINE.json.  The paper's
datasets (Table 1, P:329-347 -- Web-Images RGB histograms, Caltech101 and Oxford
HOG features) are not available here; these generators stand in for them.

Two kinds of generator:
  * counter-based (c1, c5): every entry is a pure function of
    (data_seed, row, col) through MurmurHash3's 64-bit finaliser (NOT the
    method's SplitMix64), so any row can be regenerated alone, on the host or
    by the device generator in ``datagen/gen_kernels.cu`` (bit-identical:
    integer-only, no libm);
  * numpy-Generator based (c2, c3, c4): drawn per 4096-row chunk from
    ``np.random.Generator(PCG64([data_seed, chunk]))`` so the dataset does not
    depend on how rows are later sharded over GPUs.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

MASK64 = (1 << 64) - 1
CHUNK = 4096


# ---------------------------------------------------------------- counter mixer
def fmix64_int(h: int) -> int:
    """MurmurHash3 fmix64 on a python int (reference for the vectorised form)."""
    h &= MASK64
    h ^= h >> 33
    h = (h * 0xFF51AFD7ED558CCD) & MASK64
    h ^= h >> 33
    h = (h * 0xC4CEB9FE1A85EC53) & MASK64
    h ^= h >> 33
    return h


def fmix64(h: np.ndarray) -> np.ndarray:
    h = h.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        h ^= h >> np.uint64(33)
        h *= np.uint64(0xFF51AFD7ED558CCD)
        h ^= h >> np.uint64(33)
        h *= np.uint64(0xC4CEB9FE1A85EC53)
        h ^= h >> np.uint64(33)
    return h


def entry_bits(data_seed: int, rows: np.ndarray, dim: int) -> np.ndarray:
    """64 random bits per (row, col): fmix64(fmix64(data_seed) ^ (row*dim + col))."""
    base = np.uint64(fmix64_int(data_seed))
    rows = np.asarray(rows, dtype=np.uint64)
    idx = rows[:, None] * np.uint64(dim) + np.arange(dim, dtype=np.uint64)[None, :]
    return fmix64(idx ^ base)


# c1: 0 w.p. 0.3, else uniform on {1..15}
C1_ZERO_THRESH = int(0.3 * 2**32)                  # low 32 bits below this -> 0


def gen_counter_c1_rows(data_seed: int, rows, dim: int) -> np.ndarray:
    b = entry_bits(data_seed, rows, dim)
    lo = (b & np.uint64(0xFFFFFFFF))
    hi = (b >> np.uint64(32))
    v = (np.uint64(1) + hi % np.uint64(15)).astype(np.uint8)
    v[lo < np.uint64(C1_ZERO_THRESH)] = 0
    return v


# c5: 0 w.p. 1/2 (top bit), else min(255, Geometric(p=0.3) on {1,2,..}):
# X = #{v >= 0 : u < T_v} with u the low 63 bits and T_v = floor(2^63 * 0.7^v)
# (so P(X >= v+1) = 0.7^v up to 2^-63), computed exactly with rationals.
C5_THRESH = np.array([int(Fraction(2**63) * Fraction(7, 10) ** v) for v in range(256)], dtype=np.uint64)


def gen_counter_c5_rows(data_seed: int, rows, dim: int) -> np.ndarray:
    b = entry_bits(data_seed, rows, dim)
    u = b & np.uint64((1 << 63) - 1)
    # X = #{v in 0..254 : u < T_v}; T strictly decreases and T_0 = 2^63 > u, so X in [1, 255]
    asc = C5_THRESH[:255][::-1].copy()
    x = 255 - np.searchsorted(asc, u, side="right")
    v = x.astype(np.uint8)
    v[(b >> np.uint64(63)) == np.uint64(1)] = 0
    return v


def gen_counter_c5_rows_slow(data_seed: int, rows, dim: int) -> np.ndarray:
    """Literal per-entry loop of the c5 recipe (for testing the vectorised form)."""
    out = np.zeros((len(rows), dim), np.uint8)
    base = fmix64_int(data_seed)
    for i, n in enumerate(rows):
        for c in range(dim):
            b = fmix64_int(base ^ ((int(n) * dim + c) & MASK64))
            if b >> 63:
                continue
            u = b & ((1 << 63) - 1)
            x = 0
            while x < 255 and u < int(C5_THRESH[x]):
                x += 1
            out[i, c] = x
    return out


# ------------------------------------------------- device twin (gen_kernels.cu)
_GEN_SO = None


def build_gen(force: bool = False) -> str:
    """Compile gen_kernels.cu (sm_100a) into datagen/libwmhgen.so."""
    import os
    import subprocess
    here = os.path.dirname(os.path.abspath(__file__))
    src, so = os.path.join(here, "gen_kernels.cu"), os.path.join(here, "libwmhgen.so")
    if force or not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        tmp = so + f".tmp{os.getpid()}"
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                               "-Xcompiler", "-fPIC", "-o", tmp, src])
        os.replace(tmp, so)
    return so


def gpu_counter_rows(name: str, data_seed: int, row0: int, n_rows: int, dim: int, device="cuda"):
    """Rows row0 .. row0+n_rows-1 of the c1 / c5 recipe generated on the GPU
    (bit-identical to gen_counter_c1_rows / gen_counter_c5_rows)."""
    import ctypes
    import torch
    global _GEN_SO
    if _GEN_SO is None:
        L = ctypes.CDLL(build_gen())
        L.wmhgen_counter_rows.restype = ctypes.c_int
        L.wmhgen_counter_rows.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64,
                                          ctypes.c_int64, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.c_void_p]
        _GEN_SO = L
    kind = {"c1": 1, "c5": 5}[name]
    out = torch.empty((n_rows, dim), dtype=torch.uint8, device=device)
    th = torch.from_numpy(C5_THRESH[:255].view(np.int64).copy()).to(device)
    rc = _GEN_SO.wmhgen_counter_rows(kind, fmix64_int(data_seed), row0, n_rows, dim, C1_ZERO_THRESH,
                                     ctypes.c_void_p(th.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                     ctypes.c_void_p(torch.cuda.current_stream(out.device).cuda_stream))
    if rc != 0:
        raise RuntimeError(f"wmhgen_counter_rows failed ({rc})")
    torch.cuda.current_stream(out.device).synchronize()
    del th
    return out


# ----------------------------------------------------------------- data classes
@dataclass
class Dense:
    x: np.ndarray                    # uint8 [N, D]

    @property
    def n_rows(self):
        return self.x.shape[0]

    @property
    def dim(self):
        return self.x.shape[1]

    kind = "dense"


@dataclass
class CSR:
    row_ptr: np.ndarray              # int64 [N+1]
    col: np.ndarray                  # int32 [nnz], ascending within each row
    val: np.ndarray                  # uint8 [nnz], > 0
    dim: int

    @property
    def n_rows(self):
        return len(self.row_ptr) - 1

    kind = "csr"

    def row(self, n):
        a, b = self.row_ptr[n], self.row_ptr[n + 1]
        return self.col[a:b], self.val[a:b]

    def dense_rows(self, rows):
        out = np.zeros((len(rows), self.dim), np.uint8)
        for i, n in enumerate(rows):
            c, v = self.row(n)
            out[i, c] = v
        return out

    def take(self, rows):
        rows = np.asarray(rows, np.int64)
        lens = self.row_ptr[rows + 1] - self.row_ptr[rows]
        rp = np.zeros(len(rows) + 1, np.int64)
        np.cumsum(lens, out=rp[1:])
        idx = np.concatenate([np.arange(self.row_ptr[n], self.row_ptr[n + 1]) for n in rows]) \
            if len(rows) else np.zeros(0, np.int64)
        return CSR(rp, self.col[idx].copy(), self.val[idx].copy(), self.dim)


@dataclass
class CounterRows:
    """Lazy host view of a counter-based config's rows (c1 / c5): any row can be
    regenerated alone, so full-size data need not live in host memory."""
    name: str
    data_seed: int
    row0: int
    n_rows: int
    dim: int
    kind = "dense"

    def rows(self, idx) -> np.ndarray:
        gen = {"c1": gen_counter_c1_rows, "c5": gen_counter_c5_rows}[self.name]
        return gen(self.data_seed, self.row0 + np.asarray(idx, np.int64), self.dim)


@dataclass
class Config:
    name: str
    n_rows: int
    dim: int
    k: int
    cap: int
    sig_bytes: int
    seed: int = 1                    # hash seed (config 1 states seed = 1; others silent -> 1)
    data_seed: int = 0
    fixed_bound: int | None = None   # c4: M_i = 255 for all i
    n_pairs: int = 0                 # c5: wmh_collide on 10M random pairs
    kind: str = "dense"
    extra: dict = field(default_factory=dict)


CONFIGS = {
    "c1": Config("c1", 1_000, 256, 64, 255, 1, data_seed=1001, kind="dense"),
    "c2": Config("c2", 100_000, 1024, 500, 65535, 2, data_seed=1002, kind="dense"),
    "c3": Config("c3", 1_000_000, 1 << 20, 1000, 65535, 2, data_seed=1003, kind="csr"),
    "c4": Config("c4", 200_000, 65536, 4000, 65535, 2, data_seed=1004, kind="csr", fixed_bound=255),
    "c5": Config("c5", 16_000_000, 4096, 1024, 65535, 2, data_seed=1005, kind="dense", n_pairs=10_000_000),
    # f1: c2's histograms as real values, quantised to uint16 fixed point on the device
    "c2r": Config("c2r", 100_000, 1024, 500, 65535, 2, data_seed=1002, kind="dense"),
}


def _chunk_rng(data_seed: int, chunk: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64([data_seed, chunk]))


# ------------------------------------------------------------------- c2 recipe
def gen_c2_rows(data_seed: int, row_begin: int, row_end: int, dim: int = 1024) -> np.ndarray:
    """Dense histogram: g ~ Gamma(0.5, 1); exactly round(0.6*D) entries zeroed
    uniformly; the row rescaled to L1 = 0.5*0.4*D before quantisation
    w = min(255, round(64*g)) (reading R15)."""
    out = np.empty((row_end - row_begin, dim), np.uint8)
    n_zero = int(round(0.6 * dim))
    target = 0.5 * 0.4 * dim
    c0, c1 = row_begin // CHUNK, (row_end - 1) // CHUNK
    for ch in range(c0, c1 + 1):
        rng = _chunk_rng(data_seed, ch)
        lo, hi = ch * CHUNK, (ch + 1) * CHUNK
        g = rng.gamma(0.5, 1.0, size=(CHUNK, dim))
        zero_pos = np.argpartition(rng.random((CHUNK, dim)), n_zero, axis=1)[:, :n_zero]
        np.put_along_axis(g, zero_pos, 0.0, axis=1)
        s = g.sum(axis=1, keepdims=True)
        s[s == 0] = 1.0
        g *= target / s
        w = np.minimum(255.0, np.rint(64.0 * g)).astype(np.uint8)
        a, b = max(lo, row_begin), min(hi, row_end)
        out[a - row_begin:b - row_begin] = w[a - lo:b - lo]
    return out


def gen_c2_real_rows(data_seed: int, row_begin: int, row_end: int, dim: int = 1024) -> np.ndarray:
    """c2r (f1): the c2 recipe's real histogram 64*g BEFORE rounding (float32):
    the weights the fixed-point path quantises (reading R18)."""
    out = np.empty((row_end - row_begin, dim), np.float32)
    n_zero = int(round(0.6 * dim))
    target = 0.5 * 0.4 * dim
    c0, c1 = row_begin // CHUNK, (row_end - 1) // CHUNK
    for ch in range(c0, c1 + 1):
        rng = _chunk_rng(data_seed, ch)
        lo, hi = ch * CHUNK, (ch + 1) * CHUNK
        g = rng.gamma(0.5, 1.0, size=(CHUNK, dim))
        zero_pos = np.argpartition(rng.random((CHUNK, dim)), n_zero, axis=1)[:, :n_zero]
        np.put_along_axis(g, zero_pos, 0.0, axis=1)
        s = g.sum(axis=1, keepdims=True)
        s[s == 0] = 1.0
        g *= target / s
        a, b = max(lo, row_begin), min(hi, row_end)
        out[a - row_begin:b - row_begin] = (64.0 * g[a - lo:b - lo]).astype(np.float32)
    return out


# ------------------------------------------------------------------- c3 recipe
_ZIPF_CDF = {}


def _zipf_cdf(n: int, s: float) -> np.ndarray:
    key = (n, s)
    if key not in _ZIPF_CDF:
        w = np.arange(1, n + 1, dtype=np.float64) ** (-s)
        c = np.cumsum(w)
        _ZIPF_CDF[key] = c / c[-1]
    return _ZIPF_CDF[key]


def _distinct_sorted_fill(rng, nnz: np.ndarray, sampler) -> list[np.ndarray]:
    """Per row: draw ids with `sampler`, keep the first nnz distinct ones (sequential
    sampling without replacement), return each row's ids sorted ascending."""
    n = len(nnz)
    have = [np.zeros(0, np.int64) for _ in range(n)]
    need = nnz.astype(np.int64).copy()
    todo = np.nonzero(need > 0)[0]
    while len(todo):
        m = (need[todo] * 1.3 + 8).astype(np.int64)
        cand = sampler(int(m.sum()))
        owner = np.repeat(np.arange(len(todo)), m)
        starts = np.concatenate([[0], np.cumsum(m)[:-1]])
        for t_i, r in enumerate(todo):
            c = cand[starts[t_i]:starts[t_i] + m[t_i]]
            merged = np.concatenate([have[r], c])
            _, first = np.unique(merged, return_index=True)
            keep = merged[np.sort(first)][:nnz[r]]
            have[r] = keep
            need[r] = nnz[r] - len(keep)
        del owner
        todo = np.nonzero(need > 0)[0]
    return [np.sort(h) for h in have]


def gen_c3(data_seed: int, n_rows: int, dim: int = 1 << 20) -> CSR:
    """Sparse bag-of-words: nnz ~ round(LogNormal(ln 200 - 1/2, 1)) clipped to
    [1, 8192] (mean 200); distinct column ids by Zipf(1.1) rank (id = rank-1)
    sampled without replacement; tf = min(31, 1 + Poisson(1.5))."""
    cdf = _zipf_cdf(dim, 1.1)
    rps, cols, vals = [np.zeros(1, np.int64)], [], []
    total = 0
    for ch in range((n_rows + CHUNK - 1) // CHUNK):
        rng = _chunk_rng(data_seed, ch)
        cnt = min(CHUNK, n_rows - ch * CHUNK)
        nnz = np.clip(np.rint(rng.lognormal(math.log(200) - 0.5, 1.0, size=CHUNK)), 1, 8192).astype(np.int64)
        nnz = np.minimum(nnz, dim)[:cnt]
        ids = _distinct_sorted_fill(rng, nnz, lambda m: np.minimum(np.searchsorted(cdf, rng.random(m)), dim - 1))
        v = np.minimum(31, 1 + rng.poisson(1.5, size=int(nnz.sum()))).astype(np.uint8)
        c = np.concatenate(ids).astype(np.int32) if ids else np.zeros(0, np.int32)
        cols.append(c)
        vals.append(v)
        rps.append(total + np.cumsum(nnz))
        total += int(nnz.sum())
    return CSR(np.concatenate(rps), np.concatenate(cols), np.concatenate(vals), dim)


# ------------------------------------------------------------------- c4 recipe
def gen_c4(data_seed: int, n_rows: int, dim: int = 65536, nnz_lo: int = 32, nnz_hi: int = 4096) -> CSR:
    """Low effective sparsity: nnz ~ U{32..4096}; distinct uniform columns,
    sorted; weights U{1..255}; bounds fixed at 255."""
    rps, cols, vals = [np.zeros(1, np.int64)], [], []
    total = 0
    for ch in range((n_rows + CHUNK - 1) // CHUNK):
        rng = _chunk_rng(data_seed, ch)
        cnt = min(CHUNK, n_rows - ch * CHUNK)
        nnz = rng.integers(nnz_lo, min(nnz_hi, dim) + 1, size=CHUNK)[:cnt]
        for r in range(cnt):
            cols.append(np.sort(rng.choice(dim, size=int(nnz[r]), replace=False)).astype(np.int32))
        vals.append(rng.integers(1, 256, size=int(nnz.sum())).astype(np.uint8))
        rps.append(total + np.cumsum(nnz))
        total += int(nnz.sum())
    return CSR(np.concatenate(rps), np.concatenate(cols), np.concatenate(vals), dim)


# ---------------------------------------------------------------- entry points
def make(name: str, n_rows: int | None = None, dim: int | None = None):
    """Generate config `name` (optionally with fewer rows / another dim for small
    parity cases).  Returns (Config, Dense | CSR)."""
    cfg = CONFIGS[name]
    n = cfg.n_rows if n_rows is None else n_rows
    d = cfg.dim if dim is None else dim
    if name == "c1":
        data = Dense(gen_counter_c1_rows(cfg.data_seed, np.arange(n), d))
    elif name == "c2":
        data = Dense(gen_c2_rows(cfg.data_seed, 0, n, d))
    elif name == "c3":
        data = gen_c3(cfg.data_seed, n, d)
    elif name == "c4":
        data = gen_c4(cfg.data_seed, n, d)
    elif name == "c5":
        data = Dense(gen_counter_c5_rows(cfg.data_seed, np.arange(n), d))
    else:
        raise KeyError(name)
    return cfg, data


def fig2_pairs(dim: int = 64, seed: int = 2016):
    """Nine pairs (x_j, y_j) with generalized Jaccard exactly j/10, j = 1..9 --
    SPEC's stand-in for Figure 2's unnamed pairs: a shared
    block with total 20j (x = y there), an x-only and a y-only block with total
    10(10 - j) each, the totals split over 16 coordinates per block by a seeded
    integer partition.  Returns (x [9, dim] uint8, y [9, dim] uint8, [j/10])."""
    assert dim >= 48
    rng = np.random.default_rng(seed)

    def split(total, n):
        cuts = np.sort(rng.choice(np.arange(1, total), size=min(n, total) - 1, replace=False))
        parts = np.diff(np.concatenate([[0], cuts, [total]]))
        out = np.zeros(n, np.int64)
        out[:len(parts)] = parts
        rng.shuffle(out)
        return out

    x = np.zeros((9, dim), np.uint8)
    y = np.zeros((9, dim), np.uint8)
    for j in range(1, 10):
        perm = rng.permutation(dim)
        sh, xo, yo = perm[:16], perm[16:32], perm[32:48]
        w = split(20 * j, 16)
        x[j - 1, sh] = w
        y[j - 1, sh] = w
        x[j - 1, xo] = split(10 * (10 - j), 16)
        y[j - 1, yo] = split(10 * (10 - j), 16)
    return x, y, [j / 10 for j in range(1, 10)]


def random_pairs(seed: int, n_rows: int, n_pairs: int) -> np.ndarray:
    """Uniform random (a, b) row pairs, a != b, int64 [P, 2]."""
    rng = np.random.Generator(np.random.PCG64([seed, 0xC011]))
    a = rng.integers(0, n_rows, size=n_pairs)
    b = rng.integers(0, n_rows - 1, size=n_pairs)
    b = b + (b >= a)
    return np.stack([a, b], axis=1).astype(np.int64)
