"""B200-native rejection-sampling weighted minwise hashing (arXiv 1602.08393).

Thin Python binding over the C ABI of ``libwmh.so`` (``include/wmh.h``):
argument marshalling only -- every step of the hot path runs in the sm_100a
kernels.  PyTorch is used for device memory, streams and ``torch.distributed``
(the cross-GPU maxima exchange in :func:`prepare`).  There is no CPU fallback:
every compute call raises if the extension or a CUDA device is missing.

    rows   = Rows.from_dense(x_uint8_cuda)          # or Rows.from_csr(row_ptr, col, val, dim)
    layout = prepare(rows)                          # a1-a4 (+ NCCL max over `group`)
    sig    = hash(layout, rows, seed=1, k=500, cap=65535)      # a5-a9
    m, j   = collide(sig, pairs)                    # a10 (Eq. 14)
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import WmhError  # noqa: F401

__all__ = ["Rows", "Layout", "colmax", "reduce_bounds", "shard", "prepare", "hash", "hash_host", "collide", "WmhError",
           "version", "quantize", "scale_objective", "choose_scale", "LSH", "Hasher", "gather_signatures", "Sketch",
           "sketch", "collide_sketches"]


def _stream(stream=None) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream)


def _ptr(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _need_cuda(t: torch.Tensor, name: str):
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


_WEIGHT_BYTES = {torch.uint8: 1, torch.uint16: 2, torch.float32: 4}


@dataclass
class Rows:
    """A batch of vectors x >= 0, dense or CSR, with uint8 or uint16 integer
    weights (uint16: fixed-point real data, see quantize), or float32 weights for
    scale_objective only."""
    kind: int
    n_rows: int
    dim: int
    dense: torch.Tensor | None = None
    row_ptr: torch.Tensor | None = None
    col: torch.Tensor | None = None
    val: torch.Tensor | None = None
    nnz: int = 0
    weight_bytes: int = 1

    @staticmethod
    def from_dense(x: torch.Tensor) -> "Rows":
        if x.dtype not in _WEIGHT_BYTES or x.dim() != 2:
            raise ValueError("dense rows must be a 2-D uint8 / uint16 (or float32 for scale_objective) tensor")
        return Rows(_lib.WMH_DENSE, x.shape[0], x.shape[1], dense=x, weight_bytes=_WEIGHT_BYTES[x.dtype])

    @staticmethod
    def from_csr(row_ptr: torch.Tensor, col: torch.Tensor, val: torch.Tensor, dim: int) -> "Rows":
        if row_ptr.dtype != torch.int64 or col.dtype != torch.int32 or val.dtype not in _WEIGHT_BYTES:
            raise ValueError("CSR rows need row_ptr int64, col int32, val uint8 / uint16 (or float32)")
        return Rows(_lib.WMH_CSR, row_ptr.numel() - 1, int(dim), row_ptr=row_ptr, col=col, val=val,
                    nnz=col.numel(), weight_bytes=_WEIGHT_BYTES[val.dtype])

    def _c(self, device: bool = True) -> _lib.WmhRows:
        for name in ("dense", "row_ptr", "col", "val"):
            t = getattr(self, name)
            if t is not None and device:
                _need_cuda(t, name)
        return _lib.WmhRows(self.kind, self.n_rows, self.dim,
                            None if self.dense is None else self.dense.data_ptr(),
                            None if self.row_ptr is None else self.row_ptr.data_ptr(),
                            None if self.col is None else self.col.data_ptr(),
                            None if self.val is None else self.val.data_ptr(), self.nnz,
                            self.weight_bytes if self.weight_bytes in (1, 2) else 1)

    def slice(self, begin: int, end: int) -> "Rows":
        """Rows [begin, end) as a view (dense) or a re-based copy of row_ptr (CSR)."""
        if self.kind == _lib.WMH_DENSE:
            return Rows.from_dense(self.dense[begin:end])
        rp = self.row_ptr[begin:end + 1]
        a = int(rp[0].item())
        b = int(rp[-1].item())
        return Rows.from_csr((rp - a).contiguous(), self.col[a:b], self.val[a:b], self.dim)



class _CudaArray:
    """Zero-copy view of a library-owned device array (treat as read-only)."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3}


class Layout:
    """The red-green layout: bounds m_c, CompToM (Eq. 3) and IntToComp (Alg. 4)."""

    def __init__(self, handle: int, keepalive=None):
        self._h = ctypes.c_void_p(handle)
        dim, M, flags, ub = ctypes.c_int64(), ctypes.c_uint64(), ctypes.c_uint32(), ctypes.c_uint32()
        _lib.check(_lib.load().wmh_layout_info(self._h, ctypes.byref(dim), ctypes.byref(M), ctypes.byref(flags),
                                               ctypes.byref(ub)))
        self.dim, self.M, self.flags, self.uniform_bound = dim.value, M.value, flags.value, ub.value
        dg = ctypes.c_uint64()
        _lib.check(_lib.load().wmh_layout_digest(self._h, ctypes.byref(dg)))
        self.digest = dg.value              # FNV-1a over (dim, bounds): the "same layout" key

    @property
    def handle(self):
        return self._h

    def tables(self):
        """(comp_to_m[D+1], int_to_comp[M], bounds[D]) as read-only uint32 CUDA tensors (views)."""
        c2m, i2c, b = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        _lib.check(_lib.load().wmh_layout_tables(self._h, ctypes.byref(c2m), ctypes.byref(i2c), ctypes.byref(b)))
        dev = torch.device("cuda", torch.cuda.current_device())
        mk = lambda p, n: torch.as_tensor(_CudaArray(p.value, n, "<u4"), device=dev)  # noqa: E731
        return mk(c2m, self.dim + 1), mk(i2c, self.M), mk(b, self.dim)

    def close(self):
        if self._h:
            torch.cuda.synchronize()
            _lib.load().wmh_layout_free(self._h)
            self._h = ctypes.c_void_p(0)

    def __del__(self):
        try:
            if self._h and self._h.value:
                _lib.load().wmh_layout_free(self._h)
        except Exception:
            pass


def colmax(rows: Rows, stream=None) -> torch.Tensor:
    """a1: per-column maxima of `rows` (uint32 [D] on the rows' device)."""
    _no_float(rows, "colmax")
    dev = (rows.dense if rows.dense is not None else rows.col).device
    out = torch.empty(rows.dim, dtype=torch.uint32, device=dev)
    _lib.check(_lib.load().wmh_colmax(ctypes.byref(rows._c()), _ptr(out), _stream(stream)))
    return out


def reduce_bounds(bounds: torch.Tensor, group=None) -> torch.Tensor:
    """a2: m <- elementwise max over the ranks of `group` (in place; returns it).

    `group`: None = the default group when a multi-rank job is initialised,
    False = no reduction, else a ProcessGroup.  The uint32 bounds travel as an
    int32 view (values <= 65535, so the bits are the same) so NCCL and gloo both take them."""
    dist = torch.distributed
    if group is False:
        return bounds
    world = dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1
    if world:
        dist.all_reduce(bounds.view(torch.int32), op=dist.ReduceOp.MAX, group=group)
    return bounds


def gather_signatures(sig: torch.Tensor, group=None) -> torch.Tensor:
    """The optional signature exchange of the multi-GPU path (north star: "NCCL ...
    optionally, the signatures"): every rank's [n_r, k] shard, concatenated in
    rank order on every rank (torch.distributed all-gather; shards may differ in
    size by the shard() split).  A single-process call returns `sig` itself."""
    dist = torch.distributed
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return sig
    world = dist.get_world_size(group)
    n_local = torch.tensor([sig.shape[0]], dtype=torch.int64, device=sig.device)
    sizes = [torch.zeros_like(n_local) for _ in range(world)]
    dist.all_gather(sizes, n_local, group=group)
    sizes = [int(t.item()) for t in sizes]
    n_max = max(sizes)
    row_bytes = sig.shape[1] * sig.element_size()                     # bytes travel (NCCL and gloo take uint8)
    buf = torch.zeros((n_max, row_bytes), dtype=torch.uint8, device=sig.device)
    buf[:sig.shape[0]] = sig.contiguous().view(torch.uint8).view(sig.shape[0], row_bytes)
    out = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(out, buf, group=group)
    return torch.cat([o[:n] for o, n in zip(out, sizes)]).view(sig.dtype).view(-1, sig.shape[1])


def shard(n_rows: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous row block [lo, hi) of rank `rank` out of `world` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, rem = divmod(n_rows, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def prepare(rows: Rows | None = None, bounds: torch.Tensor | None = None, group=None, validate: bool = True,
            stream=None) -> Layout:
    """a1-a4.  Without `bounds`, m_c is the column max of `rows`, reduced with an
    all-reduce(MAX) over the torch.distributed `group` (None = the default group
    when a multi-rank job is initialised; False = no reduction).  That is the
    only collective of the path: it makes M -- hence every draw -- identical on
    every rank."""
    if bounds is None:
        if rows is None:
            raise ValueError("prepare needs rows or bounds")
        bounds = reduce_bounds(colmax(rows, stream), group)
    else:
        _need_cuda(bounds, "bounds")
        if bounds.dtype not in (torch.uint32, torch.int32):
            raise ValueError("bounds must be uint32/int32")
    h = ctypes.c_void_p()
    crows = ctypes.byref(rows._c()) if (rows is not None and validate) else None
    _lib.check(_lib.load().wmh_prepare(_ptr(bounds), bounds.numel(), crows, ctypes.byref(h), _stream(stream)))
    return Layout(h.value)


def check_rows(layout: Layout, rows: Rows, stream=None) -> None:
    """Raise WmhError (EBOUND / EINVAL) unless every weight of `rows` is within the
    layout's bounds x_c <= m_c and CSR rows are well formed."""
    _no_float(rows, "check_rows")
    _lib.check(_lib.load().wmh_check_rows(layout.handle, ctypes.byref(rows._c()), _stream(stream)))


last_algo = None     # name of the kernel the last hash() call ran ('simple' / 'tiled' / 'index')
last_horizon = None  # the index horizon T of the last hash() call that ran the index kernel
last_tile = None     # the dense tile of the last hash() call that ran TILED ('bytes' / 'bitplanes' / 'bitslice')


def hash(layout: Layout, rows: Rows, seed: int, k: int, cap: int, sig_bytes: int | None = None,
         algo: str = "auto", out: torch.Tensor | None = None, n_saturated: torch.Tensor | None = None,
         chunk: int = 0, horizon: int = 0, time_kernel: bool = False, stream=None,
         tile: str = "auto", validate: bool = False, plan_out: torch.Tensor | None = None,
         isgreen: str = "table") -> torch.Tensor:
    """a5-a9: signatures sig[n][j] = h_j(x_n) (uint8 when sig_bytes = 1, else uint16).
    `tile` ("auto", "bytes", "bitplanes", "bitslice") picks the TILED kernel's dense tile
    (performance only).  `validate` checks every row against the layout's bounds
    first (wmh_check_rows: WmhError EBOUND instead of silently wrong signatures
    for rows prepare() did not see).  `plan_out` (uint8 [n_rows], tests): the INDEX
    kernel's per-row plan codes (include/wmh.h, wmh_hash_opts.plan_out).  `isgreen` ("table" or
    "bsearch"): Alg. 5's component lookup by IntToComp or by binary search over CompToM (Sec. 3.3;
    SIMPLE per draw, the bit-sliced tile's draw table) -- same results."""
    if sig_bytes is None:
        sig_bytes = 1 if cap <= 255 else 2
    dtype = torch.uint8 if sig_bytes == 1 else torch.uint16
    dev = (rows.dense if rows.dense is not None else rows.row_ptr).device
    if out is None:
        out = torch.empty((rows.n_rows, k), dtype=dtype, device=dev)
    elif out.dtype != dtype or out.numel() != rows.n_rows * k:
        raise ValueError("out has the wrong dtype or size")
    _no_float(rows, "hash")
    if n_saturated is not None and (n_saturated.dtype not in (torch.int64, torch.uint64) or not n_saturated.is_cuda):
        raise ValueError("n_saturated must be a CUDA int64 tensor")
    if tile not in ("auto", "bytes", "bitplanes", "bitslice"):
        raise ValueError(f"tile must be auto, bytes, bitplanes or bitslice, not {tile!r}")
    if isgreen not in ("table", "bsearch"):
        raise ValueError("isgreen must be 'table' (IntToComp) or 'bsearch' (binary search over CompToM)")
    flags = (_lib.WMH_OPT_TIME_KERNEL if time_kernel else 0) | (_lib.WMH_OPT_VALIDATE if validate else 0) | \
        (_lib.WMH_OPT_ISGREEN_BINSEARCH if isgreen == "bsearch" else 0) | \
        {"auto": 0, "bytes": _lib.WMH_OPT_TILE_BYTES, "bitplanes": _lib.WMH_OPT_TILE_BITPLANES,
         "bitslice": _lib.WMH_OPT_TILE_BITSLICE}[tile]
    if plan_out is not None and (plan_out.dtype != torch.uint8 or plan_out.numel() < rows.n_rows or not plan_out.is_cuda):
        raise ValueError("plan_out must be a CUDA uint8 tensor of >= n_rows elements")
    opts = _lib.WmhHashOpts(_lib.ALGOS[algo], chunk, 0, horizon, flags, None if plan_out is None else plan_out.data_ptr())
    _lib.check(_lib.load().wmh_hash_ex(layout.handle, ctypes.byref(rows._c()), seed & (2**64 - 1), k, cap, sig_bytes,
                                       _ptr(out), _ptr(n_saturated), ctypes.byref(opts), _stream(stream)))
    global last_algo, last_horizon, last_tile
    last_algo = {v: n for n, v in _lib.ALGOS.items()}.get(opts.algo_used, "?")
    last_horizon = int(opts.horizon) if last_algo == "index" else None
    last_tile = {1: "bytes", 2: "bitplanes", 3: "bitslice"}.get(int(opts.tile_used))
    return out


def hash_host(layout: Layout, rows_host, seed: int, k: int, cap: int, sig_bytes: int | None = None,
              out: np.ndarray | torch.Tensor | None = None, stream=None):
    """End-to-end through the C ABI with HOST buffers (wmh_hash_host): H2D of the
    rows, the hash, D2H of the signatures, synchronised.  `rows_host` is a Rows
    of CPU tensors (pinned for full PCIe speed)."""
    if sig_bytes is None:
        sig_bytes = 1 if cap <= 255 else 2
    dtype = torch.uint8 if sig_bytes == 1 else torch.uint16
    for name in ("dense", "row_ptr", "col", "val"):
        t = getattr(rows_host, name)
        if t is not None and (t.is_cuda or not t.is_contiguous()):
            raise ValueError(f"hash_host: rows_host.{name} must be a contiguous CPU tensor")
    if out is None:
        out = torch.empty((rows_host.n_rows, k), dtype=dtype)
    elif isinstance(out, np.ndarray):
        if out.dtype != (np.uint8 if sig_bytes == 1 else np.uint16) or not out.flags["C_CONTIGUOUS"]:
            raise ValueError("hash_host: out must be a C-contiguous uint8/uint16 array matching sig_bytes")
        out = torch.from_numpy(out)
    if out.is_cuda or out.dtype != dtype or not out.is_contiguous() or out.numel() != rows_host.n_rows * k:
        raise ValueError(f"hash_host: out must be a contiguous CPU {dtype} tensor of n_rows*k = {rows_host.n_rows * k} "
                         "elements")
    c = rows_host._c(device=False)
    _lib.check(_lib.load().wmh_hash_host(layout.handle, ctypes.byref(c), seed & (2**64 - 1), k, cap, sig_bytes,
                                         ctypes.c_void_p(out.data_ptr()), _stream(stream)))
    return out


def _no_float(rows: Rows, what: str):
    if rows.weight_bytes == 4:
        raise ValueError(f"{what} takes integer weights; quantize float32 rows first")


def quantize(x: torch.Tensor, scale: float, stream=None) -> torch.Tensor:
    """f1: uint16 fixed-point weights floor(x * scale) (float32 product, then floor;
    clamped at 65535) of a float32 CUDA tensor of weights >= 0 (Sec. 3.1 / Sec. 4)."""
    _need_cuda(x, "x")
    if x.dtype != torch.float32:
        raise ValueError("quantize takes float32 weights")
    out = torch.empty(x.shape, dtype=torch.uint16, device=x.device)
    _lib.check(_lib.load().wmh_quantize(_ptr(x), x.numel(), float(scale), _ptr(out), _stream(stream)))
    return out


def scale_objective(rows: Rows, scales, stream=None) -> list[tuple[int, int, int]]:
    """Sec. 4: for each candidate scale, (numerator, denominator, clipped) of
    the mean effective sparsity of the rows quantised at that scale: sum floor(x*s),
    n_rows * sum_c max_n floor(x*s), and the number of weights the uint16 quantiser
    would saturate.  `rows` holds float32 weights."""
    if rows.weight_bytes != 4:
        raise ValueError("scale_objective takes float32 rows")
    sc = (ctypes.c_float * len(scales))(*[float(v) for v in scales])
    out = (ctypes.c_uint64 * (3 * len(scales)))()
    _lib.check(_lib.load().wmh_scale_objective(ctypes.byref(rows._c()), sc, len(scales), out, _stream(stream)))
    return [(int(out[3 * i]), int(out[3 * i + 1]), int(out[3 * i + 2])) for i in range(len(scales))]


def choose_scale(rows: Rows, scales, stream=None) -> float:
    """Sec. 4's alpha = argmax sum alpha x / sum ceil(alpha m) over `scales`,
    chosen in C (wmh_choose_scale): the candidate with the largest mean effective
    sparsity among those that do not saturate a weight; ties: the smaller scale."""
    if rows.weight_bytes != 4:
        raise ValueError("choose_scale takes float32 rows")
    sc = (ctypes.c_float * len(scales))(*[float(v) for v in scales])
    best = ctypes.c_int32(-1)
    _lib.check(_lib.load().wmh_choose_scale(ctypes.byref(rows._c()), sc, len(scales), ctypes.byref(best),
                                            _stream(stream)))
    return float(scales[best.value])


def collide(sig: torch.Tensor, pairs: torch.Tensor, check_pairs: bool = True, stream=None):
    """a10: (matches uint32 [P], jhat float32 [P]) with jhat = matches / k (Eq. 14)."""
    _need_cuda(sig, "sig")
    _need_cuda(pairs, "pairs")
    if pairs.dtype != torch.int64:
        raise ValueError("pairs must be int64 [P, 2]")
    sb = sig.element_size()
    n_rows, k = sig.shape
    P = pairs.numel() // 2
    matches = torch.empty(P, dtype=torch.uint32, device=sig.device)
    jhat = torch.empty(P, dtype=torch.float32, device=sig.device)
    _lib.check(_lib.load().wmh_collide(_ptr(sig), sb, k, n_rows, _ptr(pairs), P, _ptr(matches), _ptr(jhat),
                                       1 if check_pairs else 0, _stream(stream)))
    return matches, jhat


@dataclass
class Sketch:
    """Signatures with the metadata that decides whether two sets of them are
    comparable: the same (seed, k, cap) over layouts with
    the same digest (equal bounds, hence the same draw stream)."""
    sig: torch.Tensor
    seed: int
    k: int
    cap: int
    digest: int

    def key(self):
        return (self.seed & (2**64 - 1), self.k, self.cap, self.digest)


def sketch(layout: Layout, rows: Rows, seed: int, k: int, cap: int, **kw) -> Sketch:
    """hash() wrapped with its metadata."""
    return Sketch(hash(layout, rows, seed, k, cap, **kw), seed, k, cap, layout.digest)


def collide_sketches(a: Sketch, b: Sketch, ia: torch.Tensor, ib: torch.Tensor, stream=None):
    """a10 across two sketches: matches / J-hat of rows a.sig[ia[p]] and b.sig[ib[p]].
    Refuses (ValueError) sketches of a different seed, k, cap or layout."""
    if a.key() != b.key():
        names = ("seed", "k", "cap", "layout digest")
        diff = [n for n, x, y in zip(names, a.key(), b.key()) if x != y]
        raise ValueError(f"sketches are not comparable: different {', '.join(diff)}")
    if a.sig.dtype != b.sig.dtype:
        raise ValueError("sketches have different signature widths")
    _need_cuda(a.sig, "a.sig")
    _need_cuda(b.sig, "b.sig")
    pairs = torch.stack([ia.to(torch.int64), ib.to(torch.int64)], dim=1).contiguous()
    P = pairs.shape[0]
    matches = torch.empty(P, dtype=torch.uint32, device=a.sig.device)
    jhat = torch.empty(P, dtype=torch.float32, device=a.sig.device)
    _lib.check(_lib.load().wmh_collide2(_ptr(a.sig), a.sig.shape[0], _ptr(b.sig), b.sig.shape[0], a.sig.element_size(),
                                        a.k, _ptr(pairs), P, _ptr(matches), _ptr(jhat), 1, _stream(stream)))
    return matches, jhat


class Hasher:
    """A prepared hash family (seed, k, cap) over `layout`: the draws are filed once
    (the index build) and every .hash(rows) call runs only the row pass -- for
    streaming many batches.  Signatures equal hash(layout, rows, seed, k, cap)."""

    def __init__(self, layout: Layout, seed: int, k: int, cap: int, horizon: int = 0, stream=None):
        self.layout, self.seed, self.k, self.cap = layout, seed, k, cap
        h = ctypes.c_void_p()
        _lib.check(_lib.load().wmh_hasher_create(layout.handle, seed & (2**64 - 1), k, cap, horizon, ctypes.byref(h),
                                                 _stream(stream)))
        self._h = h

    def hash(self, rows: Rows, sig_bytes: int | None = None, out: torch.Tensor | None = None,
             n_saturated: torch.Tensor | None = None, stream=None, validate: bool = False) -> torch.Tensor:
        """`validate`: check the batch against the layout's bounds first (check_rows)."""
        _no_float(rows, "Hasher.hash")
        if validate:
            check_rows(self.layout, rows, stream)
        if sig_bytes is None:
            sig_bytes = 1 if self.cap <= 255 else 2
        dtype = torch.uint8 if sig_bytes == 1 else torch.uint16
        dev = (rows.dense if rows.dense is not None else rows.row_ptr).device
        if out is None:
            out = torch.empty((rows.n_rows, self.k), dtype=dtype, device=dev)
        elif out.dtype != dtype or out.numel() != rows.n_rows * self.k:
            raise ValueError("out has the wrong dtype or size")
        _lib.check(_lib.load().wmh_hasher_run(self._h, ctypes.byref(rows._c()), sig_bytes, _ptr(out),
                                              _ptr(n_saturated), _stream(stream)))
        return out

    def __del__(self):
        try:
            if self._h and self._h.value:
                _lib.load().wmh_hasher_free(self._h)
        except Exception:
            pass


class LSH:
    """f3: (K, L) banding LSH over a signature tensor: band b = hashes
    [bK, (b+1)K); candidates of a query = rows equal to it in >= 1 band.  Keeps a
    reference to `sig` (the index reads it at query time)."""

    def __init__(self, sig: torch.Tensor, K: int, L: int, stream=None):
        _need_cuda(sig, "sig")
        if sig.dim() != 2 or sig.dtype not in (torch.uint8, torch.uint16):
            raise ValueError("sig must be a 2-D uint8/uint16 CUDA tensor")
        self.sig, self.K, self.L = sig, K, L
        h = ctypes.c_void_p()
        _lib.check(_lib.load().wmh_lsh_build(_ptr(sig), sig.element_size(), sig.shape[1], sig.shape[0], K, L,
                                             ctypes.byref(h), _stream(stream)))
        self._h = h

    def query(self, qsig: torch.Tensor, max_out: int = 64, stream=None):
        """(counts uint32 [n_q], rows int64 [n_q, max_out], -1 where unused)."""
        _need_cuda(qsig, "qsig")
        if qsig.dtype != self.sig.dtype or qsig.dim() != 2 or qsig.shape[1] != self.sig.shape[1]:
            raise ValueError("query signatures must match the indexed ones (dtype, k)")
        n_q = qsig.shape[0]
        counts = torch.empty(n_q, dtype=torch.uint32, device=qsig.device)
        rows = torch.full((n_q, max_out), -1, dtype=torch.int64, device=qsig.device)
        _lib.check(_lib.load().wmh_lsh_query(self._h, _ptr(qsig), n_q, max_out, _ptr(rows), _ptr(counts),
                                             _stream(stream)))
        return counts, rows

    def __del__(self):
        try:
            if self._h and self._h.value:
                torch.cuda.synchronize()
                _lib.load().wmh_lsh_free(self._h)
        except Exception:
            pass


def version() -> str:
    return _lib.load().wmh_version().decode()


def last_kernel_ms() -> float:
    """Device time of the dominant kernel of the last hash(..., time_kernel=True) call on
    this thread (CUDA events on its stream; waits for it)."""
    ms = ctypes.c_float()
    _lib.check(_lib.load().wmh_last_kernel_ms(ctypes.byref(ms)))
    return float(ms.value)


def empty_launch(stream=None) -> None:
    """One empty kernel of the library on the stream (the launch floor)."""
    _lib.check(_lib.load().wmh_empty_launch(_stream(stream)))


def kernel_launches() -> int:
    """How many CUDA kernels libwmh.so has launched in this process."""
    return int(_lib.load().wmh_kernel_launches())
