"""GPU parity: every output of the CUDA path (through the C ABI) against the CPU
oracle on the same seeded inputs.  Integer outputs are compared bit-exactly
(BASELINE.json north_star: "GPU signatures must match the oracle bit-exactly")."""
import math

import numpy as np
import pytest
import torch

import datagen
import oracle
from tests.helpers import oracle_bounds, oracle_hash, to_rows

pytestmark = pytest.mark.gpu

ALGOS = ["simple", "tiled", "index", "auto"]


@pytest.fixture(scope="module")
def wmh():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1602_08393_b200 as w
    from paper_1602_08393_b200 import build
    build.build()
    return w


def _assert_sig_equal(gpu, ref, what=""):
    gpu = gpu.cpu().numpy().astype(np.uint32)
    if not np.array_equal(gpu, ref):
        bad = np.argwhere(gpu != ref)
        r, j = bad[0]
        raise AssertionError(f"{what}: {len(bad)} mismatches; first at row {r} hash {j}: gpu {gpu[r, j]} "
                             f"oracle {ref[r, j]}")


def _run(wmh, data, cfg, k, cap, sig_bytes, algo, seed=None, fixed_bound=None, horizon=0, tile="auto"):
    rows = to_rows(data)
    seed = cfg.seed if seed is None else seed
    m = oracle_bounds(data, fixed_bound)
    if fixed_bound is not None:
        layout = wmh.prepare(rows, bounds=torch.from_numpy(m).cuda())
    else:
        layout = wmh.prepare(rows)
    L = oracle.Layout(m)
    assert layout.M == L.M
    try:
        sig = wmh.hash(layout, rows, seed, k, cap, sig_bytes, algo=algo, horizon=horizon, tile=tile)
    except wmh.WmhError as e:
        if algo == "tiled" and "does not take" in str(e):
            pytest.skip("tiled kernel does not take this shape")
        raise
    torch.cuda.synchronize()
    return sig, L, layout


# ------------------------------------------------------------------ prepare
@pytest.mark.parametrize("name,n", [("c1", 1000), ("c2", 700), ("c3", 300), ("c4", 60), ("c5", 300)])
def test_prepare_tables_match_oracle(wmh, name, n):
    """a1 colmax, a3 CompToM (Eq. 3), a4 IntToComp (Alg. 4) bit-exact."""
    cfg, data = datagen.make(name, n_rows=n)
    rows = to_rows(data)
    cm = wmh.colmax(rows).cpu().numpy()
    m = oracle_bounds(data)
    assert np.array_equal(cm, m)
    if cfg.fixed_bound is not None:
        m = oracle_bounds(data, cfg.fixed_bound)
        layout = wmh.prepare(rows, bounds=torch.from_numpy(m).cuda())
    else:
        layout = wmh.prepare(rows)
    L = oracle.Layout(m)
    c2m, i2c, b = layout.tables()
    assert layout.M == L.M
    assert np.array_equal(b.cpu().numpy(), m)
    assert np.array_equal(c2m.cpu().numpy(), L.comp_to_m)
    assert np.array_equal(i2c.cpu().numpy(), L.int_to_comp)
    assert bool(layout.flags & 1) == (m.min() == m.max())


def test_prepare_zero_width_and_errors(wmh):
    m = np.array([3, 0, 0, 5, 1, 0], np.uint32)
    layout = wmh.prepare(bounds=torch.from_numpy(m).cuda())
    L = oracle.Layout(m)
    c2m, i2c, _ = layout.tables()
    assert np.array_equal(c2m.cpu().numpy(), L.comp_to_m) and np.array_equal(i2c.cpu().numpy(), L.int_to_comp)
    with pytest.raises(wmh.WmhError, match="WMH_EEMPTY"):
        wmh.prepare(bounds=torch.zeros(5, dtype=torch.uint32).cuda())
    with pytest.raises(wmh.WmhError, match="WMH_EINVAL"):
        wmh.prepare(bounds=torch.full((5,), 70000, dtype=torch.uint32).cuda())
    wide = wmh.prepare(bounds=torch.full((5,), 300, dtype=torch.uint32).cuda())      # f1: bounds up to 65535
    assert wide.M == 1500 and wide.flags == 3
    x = torch.tensor([[1, 2], [3, 9]], dtype=torch.uint8).cuda()
    with pytest.raises(wmh.WmhError, match=r"WMH_EBOUND.*x\[1\]\[1\]"):
        wmh.prepare(wmh.Rows.from_dense(x), bounds=torch.tensor([3, 5], dtype=torch.uint32).cuda())
    # malformed CSR: descending columns
    rp = torch.tensor([0, 2], dtype=torch.int64).cuda()
    col = torch.tensor([3, 1], dtype=torch.int32).cuda()
    val = torch.tensor([1, 1], dtype=torch.uint8).cuda()
    with pytest.raises(wmh.WmhError, match="ascending"):
        wmh.prepare(wmh.Rows.from_csr(rp, col, val, 8))


def test_prepare_large_dim_scan(wmh):
    """Multi-segment scan (D > 1024^2 / ... ragged block count)."""
    rng = np.random.default_rng(1)
    m = rng.integers(0, 4, size=(1 << 21) + 77).astype(np.uint32)
    layout = wmh.prepare(bounds=torch.from_numpy(m).cuda())
    c2m, i2c, _ = layout.tables()
    ref = np.concatenate([[0], np.cumsum(m.astype(np.uint64))]).astype(np.uint32)
    assert np.array_equal(c2m.cpu().numpy(), ref)
    L = oracle.Layout(m)
    assert np.array_equal(i2c.cpu().numpy(), L.int_to_comp)


# --------------------------------------------------------------------- hash
CASES = [  # name, n_rows, k, cap, sig_bytes
    ("c1", 1000, 64, 255, 1),
    ("c2", 3000, 500, 65535, 2),
    ("c3", 150, 64, 65535, 2),
    ("c4", 80, 256, 65535, 2),
    ("c5", 1500, 128, 65535, 2),
]


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("name,n,k,cap,sb", CASES)
def test_hash_parity_configs(wmh, name, n, k, cap, sb, algo):
    """a5-a9 bit-exact on every config's recipe (smaller N; several tiles and a ragged tail)."""
    cfg, data = datagen.make(name, n_rows=n)
    sig, L, _ = _run(wmh, data, cfg, k, cap, sb, algo, fixed_bound=cfg.fixed_bound)
    ref = oracle_hash(L, data, cfg.seed, k, cap)
    _assert_sig_equal(sig, ref, f"{name}/{algo}")


@pytest.mark.parametrize("horizon", [1, 31, 33, 200, 0, 65535])
@pytest.mark.parametrize("name,n,k", [("c2", 400, 500), ("c3", 60, 200), ("c4", 30, 4000), ("c5", 300, 1500)])
def test_index_horizons(wmh, name, n, k, horizon):
    """INDEX: any horizon T (the filed draws t < T, then Alg. 3's loop from T)
    gives the oracle's signatures -- T = 1 is all fallback, T = cap all index;
    k = 4000 / 1500 / 500 select 8 / 4 / 1 warps per row."""
    cfg, data = datagen.make(name, n_rows=n)
    sig, L, _ = _run(wmh, data, cfg, k, cfg.cap, cfg.sig_bytes, "index", fixed_bound=cfg.fixed_bound,
                     horizon=horizon)
    _assert_sig_equal(sig, oracle_hash(L, data, cfg.seed, k, cfg.cap), f"{name}/index T={horizon}")


@pytest.mark.parametrize("horizon", [1, 0])
@pytest.mark.parametrize("dim", [4097, 66000, 200000])
def test_index_8warp_fallback_lookups(wmh, dim, horizon):
    """INDEX at 8 warps per row (k = 4000) on c4-recipe CSR rows: the fallback's x_c
    lookup through the row's column bitmap in shared memory when it fits the range
    buffers (D = 4097 with a ragged last word, D = 66,000 the widest that fits) and
    through the sampled binary search when it does not (D = 200,000); T = 1 makes
    every hash take the fallback."""
    cfg, data = datagen.make("c4", n_rows=24, dim=dim)
    sig, L, _ = _run(wmh, data, cfg, 4000, cfg.cap, cfg.sig_bytes, "index", fixed_bound=cfg.fixed_bound,
                     horizon=horizon)
    _assert_sig_equal(sig, oracle_hash(L, data, cfg.seed, 4000, cfg.cap), f"c4 D={dim} index T={horizon}")


@pytest.mark.parametrize("algo", ALGOS)
def test_hash_edge_cases_dense(wmh, algo):
    """Empty rows saturate (reading R12), full-green rows give 1, tiny caps
    saturate, odd D, k = 1, one row, zero rows."""
    rng = np.random.default_rng(12)
    D = 37
    x = rng.integers(0, 9, size=(67, D)).astype(np.uint8)
    x[5] = 0                                   # empty row
    x[6] = 8                                   # all at the bound -> full green
    x[7] = 0
    x[7, 3] = 1                                # one cell green
    cfg = datagen.Config("edge", 67, D, 1, 255, 1)
    data = datagen.Dense(x)
    for k, cap, sb in [(1, 255, 1), (33, 3, 1), (40, 1, 1), (70, 65535, 2), (16, 200, 2)]:
        sig, L, _ = _run(wmh, data, cfg, k, cap, sb, algo, seed=99)
        ref = oracle_hash(L, data, 99, k, cap)
        _assert_sig_equal(sig, ref, f"edge k={k} cap={cap}/{algo}")
        assert np.all(sig.cpu().numpy()[5] == cap)
    # zero rows
    layout = wmh.prepare(bounds=torch.full((D,), 8, dtype=torch.uint32).cuda())
    out = wmh.hash(layout, wmh.Rows.from_dense(torch.zeros((0, D), dtype=torch.uint8).cuda()), 1, 8, 100, algo=algo)
    assert out.shape == (0, 8)


@pytest.mark.parametrize("tile", ["bitslice", "bitplanes", "bytes"])
@pytest.mark.parametrize("D,n", [(64, 333), (1024, 200), (2048, 100), (4096, 70)])
@pytest.mark.parametrize("mx", [1, 2, 3, 7, 12, 16, 31, 50, 100, 255])
def test_tiled_bitplanes(wmh, D, n, mx, tile):
    """The three dense tiles; the bit-sliced ones (hash_bitslice.cu, hash_tiled_bs.cu) at every plane count
    NB = 1..8 (the largest bound mx), 8/4/2/1 groups of 32 rows and group- or plane-major plane blocks (D),
    ragged last tile, all-zero rows, rows at the bound, a small cap and the uint8 signature width."""
    rng = np.random.default_rng(1000 * mx + D)
    x = rng.integers(0, mx + 1, size=(n, D)).astype(np.uint8)
    x[rng.random((n, D)) < 0.7] = 0
    x[3] = 0
    x[n - 1] = 0
    x[4] = mx
    x[0, 0] = mx                               # the largest bound is mx
    data = datagen.Dense(x)
    cfg = datagen.Config("bs", n, D, 1, 255, 1)
    for k, cap, sb in [(40, 65535, 2), (24, 9, 1), (13, 65535, 2), (5, 200, 1)]:
        sig, L, layout = _run(wmh, data, cfg, k, cap, sb, "tiled", seed=mx + 7, tile=tile)
        _assert_sig_equal(sig, oracle_hash(L, data, mx + 7, k, cap), f"{tile} D={D} mx={mx} k={k} cap={cap}")
        s = sig.cpu().numpy()
        assert np.all(s[[3, n - 1]] == cap) and np.all(s[4] == 1)
        # saturation counter: every (row, j) of the all-zero rows, at most every h == cap
        nsat = torch.zeros(1, dtype=torch.int64, device="cuda")
        wmh.hash(layout, to_rows(data), mx + 7, k, cap, sb, algo="tiled", tile=tile, n_saturated=nsat)
        dead = int((x.sum(1) == 0).sum())
        assert dead * k <= int(nsat.item()) <= int((s == cap).sum())


@pytest.mark.parametrize("tile", ["bitplanes", "bitslice", "auto"])
def test_tiled_bitplanes_clamped(wmh, tile, capfd, monkeypatch):
    """Long rows whose largest bound needs one plane more than two groups can
    hold (D = 4096, bounds <= 63 except two columns at 100): the planes store
    min(x, 63) and the draws that land in the top cells of the two wide columns
    (off >= 63) are tested on the rows themselves.  Bit-exact with the oracle,
    with rows that are green only in those cells."""
    monkeypatch.setenv("WMH_TILED_STATS", "1")
    rng = np.random.default_rng(77)
    n, D = 70, 4096
    x = (rng.integers(1, 64, size=(n, D)) * (rng.random((n, D)) < 0.05)).astype(np.uint8)
    x[:, 7] = np.where(np.arange(n) % 2 == 0, 100, 0)
    x[:, 2000] = np.where(np.arange(n) % 3 == 0, 90, 5)
    x[10] = 0
    x[10, 7] = 100                               # green only in column 7, 37 of its cells above 63
    x[11] = 0
    x[11, 2000] = 90
    data = datagen.Dense(x)
    cfg = datagen.Config("bsc", n, D, 1, 255, 1)
    for k, cap in [(64, 65535), (16, 300)]:
        sig, L, _ = _run(wmh, data, cfg, k, cap, 2, "tiled", seed=31, tile=tile)
        _assert_sig_equal(sig, oracle_hash(L, data, 31, k, cap), f"clamped {tile} k={k}")
    err = capfd.readouterr().err
    if tile == "bitplanes":
        assert "planes=6" in err and "NB=7" in err, err[-300:]
    else:
        assert "[wmh bitslice] P=6 clamp=1 G=2" in err, err[-300:]


def test_bitslice_thin_tail_clamps_to_fewer_planes(wmh, capfd, monkeypatch):
    """Weights with a thin tail (geometric, a few cells at 70 and 100 so NB = 7):
    prepare's sampled fraction of weights >= 15 is ~1e-5, so the tile keeps 4
    planes and tests the draws in the top cells of the wide columns on the rows'
    bytes -- still bit-exact with the oracle, including the rows that are green
    only there."""
    monkeypatch.setenv("WMH_TILED_STATS", "1")
    rng = np.random.default_rng(79)
    n, D = 200, 4096
    x = np.minimum(rng.geometric(0.5, size=(n, D)) - 1, 12).astype(np.uint8)
    x[5, 10] = 100
    x[6, 11] = 70
    x[7] = 0
    x[7, 10] = 90                                # green only in column 10's cells 15..89
    data = datagen.Dense(x)
    cfg = datagen.Config("thin", n, D, 1, 255, 1)
    for k, cap in [(64, 65535), (16, 300)]:
        sig, L, _ = _run(wmh, data, cfg, k, cap, 2, "tiled", seed=13, tile="bitslice")
        _assert_sig_equal(sig, oracle_hash(L, data, 13, k, cap), f"thin tail k={k}")
    err = capfd.readouterr().err
    assert "[wmh bitslice] P=4 clamp=1 G=2" in err, err[-300:]


def test_bitslice_clamped_group_major(wmh, capfd, monkeypatch):
    """The bit-sliced tile with 4 clamped planes in group-major blocks (D = 2912,
    bounds up to 31: five planes would leave two groups, four give four): the
    draws in cells >= 15 of a column are tested on the candidate rows' bytes
    whenever the group's column maximum says one of them can be green."""
    monkeypatch.setenv("WMH_TILED_STATS", "1")
    rng = np.random.default_rng(78)
    n, D = 300, 2912
    x = rng.integers(0, 16, size=(n, D)).astype(np.uint8)
    x[rng.random((n, D)) < 0.6] = 0
    hi = rng.random((n, D)) < 0.01
    x[hi] = rng.integers(16, 32, size=int(hi.sum())).astype(np.uint8)
    x[0, 0] = 31
    x[20] = 0
    x[20, 5] = 31                                # green only in cells 0..30 of column 5
    data = datagen.Dense(x)
    cfg = datagen.Config("bvc", n, D, 1, 255, 1)
    for k, cap in [(96, 65535), (24, 50)]:
        sig, L, _ = _run(wmh, data, cfg, k, cap, 2, "tiled", seed=5, tile="bitslice")
        _assert_sig_equal(sig, oracle_hash(L, data, 5, k, cap), f"bitslice clamped P=4 k={k}")
    err = capfd.readouterr().err
    assert "[wmh bitslice] P=4 clamp=1 G=4" in err, err[-300:]


@pytest.mark.parametrize("name,n,k,algo,tile", [("c1", 300, 64, "simple", "auto"), ("c5", 150, 96, "simple", "auto"),
                                                 ("c5", 150, 96, "tiled", "bitslice"), ("c3", 50, 64, "simple", "auto"),
                                                 ("zero", 90, 48, "simple", "auto"), ("zero", 90, 48, "tiled", "bitslice")])
def test_isgreen_binary_search(wmh, name, n, k, algo, tile):
    """Sec. 3.3's alternative ISGREEN: the component by binary search over
    CompToM instead of the IntToComp table, in SIMPLE (every draw) and the
    bit-sliced tile's draw table -- bit-identical signatures, including layouts
    with zero-width components (m_c = 0, reading R11) that the search must skip."""
    if name == "zero":
        rng = np.random.default_rng(21)
        x = rng.integers(0, 12, size=(n, 256)).astype(np.uint8)
        x[:, ::3] = 0                              # every third column absent: zero-width intervals
        x[:, 255] = 0
        cfg, data = datagen.Config("zero", n, 256, k, 65535, 2), datagen.Dense(x)
    else:
        cfg, data = datagen.make(name, n_rows=n)
    rows = to_rows(data)
    layout = wmh.prepare(rows)
    L = oracle.Layout(oracle_bounds(data))
    ref = oracle_hash(L, data, 3, k, 65535)
    for isg in ("table", "bsearch"):
        sig = wmh.hash(layout, rows, 3, k, 65535, 2, algo=algo, tile=tile, isgreen=isg)
        _assert_sig_equal(sig, ref, f"{name}/{algo}/{tile}/{isg}")


@pytest.mark.parametrize("algo", ALGOS)
def test_hash_maximum_sizes(wmh, algo):
    """Limits: k = 65536 on CSR rows (the INDEX kernel keeps h[k] in shared
    memory, so it takes k = 50,000 here and rejects 65,536 with a clean
    WMH_EINVAL that leaves no error behind; AUTO picks another kernel), and
    dense rows too long for any shared-memory tile (D = 20000), each bit-exact
    with the oracle."""
    rng = np.random.default_rng(99)
    D = 512
    dense = ((rng.random((3, D)) < 0.5) * rng.integers(1, 16, (3, D))).astype(np.uint8)
    rp = np.concatenate([[0], np.cumsum((dense > 0).sum(1))]).astype(np.int64)
    col = np.concatenate([np.nonzero(r)[0] for r in dense]).astype(np.int32)
    val = np.concatenate([r[r > 0] for r in dense]).astype(np.uint8)
    data = datagen.CSR(rp, col, val, D)
    cfg = datagen.Config("kmax", 3, D, 1, 255, 1)
    kk = 50000 if algo == "index" else 65536
    if algo == "index":
        with pytest.raises(wmh.WmhError, match="index kernel takes k"):
            _run(wmh, data, cfg, 65536, 65535, 2, algo, seed=4)
    sig, L, _ = _run(wmh, data, cfg, kk, 65535, 2, algo, seed=4)
    _assert_sig_equal(sig, oracle_hash(L, data, 4, kk, 65535), f"k={kk}/{algo}")
    D = 20000
    x = ((rng.random((40, D)) < 0.3) * rng.integers(1, 16, (40, D))).astype(np.uint8)
    x[7] = 0
    data = datagen.Dense(x)
    cfg = datagen.Config("dlong", 40, D, 1, 255, 1)
    sig, L, _ = _run(wmh, data, cfg, 24, 65535, 2, algo, seed=6)
    _assert_sig_equal(sig, oracle_hash(L, data, 6, 24, 65535), f"D=20000/{algo}")


def test_index_key_space_limit(wmh):
    """A key space beyond the index build (D = 2^20 columns at bound 255: M =
    2.7e8 cells, E*M > 5.4e8): an explicit index request gets a clean
    WMH_EINVAL, AUTO hashes with another kernel, bit-exact with the oracle."""
    rng = np.random.default_rng(8)
    D = 1 << 20
    rp = np.arange(0, 7 * 3000, 3000, dtype=np.int64)
    col = np.concatenate([np.sort(rng.choice(D, 3000, replace=False)) for _ in range(6)]).astype(np.int32)
    val = rng.integers(1, 256, 6 * 3000).astype(np.uint8)
    data = datagen.CSR(rp, col, val, D)
    cfg = datagen.Config("widekeys", 6, D, 1, 255, 1)
    with pytest.raises(wmh.WmhError, match="key space"):
        _run(wmh, data, cfg, 64, 65535, 2, "index", seed=9, fixed_bound=255)
    sig, L, _ = _run(wmh, data, cfg, 64, 65535, 2, "auto", seed=9, fixed_bound=255)
    assert wmh.last_algo != "index"
    _assert_sig_equal(sig, oracle_hash(L, data, 9, 64, 65535), "wide key space/auto")


@pytest.mark.parametrize("algo", ALGOS)
def test_hash_edge_cases_csr(wmh, algo):
    rng = np.random.default_rng(13)
    D = 5000
    dense = ((rng.random((90, D)) < 0.01) * rng.integers(1, 40, (90, D))).astype(np.uint8)
    dense[0] = 0
    dense[44] = 0
    dense[89] = 0
    rp = np.concatenate([[0], np.cumsum((dense > 0).sum(1))]).astype(np.int64)
    col = np.concatenate([np.nonzero(r)[0] for r in dense]).astype(np.int32)
    val = np.concatenate([r[r > 0] for r in dense]).astype(np.uint8)
    data = datagen.CSR(rp, col, val, D)
    cfg = datagen.Config("edge", 90, D, 1, 255, 1)
    for k, cap, sb in [(50, 2000, 2), (7, 255, 1)]:
        sig, L, _ = _run(wmh, data, cfg, k, cap, sb, algo, seed=5)
        ref = oracle_hash(L, data, 5, k, cap)
        _assert_sig_equal(sig, ref, f"csr edge k={k}/{algo}")
        assert np.all(sig.cpu().numpy()[[0, 44, 89]] == cap)


def test_hash_seeds_and_uniform_layout(wmh):
    """Different master seeds; a uniform-bound layout (division path) and a
    non-uniform one give oracle-identical results."""
    rng = np.random.default_rng(3)
    x = rng.integers(0, 16, size=(500, 256)).astype(np.uint8)
    data = datagen.Dense(x)
    cfg = datagen.Config("u", 500, 256, 1, 255, 1)
    for fb in (15, 200, None):
        for seed in (0, 2**64 - 1, 123456789):
            sig, L, layout = _run(wmh, data, cfg, 48, 65535, 2, "auto", seed=seed, fixed_bound=fb)
            _assert_sig_equal(sig, oracle_hash(L, data, seed, 48, 65535), f"fb={fb} seed={seed}")


def test_saturation_counter(wmh):
    D = 64
    x = np.zeros((4, D), np.uint8)
    x[1, 0] = 1
    layout = wmh.prepare(bounds=torch.full((D,), 200, dtype=torch.uint32).cuda())
    nsat = torch.zeros(1, dtype=torch.int64, device="cuda")
    sig = wmh.hash(layout, wmh.Rows.from_dense(torch.from_numpy(x).cuda()), 1, 100, 50, n_saturated=nsat)
    s = sig.cpu().numpy()
    # rows 0, 2, 3 are empty: 300 saturations; row 1 saturates when no green in 50 draws
    assert int(nsat.item()) >= 300
    assert int(nsat.item()) <= 300 + int((s[1] == 50).sum())


def test_hash_host_e2e_equals_device(wmh):
    cfg, data = datagen.make("c2", n_rows=600)
    rows = to_rows(data)
    layout = wmh.prepare(rows)
    dev = wmh.hash(layout, rows, 1, 100, 65535).cpu()
    host_rows = wmh.Rows.from_dense(torch.from_numpy(data.x).pin_memory())
    host = wmh.hash_host(layout, host_rows, 1, 100, 65535)
    assert torch.equal(dev, host)
    cfg, c = datagen.make("c3", n_rows=50)
    rows = to_rows(c)
    layout = wmh.prepare(rows)
    dev = wmh.hash(layout, rows, 1, 20, 65535).cpu()
    hr = wmh.Rows.from_csr(torch.from_numpy(c.row_ptr), torch.from_numpy(c.col), torch.from_numpy(c.val), c.dim)
    assert torch.equal(dev, wmh.hash_host(layout, hr, 1, 20, 65535))


def test_hash_host_e2e_ramped_chunks(wmh):
    """Batches of >= 30 * 2048 rows go through wmh_hash_host in ramped chunks
    (sizes 1 2 4 ... 4 2 1): every row's signatures equal the device path's,
    dense (tile) and CSR (index built once)."""
    rng = np.random.default_rng(21)
    n, D = 70001, 64
    x = (rng.integers(0, 16, size=(n, D)) * (rng.random((n, D)) < 0.5)).astype(np.uint8)
    rows = wmh.Rows.from_dense(torch.from_numpy(x).cuda())
    layout = wmh.prepare(rows)
    dev = wmh.hash(layout, rows, 5, 24, 65535).cpu()
    host = wmh.hash_host(layout, wmh.Rows.from_dense(torch.from_numpy(x).pin_memory()), 5, 24, 65535)
    assert torch.equal(dev, host)
    cfg, c = datagen.make("c3", n_rows=62000)
    rows = to_rows(c)
    layout = wmh.prepare(rows)
    dev = wmh.hash(layout, rows, 3, 16, 65535).cpu()
    hr = wmh.Rows.from_csr(torch.from_numpy(c.row_ptr).pin_memory(), torch.from_numpy(c.col).pin_memory(),
                           torch.from_numpy(c.val).pin_memory(), c.dim)
    assert torch.equal(dev, wmh.hash_host(layout, hr, 3, 16, 65535))


def test_hash_host_e2e_index_chunks(wmh):
    """wmh_hash_host with CSR rows large enough for AUTO's index kernel: the index
    is built once per call and reused by every row chunk; signatures equal the
    device path and the oracle."""
    cfg, c = datagen.make("c4", n_rows=300)
    rows = to_rows(c)
    bounds = torch.full((c.dim,), 255, dtype=torch.uint32, device="cuda")
    layout = wmh.prepare(rows, bounds=bounds)
    k = 4000
    dev = wmh.hash(layout, rows, 7, k, 65535).cpu()
    assert wmh.last_algo == "index"
    hr = wmh.Rows.from_csr(torch.from_numpy(c.row_ptr).pin_memory(), torch.from_numpy(c.col).pin_memory(),
                           torch.from_numpy(c.val).pin_memory(), c.dim)
    host = wmh.hash_host(layout, hr, 7, k, 65535)
    assert torch.equal(dev, host)
    L = oracle.Layout(np.full(c.dim, 255, np.uint32))
    pick = [0, 1, 150, 299]
    _assert_sig_equal(torch.from_numpy(host.numpy()[pick]), oracle_hash(L, c, 7, k, 65535, rows=pick), "e2e index")


# ------------------------------------------------------------------ collide
def test_sketches_and_layout_digest(wmh):
    """The layout digest is a function of (dim, bounds): equal for two prepares
    of the same rows, different when one bound changes.  collide_sketches over
    two batches equals collide over their concatenation, and refuses a sketch
    of another layout."""
    cfg, data = datagen.make("c2", n_rows=300)
    x = torch.from_numpy(data.x).cuda()
    la, lb = wmh.prepare(wmh.Rows.from_dense(x[:150])), wmh.prepare(wmh.Rows.from_dense(x))
    bounds = la.tables()[2].view(torch.int32).clone()
    l1 = wmh.prepare(bounds=bounds.view(torch.uint32))
    assert l1.digest == la.digest
    b2 = bounds.clone()
    b2[3] += 1
    assert wmh.prepare(bounds=b2.view(torch.uint32)).digest != la.digest
    full = wmh.prepare(bounds=lb.tables()[2].view(torch.int32).clone().view(torch.uint32))
    sa = wmh.sketch(full, wmh.Rows.from_dense(x[:150]), 5, 64, 65535)
    sb = wmh.sketch(full, wmh.Rows.from_dense(x[150:]), 5, 64, 65535)
    ia = torch.arange(0, 150, device="cuda")
    ib = torch.arange(149, -1, -1, device="cuda")
    m1, j1 = wmh.collide_sketches(sa, sb, ia, ib)
    allsig = wmh.hash(full, wmh.Rows.from_dense(x), 5, 64, 65535)
    m2, j2 = wmh.collide(allsig, torch.stack([ia, ib + 150], 1).contiguous())
    assert torch.equal(m1, m2) and torch.equal(j1, j2)
    if la.digest != full.digest:
        with pytest.raises(ValueError, match="layout digest"):
            wmh.collide_sketches(wmh.sketch(la, wmh.Rows.from_dense(x[:150]), 5, 64, 65535), sb, ia, ib)


@pytest.mark.parametrize("sb,k", [(2, 128), (1, 64), (2, 37), (1, 5)])
def test_collide_matches_oracle(wmh, sb, k):
    """a10 (Eq. 14): match counts bit-exact; J-hat = matches/k IEEE-rounded."""
    rng = np.random.default_rng(k)
    n = 300
    hi = 255 if sb == 1 else 65535
    sig = rng.integers(1, 4, size=(n, k)).astype(np.uint32)      # many collisions
    sig[::7] = rng.integers(1, hi, size=sig[::7].shape)
    pairs = np.stack([rng.integers(0, n, 5000), rng.integers(0, n, 5000)], 1).astype(np.int64)
    tdt = torch.uint8 if sb == 1 else torch.uint16
    st = torch.from_numpy(sig.astype(np.uint8 if sb == 1 else np.uint16)).cuda()
    matches, jhat = wmh.collide(st, torch.from_numpy(pairs).cuda())
    ref = oracle.collide(sig, pairs)
    assert np.array_equal(matches.cpu().numpy(), ref)
    assert np.array_equal(jhat.cpu().numpy(), (ref.astype(np.float32) / np.float32(k)))
    assert st.dtype == tdt
    bad = torch.tensor([[0, n]], dtype=torch.int64).cuda()
    with pytest.raises(wmh.WmhError, match="outside"):
        wmh.collide(st, bad)


def test_collide_estimates_jaccard_c5_recipe(wmh):
    """BASELINE north_star: |J-hat - J| within 3 sqrt(J(1-J)/k), read per pair as
    z-scores (reading R16): the count of |z| > 3 near its binomial expectation,
    mean z near 0, var z near 1; match counts bit-exact with the oracle."""
    cfg, data = datagen.make("c5", n_rows=400)
    rows = to_rows(data)
    layout = wmh.prepare(rows)
    k = cfg.k
    sig = wmh.hash(layout, rows, cfg.seed, k, cfg.cap)
    pairs = datagen.random_pairs(7, 400, 3000)
    matches, jhat = wmh.collide(sig, torch.from_numpy(pairs).cuda())
    L = oracle.Layout(oracle.colmax_dense(data.x))
    ref_sig = L.hash_dense(data.x, cfg.seed, k, cfg.cap)
    assert np.array_equal(matches.cpu().numpy(), oracle.collide(ref_sig, pairs))
    J = np.array([float(oracle.jaccard_dense(data.x[a], data.x[b])) for a, b in pairs])
    z = (jhat.cpu().numpy() - J) / np.sqrt(J * (1 - J) / k)
    P = len(pairs)
    # one seed: the pairs share the draw streams, so their errors share a common
    # shift (reading R16) -- check the fraction within 3 sigma and the spread
    assert np.sum(np.abs(z) > 3) <= 0.01 * P + 2
    assert abs(z.mean()) <= 1.0
    assert 0.75 <= z.var() <= 1.25


def test_collide_unbiased_over_seeds(wmh):
    """Eq. 14-15 on the GPU path across independent hash seeds:
    E[J-hat] = J(1 - q) + q ~ J and Var(J-hat) = J(1-J)/k per seed, so the
    mean over 16 seeds of J-hat for each of 10^5 pairs has z-scores
    (mean - J) / sqrt(J(1-J)/(16k)) with mean ~0 and variance ~1.  The pairs
    span J in (0.25, 1): x from the c5 recipe (D = 1024) and y = x with every
    entry replaced, with a per-pair probability, by an independent c5 entry.
    The per-seed common shift of reading R16 (sd ~0.2 in z for one seed)
    averages down to ~0.05 over 16 seeds."""
    n, D, k, S = 100_000, 1024, 1024, 16
    x = datagen.gen_counter_c5_rows(2101, np.arange(n), D)
    alt = datagen.gen_counter_c5_rows(2102, np.arange(n), D)
    q = np.random.default_rng(5).random(n)[:, None]
    repl = np.random.default_rng(6).random((n, D)) < q
    y = np.where(repl, alt, x)
    xy = torch.from_numpy(np.concatenate([x, y])).cuda()
    rows = wmh.Rows.from_dense(xy)
    layout = wmh.prepare(rows)
    pairs = torch.stack([torch.arange(n), torch.arange(n) + n], 1).cuda()
    xa, xb = xy[:n].int(), xy[n:].int()
    J = (torch.minimum(xa, xb).sum(1).double() / torch.maximum(xa, xb).sum(1).double())
    ok = (J > 0) & (J < 1)
    assert float(J[ok].min()) < 0.35 and float(J[ok].max()) > 0.95
    acc = torch.zeros(n, dtype=torch.float64, device="cuda")
    seed_mean_z = []
    for seed in range(S):
        sig = wmh.hash(layout, rows, 1000 + seed, k, 65535)
        _, jhat = wmh.collide(sig, pairs)
        acc += jhat.double()
        zs = ((jhat.double() - J) / torch.sqrt(J * (1 - J) / k))[ok]
        seed_mean_z.append(float(zs.mean()))
    z = ((acc / S - J) / torch.sqrt(J * (1 - J) / (S * k)))[ok]
    P = int(ok.sum().item())
    assert abs(float(z.mean())) <= 0.25, (float(z.mean()), seed_mean_z)
    assert 0.85 <= float(z.var()) <= 1.15, float(z.var())
    assert int((z.abs() > 3).sum().item()) <= 0.01 * P
    sd = float(np.std(seed_mean_z))
    assert sd < 0.5 and abs(float(np.mean(seed_mean_z))) <= 3 * max(sd, 0.05) / math.sqrt(S), seed_mean_z


def test_hasher_streams_batches(wmh):
    """wmh_hasher: the draws filed once, several row batches hashed with the row
    pass only -- identical to wmh_hash on the whole matrix and to the oracle."""
    cfg, data = datagen.make("c3", n_rows=400)
    rows = to_rows(data)
    layout = wmh.prepare(rows)
    whole = wmh.hash(layout, rows, 3, 200, 65535, algo="index").view(torch.int16).cpu()
    hz = wmh.Hasher(layout, 3, 200, 65535)
    parts = [hz.hash(rows.slice(a, b)).view(torch.int16).cpu() for a, b in ((0, 150), (150, 151), (151, 400))]
    assert torch.equal(torch.cat(parts), whole)
    L = oracle.Layout(oracle_bounds(data))
    got = parts[1].numpy().view(np.uint16).astype(np.uint32)
    assert np.array_equal(got, oracle_hash(L, data, 3, 200, 65535, rows=[150]))


@pytest.mark.parametrize("name,n,k", [("c2", 900, 128), ("c3", 300, 100), ("c5", 700, 64)])
def test_sharding_invariance(wmh, name, n, k):
    """SURVEY P10 on the CUDA path: G row shards, each with its local column max
    reduced to the global one (the all-reduce(MAX) of prepare, here an elementwise
    max), hashed separately, give byte-identical signatures for G = 1, 2, 4, 8 --
    every draw depends on (seed, j, t, M) only."""
    cfg, data = datagen.make(name, n_rows=n)
    rows = to_rows(data)
    ref = wmh.hash(wmh.prepare(rows), rows, cfg.seed, k, cfg.cap, cfg.sig_bytes).view(torch.int16).cpu()
    for G in (2, 4, 8):
        shards = [rows.slice(*wmh.shard(n, r, G)) for r in range(G)]
        bounds = torch.stack([wmh.colmax(s).to(torch.int64) for s in shards]).amax(0).to(torch.int32)
        parts = []
        for s in shards:
            layout = wmh.prepare(s, bounds=bounds.view(torch.int32))
            parts.append(wmh.hash(layout, s, cfg.seed, k, cfg.cap, cfg.sig_bytes).view(torch.int16).cpu())
        assert torch.equal(torch.cat(parts), ref), G


def test_check_rows_and_validate_against_oracle(wmh):
    """wmh_check_rows / hash(validate=True): rows a layout did not see
    are checked against its bounds -- the same first offender as the oracle's
    dense and CSR checks, and no error on conforming rows (x_c <= m_c)."""
    rng = np.random.default_rng(9)
    x = rng.integers(0, 6, size=(300, 64)).astype(np.uint8)
    bounds = np.full(64, 5, np.uint32)
    layout = wmh.prepare(bounds=torch.from_numpy(bounds).cuda())
    L = oracle.Layout(bounds)
    rows = to_rows(datagen.Dense(x))
    wmh.check_rows(layout, rows)                          # conforming
    wmh.hash(layout, rows, 1, 16, 100, validate=True)
    x2 = x.copy()
    x2[123, 7] = 6
    x2[200, 1] = 9
    assert L.check_bounds_dense(x2) == (123, 7)
    with pytest.raises(wmh.WmhError, match=r"x\[123\]\[7\]"):
        wmh.check_rows(layout, to_rows(datagen.Dense(x2)))
    with pytest.raises(wmh.WmhError, match="exceeds its bound"):
        wmh.hash(layout, to_rows(datagen.Dense(x2)), 1, 16, 100, validate=True)
    # CSR
    rp = np.zeros(301, np.int64)
    cols, vals = [], []
    for n in range(300):
        c = np.flatnonzero(x2[n])
        cols.append(c.astype(np.int32))
        vals.append(x2[n, c])
        rp[n + 1] = rp[n] + len(c)
    csr = datagen.CSR(rp, np.concatenate(cols), np.concatenate(vals).astype(np.uint8), 64)
    want = L.check_bounds_csr(csr.row_ptr, csr.col, csr.val)
    assert want is not None and want[1] == 3
    with pytest.raises(wmh.WmhError, match=f"nonzero {want[0]}: value exceeds its bound"):
        wmh.check_rows(layout, to_rows(csr))



@pytest.mark.parametrize("D,offset", [(1032, 0), (4096, 8)])
def test_bitslice_rows_without_bulk_prefetch(wmh, D, offset):
    """The bit-sliced tile warms L2 with the next tile's rows by TMA bulk prefetches
    only when the rows are 16-byte aligned (D % 16 == 0 and an aligned base);
    D = 1032 and a view 8 bytes into its allocation take the per-line prefetch
    loop.  Prefetching changes no result: bit-exact with the oracle either way."""
    rng = np.random.default_rng(7000 + D + offset)
    n = 200
    x = np.minimum(rng.geometric(0.3, size=(n, D)), 40).astype(np.uint8)
    x[rng.random((n, D)) < 0.5] = 0
    flat = np.zeros(n * D + offset, np.uint8)
    flat[offset:] = x.reshape(-1)
    xt = torch.from_numpy(flat).cuda()[offset:].view(n, D)
    assert xt.data_ptr() % 16 == offset % 16
    rows = wmh.Rows.from_dense(xt)
    layout = wmh.prepare(rows)
    L = oracle.Layout(oracle.colmax_dense(x))
    assert layout.M == L.M
    sig = wmh.hash(layout, rows, 29, 96, 65535, 2, algo="tiled", tile="bitslice")
    _assert_sig_equal(sig, L.hash_dense(x, 29, 96, 65535), f"bitslice D={D} offset={offset}")
