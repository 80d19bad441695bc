"""f1 GPU parity: uint16 weights / wide layouts (bounds > 255) through the C ABI,
the fixed-point quantiser and Sec. 4's scale objective, against the oracle."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def wmh():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1602_08393_b200 as w
    from paper_1602_08393_b200 import build
    build.build()
    return w


def _csr(x):
    rp = np.concatenate([[0], np.cumsum((x > 0).sum(1))]).astype(np.int64)
    col = np.concatenate([np.nonzero(r)[0] for r in x]).astype(np.int32)
    val = np.concatenate([r[r > 0] for r in x]).astype(x.dtype)
    return rp, col, val


def _rows16(wmh, x, csr):
    if not csr:
        return wmh.Rows.from_dense(torch.from_numpy(x.astype(np.int32)).to(torch.uint16).cuda())
    rp, col, val = _csr(x)
    return wmh.Rows.from_csr(torch.from_numpy(rp).cuda(), torch.from_numpy(col).cuda(),
                             torch.from_numpy(val.astype(np.int32)).to(torch.uint16).cuda(), x.shape[1])


def _sig(s):
    return s.cpu().to(torch.int32).numpy().astype(np.uint32) if s.dtype == torch.uint8 else \
        s.view(torch.int16).cpu().numpy().view(np.uint16).astype(np.uint32)


def _random16(seed, n, d, hi, p=0.3):
    rng = np.random.default_rng(seed)
    x = ((rng.random((n, d)) < p) * rng.integers(1, hi, (n, d))).astype(np.uint16)
    x[1] = 0                                  # an empty row (reading R12)
    return x


@pytest.mark.parametrize("algo", ["index", "simple", "auto"])
@pytest.mark.parametrize("csr", [False, True])
@pytest.mark.parametrize("hi,k", [(4000, 300), (300, 64), (60000, 40)])
def test_u16_weights_match_oracle(wmh, algo, csr, hi, k):
    x = _random16(hi + k, 90, 77 if not csr else 3000, hi)
    rows = _rows16(wmh, x, csr)
    layout = wmh.prepare(rows)
    m = oracle.colmax_dense(x)
    assert np.array_equal(wmh.colmax(rows).cpu().numpy(), m)
    L = oracle.Layout(m)
    assert layout.M == L.M and bool(layout.flags & 2) == (m.max() > 255)
    c2m, i2c, _ = layout.tables()
    assert np.array_equal(i2c.cpu().numpy(), L.int_to_comp)
    sig = wmh.hash(layout, rows, 21, k, 65535, 2, algo=algo)
    ref = L.hash_dense(x, 21, k, 65535)
    assert np.array_equal(_sig(sig), ref)


def test_u16_index_horizons_and_uint8_sigs(wmh):
    x = _random16(5, 60, 200, 2000, p=0.5)
    rows = _rows16(wmh, x, False)
    layout = wmh.prepare(rows)
    L = oracle.Layout(oracle.colmax_dense(x))
    for T in (1, 40, 0):
        sig = wmh.hash(layout, rows, 3, 50, 255, 1, algo="index", horizon=T)
        assert np.array_equal(_sig(sig), L.hash_dense(x, 3, 50, 255)), T


def test_scale_invariance_across_kernels(wmh):
    """uint8 data on the tile == the same data x 2^f as uint16 on the index kernel
    (exact scale invariance, tests/test_oracle_real.py)."""
    rng = np.random.default_rng(8)
    x8 = ((rng.random((400, 256)) < 0.6) * rng.integers(1, 200, (400, 256))).astype(np.uint8)
    r8 = wmh.Rows.from_dense(torch.from_numpy(x8).cuda())
    l8 = wmh.prepare(r8)
    s8 = wmh.hash(l8, r8, 4, 128, 65535, algo="tiled")
    for f in (2, 8):
        x16 = x8.astype(np.uint16) << f
        r16 = _rows16(wmh, x16, False)
        l16 = wmh.prepare(r16)
        assert l16.M == l8.M << f
        for algo in ("index", "simple", "auto"):
            s16 = wmh.hash(l16, r16, 4, 128, 65535, algo=algo)
            assert torch.equal(s8, s16), (f, algo)


def test_tiled_rejects_wide(wmh):
    x = _random16(1, 10, 32, 1000)
    rows = _rows16(wmh, x, False)
    layout = wmh.prepare(rows)
    with pytest.raises(wmh.WmhError, match="does not take"):
        wmh.hash(layout, rows, 1, 8, 100, algo="tiled")
    with pytest.raises(wmh.WmhError, match="EINVAL"):
        wmh.prepare(bounds=torch.full((4,), 70000, dtype=torch.uint32).cuda())


def test_quantize_matches_oracle(wmh):
    rng = np.random.default_rng(2)
    x = (rng.gamma(0.5, 1.0, 200000) * rng.choice([0, 1], 200000, p=[0.6, 0.4])).astype(np.float32)
    x[:5] = [0.0, 1e9, 3.999, 2.75, 0.125]
    for scale in (1.0, 64.0, 1000.0, 0.37, 4096.0):
        q = wmh.quantize(torch.from_numpy(x).cuda(), scale)
        assert np.array_equal(q.to(torch.int32).cpu().numpy(), oracle.quantize(x, scale).astype(np.int32)), scale
    with pytest.raises(wmh.WmhError, match="negative or NaN"):
        wmh.quantize(torch.tensor([1.0, -2.0], device="cuda"), 2.0)
    with pytest.raises(wmh.WmhError, match="scale"):
        wmh.quantize(torch.tensor([1.0], device="cuda"), 0.0)


def test_scale_objective_and_choice(wmh):
    rng = np.random.default_rng(4)
    x = (rng.gamma(0.5, 1.0, (300, 64)) * (rng.random((300, 64)) < 0.4)).astype(np.float32)
    scales = [1.0, 3.0, 10.0, 64.0, 256.0]
    rows = wmh.Rows.from_dense(torch.from_numpy(x).cuda())
    assert wmh.scale_objective(rows, scales) == oracle.scale_objective(x, scales)
    assert wmh.choose_scale(rows, scales) == oracle.choose_scale(x, scales)
    rp, col, val = _csr(x)
    crow = wmh.Rows.from_csr(torch.from_numpy(rp).cuda(), torch.from_numpy(col).cuda(), torch.from_numpy(val).cuda(), 64)
    assert wmh.scale_objective(crow, scales) == oracle.scale_objective(x, scales)
    one = wmh.Rows.from_dense(torch.tensor([[0.5]], device="cuda"))
    assert wmh.choose_scale(one, [1.0, 2.0]) == 2.0               # S:237-245 worked example


def test_real_valued_pipeline(wmh):
    """Real histograms (c2's Gamma recipe before rounding) -> quantize at the chosen
    scale -> prepare -> hash == the oracle on the same quantised weights."""
    rng = np.random.default_rng(6)
    g = (rng.gamma(0.5, 1.0, (500, 1024)) * (rng.random((500, 1024)) < 0.4)).astype(np.float32)
    xr = torch.from_numpy(g).cuda()
    scale = wmh.choose_scale(wmh.Rows.from_dense(xr), [16.0, 64.0, 256.0, 1024.0])
    q = wmh.quantize(xr, scale)
    rows = wmh.Rows.from_dense(q)
    layout = wmh.prepare(rows)
    sig = wmh.hash(layout, rows, 1, 256, 65535)
    qn = oracle.quantize(g, scale)
    L = oracle.Layout(oracle.colmax_dense(qn))
    assert np.array_equal(_sig(sig), L.hash_dense(qn, 1, 256, 65535))
    host = wmh.hash_host(layout, wmh.Rows.from_dense(q.cpu().pin_memory()), 1, 256, 65535)
    assert torch.equal(host, sig.cpu())
