"""f1 pins (CPU): the uint16 / fixed-point oracle against what the paper fixes.

* Scale invariance, exact: hashing integer data x with bounds m gives the same
  signatures as hashing x * 2^f with bounds m * 2^f (r' = floor(z M 2^f / 2^64)
  has r' >> f = r, and r' - 2^f lo < 2^f x  <=>  r - lo < x).  P:324: "If all
  the values are integers, scaling up does not matter".  This ties the uint16
  code to the already-pinned uint8 oracle.
* Theorem 2 and the collision law (Theorem 1, Eq. 14-15) on wide
  layouts (bounds > 255).
* Sec. 4's scale choice on SPEC's worked example."""
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle


def _csr(x):
    rp = np.concatenate([[0], np.cumsum((x > 0).sum(1))]).astype(np.int64)
    col = np.concatenate([np.nonzero(r)[0] for r in x]).astype(np.int32)
    val = np.concatenate([r[r > 0] for r in x])
    return rp, col, val


@pytest.mark.parametrize("f", [1, 4, 8])
def test_scale_invariance_dense_and_csr(f):
    rng = np.random.default_rng(f)
    x = (rng.random((25, 40)) < 0.4) * rng.integers(1, 30, (25, 40))
    x = x.astype(np.uint8)
    x[3] = 0
    m = oracle.colmax_dense(x)
    m[m == 0] = 1                       # keep every column drawable
    ref = oracle.Layout(m).hash_dense(x, 11, 24, 500)
    Lw = oracle.Layout(m.astype(np.uint32) << f)
    xw = x.astype(np.uint16) << f
    assert np.array_equal(Lw.hash_dense(xw, 11, 24, 500), ref)
    rp, col, val = _csr(xw)
    assert np.array_equal(Lw.hash_csr(rp, col, val, 11, 24, 500), ref)
    assert np.array_equal(oracle.colmax_dense(xw), oracle.colmax_csr(rp, col, val, 40))


def test_geometric_law_wide_layout():
    """Theorem 2: h ~ Geom(s) capped, s = |x|_1 / M, on a layout with bounds > 255."""
    m = np.array([700, 300, 1000, 45], np.uint32)
    x = np.array([[350, 0, 123, 45]], np.uint16)
    L = oracle.Layout(m)
    s = Fraction(int(x.sum()), int(m.sum()))
    k, cap = 20000, 400
    h = L.hash_dense(x, 3, k, cap)[0].astype(np.float64)
    sf = float(s)
    mean = (1 - (1 - sf) ** cap) / sf
    var = (1 - sf) / sf ** 2                            # (cap effect < 1e-20 here)
    assert abs(h.mean() - mean) <= 4 * math.sqrt(var / k)
    assert abs(h.var() / var - 1) <= 0.1


def test_collision_law_wide_layout():
    """Theorem 1 / Eq. 14: P(h_x = h_y) = J = sum min / sum max (no saturation)."""
    m = np.array([1000, 600, 300], np.uint32)
    L = oracle.Layout(m)
    x = np.array([[900, 100, 0]], np.uint16)
    y = np.array([[400, 550, 200]], np.uint16)
    J = (400 + 100 + 0) / (900 + 550 + 200)
    k = 20000
    hx = L.hash_dense(x, 9, k, 65535)[0]
    hy = L.hash_dense(y, 9, k, 65535)[0]
    jhat = float((hx == hy).mean())
    assert abs(jhat - J) <= 4 * math.sqrt(J * (1 - J) / k)


def test_quantize_definition():
    x = np.array([0.0, 0.49, 0.5, 1.0, 2.75, 1e9, 3.999], np.float32)
    q = oracle.quantize(x, 4.0)
    assert q.dtype == np.uint16
    assert q.tolist() == [0, 1, 2, 4, 11, 65535, 15]
    dy = np.array([3 / 8, 5 / 8, 255 / 8], np.float32)       # dyadic weights are exact
    assert oracle.quantize(dy, 8).tolist() == [3, 5, 255]
    with pytest.raises(ValueError):
        oracle.quantize(np.array([-1.0], np.float32), 2)


def test_choose_scale_spec_examples():
    """maxima=[0.5], x=(0.5), grid {1,2} -> 2; a singleton grid returns
    its only candidate; integer data: scaling up does not change s, so the
    tie goes to the smaller scale."""
    assert oracle.choose_scale(np.array([[0.5]], np.float32), [1, 2]) == 2.0
    assert oracle.choose_scale(np.array([[0.5, 1.0]], np.float32), [3.0]) == 3.0
    xi = np.array([[1, 4, 0], [2, 2, 3]], np.float32)
    o = oracle.scale_objective(xi, [1, 2, 4])
    assert Fraction(*o[0][:2]) == Fraction(*o[1][:2]) == Fraction(*o[2][:2])
    assert oracle.choose_scale(xi, [4, 2, 1]) == 1.0
    # a scale that would saturate a uint16 weight is not a candidate
    big = np.array([[300.0, 1.0]], np.float32)
    assert oracle.scale_objective(big, [256.0])[0][2] == 1
    assert oracle.choose_scale(big, [1.0, 256.0]) == 1.0
