"""Pins for the CPU oracle (oracle/) against what the paper and mathematics fix.

Each test names the passage it pins (P:n = PAPER.md line, with section /
equation / algorithm; S:n = SPEC.md line).  None of these re-types the
oracle's formula and compares it with itself: they use closed forms (Theorem
1 with the cap, Theorem 2), brute-force enumeration of every draw sequence,
worked examples and published known answers, invariants and special cases.
"""
import itertools
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _read(name):
    rows = []
    with open(os.path.join(GOLD, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(line)
    return rows


# ------------------------------------------------------------------ RNG pins
def test_splitmix64_published_known_answer():
    """Reading R6: the mixer is the standard SplitMix64 output function."""
    for line in _read("splitmix64_known.txt"):
        v, want = line.split()
        assert oracle.splitmix64(int(v, 0)) == int(want, 16)


def test_draws_match_independent_survey_values():
    """Readings R6-R8 (key = splitmix64(seed) ^ (j<<32) ^ t; 64x32 multiply-high)."""
    for line in _read("survey_rng_draws.txt"):
        seed, j, t, M, r = map(int, line.split())
        assert oracle.draw(seed, j, t, M) == r


def test_draw_range_and_uniformity_ks():
    """P:170 (Alg. 3): r is uniform on [0, M).  KS test at alpha = 0.001."""
    M = 261120
    r = np.array([oracle.draw(1, j, t, M) for j in range(200) for t in range(500)], dtype=np.float64)
    assert r.min() >= 0 and r.max() < M
    u = np.sort((r + 0.5) / M)
    n = len(u)
    ecdf_hi = np.arange(1, n + 1) / n
    ecdf_lo = np.arange(0, n) / n
    D = max(np.max(ecdf_hi - u), np.max(u - ecdf_lo))
    assert D < 1.95 / math.sqrt(n)          # KS critical value at alpha = 0.001


def test_hash_streams_independent():
    """Reading R7: hashes j and j^1, and master seeds 1 and 2, must be independent
    (the literal seed^j^t aliases them; P:235's Var(J-hat) = J(1-J)/k needs
    independence).  |rho| <= 4/sqrt(n)."""
    m = np.full(16, 10, np.uint32)
    L = oracle.Layout(m)
    rng = np.random.default_rng(7)
    x = rng.integers(0, 11, 16).astype(np.uint8)
    y = np.minimum(10, x + rng.integers(0, 4, 16)).astype(np.uint8)
    k = 8192
    sx = L.hash_dense(x, 1, k, 65535)[0]
    sy = L.hash_dense(y, 1, k, 65535)[0]
    coll = (sx == sy).astype(np.float64)
    a, b = coll[0::2], coll[1::2]
    rho = np.corrcoef(a, b)[0, 1]
    assert abs(rho) <= 4 / math.sqrt(len(a))
    s2 = L.hash_dense(x, 2, k, 65535)[0]
    rho2 = np.corrcoef(sx.astype(float), s2.astype(float))[0, 1]
    assert abs(rho2) <= 4 / math.sqrt(k)


# --------------------------------------------------------------- layout pins
def test_layout_spec_examples():
    """Alg. 4; SPEC examples S:193-194 (maxima [2,2] and [1])."""
    L = oracle.Layout([2, 2])
    assert L.M == 4 and list(L.comp_to_m) == [0, 2, 4] and list(L.int_to_comp) == [0, 0, 1, 1]
    L = oracle.Layout([1])
    assert L.M == 1 and list(L.int_to_comp) == [0]


def test_layout_worked_example_and_zero_width():
    """Alg. 4 with a zero bound (reading R11: zero-width interval, no cells)."""
    L = oracle.Layout([2, 3, 1, 4])
    assert list(L.comp_to_m) == [0, 2, 5, 6, 10]
    assert list(L.int_to_comp) == [0, 0, 1, 1, 1, 2, 3, 3, 3, 3]
    L = oracle.Layout([3, 0, 2])
    assert list(L.comp_to_m) == [0, 3, 3, 5] and list(L.int_to_comp) == [0, 0, 0, 2, 2]


def test_layout_invariants_random():
    """Eq. 3: CompToM is the exclusive prefix sum, every cell t lies in
    [CompToM[c], CompToM[c] + m_c) of c = IntToComp[t] (S:171-176 invariant)."""
    rng = np.random.default_rng(3)
    for _ in range(20):
        m = rng.integers(0, 9, rng.integers(1, 40)).astype(np.uint32)
        if m.sum() == 0:
            m[0] = 1
        L = oracle.Layout(m)
        assert L.M == int(m.sum())
        assert np.array_equal(L.comp_to_m[1:] - L.comp_to_m[:-1], m)
        t = np.arange(L.M)
        c = L.int_to_comp
        assert np.all(L.comp_to_m[c] <= t) and np.all(t < L.comp_to_m[c] + m[c])


def test_layout_errors():
    with pytest.raises(ValueError):
        oracle.Layout([0, 0, 0])
    with pytest.raises(ValueError):
        oracle.Layout(np.array([2**31, 2**31], dtype=np.uint64).astype(np.uint32))


# ------------------------------------------------------------ ISGREEN pins
def test_isgreen_three_ways_agree():
    """Alg. 5 O(1) lookup == Sec. 3.3 binary search over the row's d
    intervals == Eq. 4 membership read directly, for every
    cell of random layouts and rows."""
    rng = np.random.default_rng(11)
    for _ in range(40):
        D = int(rng.integers(1, 30))
        m = rng.integers(0, 7, D).astype(np.uint32)
        if m.sum() == 0:
            m[0] = 3
        L = oracle.Layout(m)
        x = (rng.random(D) * (m + 1)).astype(np.uint8)
        x = np.minimum(x, m).astype(np.uint8)
        cols = np.nonzero(x)[0].astype(np.int32)
        for r in range(L.M):
            a = L.is_green_o1(x, r)
            b = L.is_green_binsearch(cols, x[cols], r)
            c = L.is_green_direct(x, r)
            assert a == b == c
        # exactly sum(x) green cells (strict boundary, reading R2)
        assert sum(L.is_green_o1(x, r) for r in range(L.M)) == int(x.sum())


def test_isgreen_boundaries():
    """Reading R2 (strict '<'): x_c green cells at the start of interval c."""
    L = oracle.Layout([2, 3])
    x = np.array([1, 2], np.uint8)
    assert [L.is_green_o1(x, r) for r in range(5)] == [True, False, True, True, False]
    x0 = np.zeros(2, np.uint8)
    assert not any(L.is_green_o1(x0, r) for r in range(5))   # zero weight: all red


# ------------------------------------------------------------- brute force
def _brute(m, x, y, cap):
    """Enumerate all M^cap draw sequences; return exact P(h_x = h_y), E[h_x]."""
    L = oracle.Layout(m)
    M = L.M
    coll = 0
    hsum = 0
    for seq in itertools.product(range(M), repeat=cap):
        hx = L.hash_from_draws(x, list(seq), cap)
        hy = L.hash_from_draws(y, list(seq), cap)
        coll += hx == hy
        hsum += hx
    tot = M ** cap
    return Fraction(coll, tot), Fraction(hsum, tot), L


@pytest.mark.parametrize("m,x,y,cap", [
    ([2, 3], [1, 2], [2, 1], 5),
    ([1, 2, 2], [1, 0, 2], [0, 2, 1], 5),
    ([3, 2], [2, 0], [0, 1], 6),
    ([2, 2, 1], [2, 1, 0], [1, 1, 1], 4),
])
def test_theorem1_and_theorem2_by_brute_force(m, x, y, cap):
    """Theorem 1 with the cap (reading R9): over every draw sequence,
    P(h_x = h_y) = J (1 - q) + q with q = (1 - sum max / M)^(cap-1), and
    J = sum min / sum max (Eq. 1).  Theorem 2 capped:
    E[h] = sum_{t<cap} (1-s)^t = (1 - (1-s)^cap) / s with s = |x|_1 / M (Eq. 17)."""
    x = np.array(x, np.uint8)
    y = np.array(y, np.uint8)
    P, Eh, L = _brute(m, x, y, cap)
    M = L.M
    smin = int(np.minimum(x, y).sum())
    smax = int(np.maximum(x, y).sum())
    J = Fraction(smin, smax)
    q = (1 - Fraction(smax, M)) ** (cap - 1)
    assert P == J * (1 - q) + q
    s = Fraction(int(x.sum()), M)
    assert Eh == (1 - (1 - s) ** cap) / s
    # proof events: |G_x & G_y| = sum min, |G_x | G_y| = sum max
    gx = [L.is_green_o1(x, r) for r in range(M)]
    gy = [L.is_green_o1(y, r) for r in range(M)]
    assert sum(a and b for a, b in zip(gx, gy)) == smin
    assert sum(a or b for a, b in zip(gx, gy)) == smax
    assert oracle.jaccard_dense(x, y) == J


# ----------------------------------------------------------- worked example
def test_survey_worked_example_hashes():
    """Independent implementation's hashes of a 4-dim example."""
    L = oracle.Layout([2, 3, 1, 4])
    sigs = {}
    for line in _read("survey_hashes.txt"):
        name, xs, seed, cap, hs = [p.strip() for p in line.split("|")]
        x = np.array(list(map(int, xs.split())), np.uint8)
        h = L.hash_dense(x, int(seed), 16, int(cap))[0]
        assert list(h) == list(map(int, hs.split())), name
        sigs[name] = h
    assert int((sigs["x"] == sigs["y"]).sum()) == 3
    assert oracle.jaccard_dense([1, 0, 1, 3], [2, 3, 0, 1]) == Fraction(2, 9)


# --------------------------------------------------------------- laws, real RNG
@pytest.mark.parametrize("s_num", [20, 81, 300])
def test_theorem2_geometric_law(s_num):
    """Theorem 2: with s in {0.02, 0.081, 0.3} (0.081 is
    Table 1's Web-Images value), 10^5 hashes: mean within 3 SE of 1/s,
    variance within 10% of (1-s)/s^2, and the Eq. 16 tail P(h > n_delta) <= delta
    (reading R10: '>' not '>=') up to 4 binomial SE."""
    D = 10
    M = 1000
    m = np.full(D, M // D, np.uint32)
    L = oracle.Layout(m)
    x = np.zeros(D, np.uint8)
    rem = s_num
    for c in range(D):                       # spread sum(x) = s_num over the columns
        take = min(100, rem)
        x[c] = take
        rem -= take
    s = s_num / M
    k = 100_000
    h = L.hash_dense(x, 12345, k, 65535)[0].astype(np.float64)
    mean, var = h.mean(), h.var()
    assert abs(mean - 1 / s) <= 3 * math.sqrt((1 - s) / s**2 / k)
    assert abs(var / ((1 - s) / s**2) - 1) <= 0.10
    for delta in (0.1, 0.01):
        n = math.ceil(math.log(delta) / math.log(1 - s))
        p = float(np.mean(h > n))
        assert p <= delta + 4 * math.sqrt(delta * (1 - delta) / k)
    # Corollary: E[log2 h] <= log2 E[h] = log2(1/s) (Jensen)
    assert np.mean(np.log2(h)) <= math.log2(1 / s) + 0.01


def test_theorem1_collision_law_nine_pairs():
    """Theorem 1 / Eq. 14-15: nine pairs with J in {0.1..0.9},
    k = 10^4: |J-hat - J| <= 3 sqrt(J(1-J)/k) (cap 65535 makes q negligible)."""
    D = 20
    m = np.full(D, 50, np.uint32)
    L = oracle.Layout(m)
    rng = np.random.default_rng(5)
    k = 10_000
    for target in [i / 10 for i in range(1, 10)]:
        # x = full 50s on the first 10 columns; y overlaps x by a fraction
        x = np.zeros(D, np.uint8)
        y = np.zeros(D, np.uint8)
        x[:10] = 50
        # J = min/max: choose y = x on a columns-prefix scaled to hit target
        # y[c] = 50 for c < a, then a partial column; J = |y| / |x| when y <= x
        tot = int(round(target * 500))
        full, part = divmod(tot, 50)
        y[:full] = 50
        if part:
            y[full] = part
        J = oracle.jaccard_dense(x, y)
        sig = L.hash_dense(np.stack([x, y]), int(rng.integers(1, 2**63)), k, 65535)
        jhat = float(np.mean(sig[0] == sig[1]))
        Jf = float(J)
        assert abs(jhat - Jf) <= 3 * math.sqrt(Jf * (1 - Jf) / k) + 1e-12, (target, jhat, Jf)


def test_estimator_unbiased_and_variance_over_seeds():
    """Eq. 14-15: over 200 master seeds with k = 50, the mean
    of J-hat is within 3 sqrt(J(1-J)/(200*50)) of J and Var(J-hat) is within 25%
    of J(1-J)/50."""
    m = np.array([4, 4, 4, 4, 4, 4], np.uint32)
    L = oracle.Layout(m)
    x = np.array([4, 3, 0, 2, 1, 0], np.uint8)
    y = np.array([2, 3, 1, 0, 1, 4], np.uint8)
    J = float(oracle.jaccard_dense(x, y))
    est = []
    for seed in range(1, 201):
        sig = L.hash_dense(np.stack([x, y]), seed, 50, 65535)
        est.append(np.mean(sig[0] == sig[1]))
    est = np.array(est)
    assert abs(est.mean() - J) <= 3 * math.sqrt(J * (1 - J) / (200 * 50))
    assert abs(est.var(ddof=1) / (J * (1 - J) / 50) - 1) <= 0.25


# ------------------------------------------------------------- special cases
def test_special_cases():
    """Proof events and S:223/S:235/S:379-381:
    identical rows always collide; disjoint supports collide only when both
    saturate; x = m gives h = 1; x <= y coordinatewise gives h(x) >= h(y)
    (G_x subset of G_y); an empty row saturates (reading R12)."""
    rng = np.random.default_rng(9)
    m = rng.integers(1, 20, 64).astype(np.uint32)
    L = oracle.Layout(m)
    k = 512
    x = np.minimum(m, rng.integers(0, 20, 64)).astype(np.uint8)
    x[::3] = 0
    y = x.copy()
    sig = L.hash_dense(np.stack([x, y]), 77, k, 65535)
    assert np.all(sig[0] == sig[1])
    # disjoint supports
    a = np.zeros(64, np.uint8)
    b = np.zeros(64, np.uint8)
    a[:32] = m[:32]
    b[32:40] = 1
    cap = 40
    sig = L.hash_dense(np.stack([a, b]), 78, k, cap)
    eq = sig[0] == sig[1]
    assert np.all(sig[0][eq] == cap) and np.all(sig[1][eq] == cap)
    # full green
    sig = L.hash_dense(m.astype(np.uint8), 79, k, 65535)
    assert np.all(sig == 1)
    # monotone: x <= y  =>  h(x) >= h(y)
    lo = (x // 2).astype(np.uint8)
    sig = L.hash_dense(np.stack([lo, x]), 80, k, 65535)
    assert np.all(sig[0] >= sig[1])
    # empty -> cap
    sig = L.hash_dense(np.zeros(64, np.uint8), 81, k, 300)
    assert np.all(sig == 300)
    # saturation never exceeds cap and h >= 1
    sig = L.hash_dense(np.stack([lo, x]), 82, k, 7)
    assert sig.min() >= 1 and sig.max() <= 7


def test_single_nonzero_is_geometric():
    """Theorem 2: a single nonzero x_c gives Geom(x_c / M)."""
    m = np.array([10, 20, 30], np.uint32)
    L = oracle.Layout(m)
    x = np.array([0, 6, 0], np.uint8)
    s = 6 / 60
    h = L.hash_dense(x, 5, 50_000, 65535)[0]
    assert abs(h.mean() - 1 / s) <= 3 * math.sqrt((1 - s) / s**2 / 50_000)


def test_sequence_sharing():
    """P:190-191 ('consistency ... the sequence of random numbers is the same')
    and S:146: the draw stream is independent of x; hashing through the
    explicit stream reproduces the counter-based hash for any row."""
    m = np.array([3, 5, 2, 6], np.uint32)
    L = oracle.Layout(m)
    for x in ([1, 0, 2, 3], [3, 5, 0, 0], [0, 1, 0, 0]):
        x = np.array(x, np.uint8)
        for j in range(8):
            draws = [oracle.draw(4, j, t, L.M) for t in range(200)]
            assert L.hash_from_draws(x, draws, 200) == L.hash_one(x, 4, j, 200)


# ----------------------------------------------------------- estimation pins
def test_jaccard_examples():
    """Eq. 1."""
    assert oracle.jaccard_dense([1, 2], [2, 1]) == Fraction(1, 2)
    assert oracle.jaccard_dense([3, 0, 4], [3, 0, 4]) == 1
    assert oracle.jaccard_dense([3, 0, 0], [0, 0, 4]) == 0
    assert oracle.jaccard_dense([0, 0], [0, 0]) is None
    # binary special case: |x & y| / |x | y|
    a = np.array([1, 1, 0, 1, 0], np.uint8)
    b = np.array([0, 1, 1, 1, 0], np.uint8)
    assert oracle.jaccard_dense(a, b) == Fraction(2, 4)


def test_jaccard_csr_matches_dense():
    rng = np.random.default_rng(2)
    dense = (rng.random((6, 40)) < 0.3) * rng.integers(1, 9, (6, 40))
    dense = dense.astype(np.uint8)
    rp = np.concatenate([[0], np.cumsum((dense > 0).sum(1))]).astype(np.int64)
    col = np.concatenate([np.nonzero(r)[0] for r in dense]).astype(np.int32)
    val = np.concatenate([r[r > 0] for r in dense]).astype(np.uint8)
    for a in range(6):
        for b in range(6):
            assert oracle.jaccard_csr(rp, col, val, a, b) == oracle.jaccard_dense(dense[a], dense[b])


def test_collide_counts():
    sig = np.array([[1, 2, 3, 4], [1, 0, 3, 0], [9, 9, 9, 9]], np.uint32)
    pairs = np.array([[0, 1], [0, 2], [1, 1]], np.int64)
    assert list(oracle.collide(sig, pairs)) == [2, 0, 4]


def test_csr_hash_equals_dense_hash():
    """The CSR front end scatters to a dense row; hashes must equal the dense path."""
    rng = np.random.default_rng(4)
    dense = ((rng.random((12, 300)) < 0.1) * rng.integers(1, 30, (12, 300))).astype(np.uint8)
    dense[3] = 0
    m = oracle.colmax_dense(dense)
    m[m == 0] = 1
    L = oracle.Layout(m)
    rp = np.concatenate([[0], np.cumsum((dense > 0).sum(1))]).astype(np.int64)
    col = np.concatenate([np.nonzero(r)[0] for r in dense]).astype(np.int32)
    val = np.concatenate([r[r > 0] for r in dense]).astype(np.uint8)
    assert np.array_equal(oracle.colmax_csr(rp, col, val, 300)[dense.max(0) > 0], dense.max(0)[dense.max(0) > 0])
    a = L.hash_dense(dense, 3, 40, 1000)
    b = L.hash_csr(rp, col, val, 3, 40, 1000)
    assert np.array_equal(a, b)
    assert np.all(a[3] == 1000)


def test_colmax_and_bounds():
    x = np.array([[1, 5, 0], [3, 2, 0]], np.uint8)
    assert list(oracle.colmax_dense(x)) == [3, 5, 0]
    L = oracle.Layout([3, 4, 1])
    assert L.check_bounds_dense(x) == (0, 1)
    L = oracle.Layout([3, 5, 1])
    assert L.check_bounds_dense(x) is None


def test_csr_bounds_and_structure():
    """The CSR twin of the bounds check (hand examples): x = [[1, 5, 0], [3, 2, 0]]
    as CSR against bounds [3, 4, 1] fails at nonzero 1 (value 5 in column 1)."""
    rp = np.array([0, 2, 4], np.int64)
    col = np.array([0, 1, 0, 1], np.int32)
    val = np.array([1, 5, 3, 2], np.uint8)
    assert oracle.Layout([3, 4, 1]).check_bounds_csr(rp, col, val) == (1, 3)
    L = oracle.Layout([3, 5, 1])
    assert L.check_bounds_csr(rp, col, val) is None
    assert L.check_bounds_csr(rp, np.array([0, 1, 1, 0], np.int32), val) == (3, 2)        # not ascending
    assert L.check_bounds_csr(rp, np.array([0, 3, 0, 1], np.int32), val) == (1, 1)        # column >= dim
    assert L.check_bounds_csr(np.array([0, 5, 4], np.int64), col, val) == (0, 4)          # row_ptr past nnz
    assert L.check_bounds_csr(np.array([0, 2, 4, 4], np.int64), col, val) is None          # an empty last row
