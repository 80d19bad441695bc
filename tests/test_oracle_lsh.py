"""f3 pins (CPU): the banding LSH oracle against the S-curve of (K, L) LSH
-- a pair whose hashes collide with probability J (Theorem 1) is a candidate with
probability 1 - (1 - J^K)^L -- and its special cases."""
import math

import numpy as np

import datagen
import oracle


def test_lsh_s_curve_on_fig2_pairs():
    x, y, J = datagen.fig2_pairs()
    rows = np.concatenate([x, y])
    L_ = oracle.Layout(oracle.colmax_dense(rows))
    K, L, R = 3, 4, 300
    hit = np.zeros(9)
    for seed in range(1, R + 1):
        s = L_.hash_dense(rows, seed, K * L, 65535)
        cands = oracle.lsh_candidates(s[9:], K, L, s[:9])           # index the y's, query with the x's
        hit += [p in c for p, c in enumerate(cands)]
    for p, Jp in enumerate(J):
        P = 1 - (1 - Jp ** K) ** L
        assert abs(hit[p] / R - P) <= 4 * math.sqrt(P * (1 - P) / R) + 1e-9, (Jp, hit[p] / R, P)


def test_lsh_special_cases():
    rng = np.random.default_rng(0)
    sig = rng.integers(1, 50, size=(40, 12)).astype(np.uint16)
    sig[7] = sig[3]                                    # an identical pair
    c = oracle.lsh_candidates(sig, 3, 4, sig)
    assert all(n in c[n] for n in range(40))           # every row is its own candidate
    assert 7 in c[3] and 3 in c[7]
    q = sig[5].copy()
    q[:9] = 0                                          # only band 3 still equal
    assert 5 in oracle.lsh_candidates(sig, 3, 4, q[None])[0]
    q[9:] = 0
    assert len(oracle.lsh_candidates(sig, 3, 4, q[None])[0]) == 0
