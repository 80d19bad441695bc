"""Figure 2 protocol on the oracle (CPU): the error curves follow the exact law
of an unbiased WMH estimator (Theorem 1), pointwise within 5 standard errors."""
import numpy as np

import datagen
import oracle
from tests.fig2 import K_MAX, error_curves, exact_mae


def test_fig2_error_curves_oracle():
    x, y, J = datagen.fig2_pairs()
    rows = np.concatenate([x, y])
    L = oracle.Layout(oracle.colmax_dense(rows))
    mae, z = error_curves(lambda seed: L.hash_dense(rows, seed, K_MAX, 65535), J)
    assert np.abs(z).max() <= 5.0, np.abs(z).max()
    assert np.all(mae[:, -1] < mae[:, 0])                 # error at k=50 < error at k=1
    assert abs(exact_mae(0.5, 1) - 0.5) < 1e-12
