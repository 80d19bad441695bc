"""Figure 2 protocol through the C ABI: 200 seeds x 50 hashes of the
nine J = 0.1..0.9 pairs; signatures bit-identical to the oracle for every seed,
and the error curves within 5 standard errors of the exact binomial law."""
import numpy as np
import pytest
import torch

import datagen
import oracle
from tests.fig2 import K_MAX, error_curves

pytestmark = pytest.mark.gpu


def test_fig2_error_curves_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1602_08393_b200 as wmh
    x, y, J = datagen.fig2_pairs()
    rows_np = np.concatenate([x, y])
    rows = wmh.Rows.from_dense(torch.from_numpy(rows_np).cuda())
    layout = wmh.prepare(rows)
    L = oracle.Layout(oracle.colmax_dense(rows_np))

    def sig(seed):
        s = wmh.hash(layout, rows, seed, K_MAX, 65535).view(torch.int16).cpu().numpy().view(np.uint16)
        s = s.astype(np.uint32)
        assert np.array_equal(s, L.hash_dense(rows_np, seed, K_MAX, 65535)), seed
        return s

    mae, z = error_curves(sig, J)
    assert np.abs(z).max() <= 5.0
    assert np.all(mae[:, -1] < mae[:, 0])
