"""Figure 2 protocol on the GPU path: writes the mean absolute error
of J-hat_k (200 seeds, k = 1..50, nine pairs J = 0.1..0.9) next to the exact
binomial law to a CSV.  Usage: python scripts/fig2_accuracy.py out.csv"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402
import paper_1602_08393_b200 as wmh  # noqa: E402
from tests.fig2 import K_MAX, error_curves, exact_mae  # noqa: E402


def main(out):
    x, y, J = datagen.fig2_pairs()
    rows = wmh.Rows.from_dense(torch.from_numpy(np.concatenate([x, y])).cuda())
    layout = wmh.prepare(rows)
    mae, z = error_curves(
        lambda seed: wmh.hash(layout, rows, seed, K_MAX, 65535).view(torch.int16).cpu().numpy().view(np.uint16)
        .astype(np.uint32), J)
    with open(out, "w") as f:
        f.write("k," + ",".join(f"mae_J{j:.1f}" for j in J) + "," + ",".join(f"exact_J{j:.1f}" for j in J) + "\n")
        for k in range(1, K_MAX + 1):
            f.write(f"{k}," + ",".join(f"{mae[p, k - 1]:.5f}" for p in range(9)) + "," +
                    ",".join(f"{exact_mae(J[p], k):.5f}" for p in range(9)) + "\n")
    print(f"max |z| = {np.abs(z).max():.2f} over {z.size} (pair, k) points; wrote {out}")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "fig2_accuracy.csv")
