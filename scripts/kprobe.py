#!/usr/bin/env python
"""Kernel-time probe: hash N rows of a config's recipe (device-generated for
c1/c5) with a chosen k / tile / algo and print the dominant kernel's CUDA-event
time (ms) over a few launches.  For A/B experiments, not a bench line.

    python scripts/kprobe.py --config c5 --rows 1048576 --k 1024 8 --tile bitslice
"""
import argparse
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--rows", type=int, default=1 << 20)
    ap.add_argument("--k", type=int, nargs="+", default=[1024])
    ap.add_argument("--tile", default="auto")
    ap.add_argument("--algo", default="auto")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--isgreen", default="table", choices=["table", "bsearch"])
    a = ap.parse_args()
    import datagen
    import paper_1602_08393_b200 as wmh
    cfg = datagen.CONFIGS[a.config]
    if a.config in ("c1", "c5"):
        x = torch.empty((a.rows, cfg.dim), dtype=torch.uint8, device="cuda")
        for r0 in range(0, a.rows, 1 << 20):
            r1 = min(a.rows, r0 + (1 << 20))
            x[r0:r1] = datagen.gpu_counter_rows(a.config, cfg.data_seed, r0, r1 - r0, cfg.dim)
        rows = wmh.Rows.from_dense(x)
    else:
        from tests.helpers import to_rows
        _, data = datagen.make(a.config, n_rows=a.rows)
        rows = to_rows(data)
    layout = wmh.prepare(rows) if cfg.fixed_bound is None else \
        wmh.prepare(rows, bounds=torch.full((cfg.dim,), cfg.fixed_bound, dtype=torch.uint32, device="cuda"))
    for k in a.k:
        out = torch.empty((rows.n_rows, k), dtype=torch.uint16, device="cuda")
        ms = []
        for i in range(a.reps + 1):
            wmh.hash(layout, rows, cfg.seed, k, cfg.cap, 2, algo=a.algo, out=out, tile=a.tile, time_kernel=True,
                     isgreen=a.isgreen)
            ms.append(wmh.last_kernel_ms())
        print(f"{a.config} rows={rows.n_rows} k={k} tile={a.tile} algo={wmh.last_algo} isgreen={a.isgreen}: "
              f"{statistics.median(ms[1:]):.3f} ms (kernel)", flush=True)


if __name__ == "__main__":
    main()
