import sys, os, numpy as np, torch
sys.path.insert(0, '/root/repo')
import datagen, oracle, paper_1602_08393_b200 as wmh
from tests.helpers import oracle_bounds, oracle_hash, to_rows
cfg, data_all = datagen.make("c3", n_rows=80)
for n in [20, 25, 30, 35, 40, 45, 50, 55, 60, 80]:
    data = data_all.take(np.arange(n))
    rows = to_rows(data)
    layout = wmh.prepare(rows)
    L = oracle.Layout(oracle_bounds(data))
    ref = oracle_hash(L, data, 7, 64, cfg.cap)
    sig = wmh.hash(layout, rows, 7, 64, cfg.cap, 2, algo="tiled")
    got = sig.view(torch.int16).cpu().numpy().view(np.uint16).astype(np.uint32)
    bad = np.argwhere(got != ref)
    print(n, "M", layout.M, "nnz", len(data.col), "mismatch", len(bad), "ref t of bad", sorted(set(ref[got != ref].tolist()))[:10], flush=True)
