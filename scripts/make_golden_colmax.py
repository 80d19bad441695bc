#!/usr/bin/env python
"""Write tests/golden/<cfg>_colmax.txt: the per-column maxima m_c of a
full-size counter-based config, computed by the ORACLE (oracle.colmax_dense)
over rows regenerated on the host by datagen.  Nothing here touches the CUDA
path; the file is an expected value for the full-size parity tests.

    python scripts/make_golden_colmax.py c5 [--procs 8]
"""
import argparse
import os
import sys
from multiprocessing import Pool

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _chunk(args):
    name, lo, hi = args
    import datagen
    import oracle
    cfg = datagen.CONFIGS[name]
    gen = {"c1": datagen.gen_counter_c1_rows, "c5": datagen.gen_counter_c5_rows}[name]
    m = np.zeros(cfg.dim, np.uint32)
    step = 8192
    for a in range(lo, hi, step):
        x = gen(cfg.data_seed, np.arange(a, min(hi, a + step)), cfg.dim)
        m = np.maximum(m, oracle.colmax_dense(x))
    return m


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("name")
    ap.add_argument("--procs", type=int, default=os.cpu_count())
    a = ap.parse_args()
    import datagen
    cfg = datagen.CONFIGS[a.name]
    n = cfg.n_rows
    parts = 256
    spans = [(a.name, i * n // parts, (i + 1) * n // parts) for i in range(parts)]
    with Pool(a.procs) as pool:
        ms = pool.map(_chunk, spans)
    m = np.max(np.stack(ms), axis=0)
    out = os.path.join(ROOT, "tests", "golden", f"{a.name}_colmax.txt")
    with open(out, "w") as f:
        f.write(f"# column maxima of the full {a.name} recipe (N={n}, D={cfg.dim}, data_seed={cfg.data_seed}),\n")
        f.write("# written by scripts/make_golden_colmax.py via oracle.colmax_dense on host-regenerated rows.\n")
        f.write(" ".join(str(int(v)) for v in m) + "\n")
    print(out, "M =", int(m.sum()))


if __name__ == "__main__":
    main()
