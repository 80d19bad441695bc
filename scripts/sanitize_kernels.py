#!/usr/bin/env python
"""Every kernel of libwmh.so on small inputs, for compute-sanitizer:

    compute-sanitizer --tool memcheck  python scripts/sanitize_kernels.py
    compute-sanitizer --tool racecheck python scripts/sanitize_kernels.py
    compute-sanitizer --tool synccheck python scripts/sanitize_kernels.py

Inputs are c1/c2/c3/c4/c5-recipe slices (several tiles and a ragged tail) plus
the shapes that select the clamped and group-major bit-sliced tiles.  Results
are also checked against the oracle, so a sanitizer run is a parity run too.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402
import oracle  # noqa: E402
import paper_1602_08393_b200 as wmh  # noqa: E402
from tests.helpers import oracle_bounds, oracle_hash, to_rows  # noqa: E402


def check(sig, ref, what):
    got = sig.view(torch.int16).cpu().numpy().view(np.uint16).astype(np.uint32) if sig.dtype == torch.uint16 \
        else sig.cpu().numpy().astype(np.uint32)
    assert np.array_equal(got, ref), what
    print("ok", what, flush=True)


def run_dense(name, n, k, cap, sb, x=None):
    if x is None:
        cfg, data = datagen.make(name, n_rows=n)
    else:
        data = datagen.Dense(x)
    rows = to_rows(data)
    layout = wmh.prepare(rows)
    wmh.check_rows(layout, rows)
    L = oracle.Layout(oracle_bounds(data))
    ref = oracle_hash(L, data, 7, k, cap)
    for algo, tile in [("simple", "auto"), ("tiled", "bytes"), ("tiled", "bitplanes"), ("tiled", "bitslice"),
                       ("index", "auto")]:
        try:
            sig = wmh.hash(layout, rows, 7, k, cap, sb, algo=algo, tile=tile)
        except wmh.WmhError as e:
            print("skip", name, algo, tile, str(e)[:60])
            continue
        torch.cuda.synchronize()
        check(sig, ref, f"{name} {algo}/{tile}")
    return rows, layout, data


def main():
    torch.cuda.set_device(0)
    from paper_1602_08393_b200 import build
    build.build()
    run_dense("c1", 300, 64, 255, 1)
    run_dense("c2", 300, 96, 65535, 2)
    rows5, layout5, data5 = run_dense("c5", 200, 128, 65535, 2)
    # clamped bit-sliced tiles: D = 4096 with two wide columns (P = 6 of 7), D = 2912 with bounds to 31 (P = 4 of 5)
    rng = np.random.default_rng(1)
    x = (rng.integers(1, 64, size=(70, 4096)) * (rng.random((70, 4096)) < 0.05)).astype(np.uint8)
    x[:, 7] = np.where(np.arange(70) % 2 == 0, 100, 0)
    run_dense("clamp7", 70, 32, 65535, 2, x)
    x = rng.integers(0, 16, size=(150, 2912)).astype(np.uint8)
    x[rng.random(x.shape) < 0.6] = 0
    x[0, 0] = 31
    run_dense("clamp5", 150, 32, 65535, 2, x)
    # sparse rows: index and simple
    for name, n, k in [("c3", 60, 200), ("c4", 40, 400)]:
        cfg, data = datagen.make(name, n_rows=n)
        rows = to_rows(data)
        layout = wmh.prepare(rows, bounds=None if cfg.fixed_bound is None else
                             torch.full((cfg.dim,), cfg.fixed_bound, dtype=torch.uint32, device="cuda"))
        L = oracle.Layout(oracle_bounds(data, cfg.fixed_bound))
        ref = oracle_hash(L, data, 7, k, cfg.cap)
        for algo in ("index", "simple"):
            check(wmh.hash(layout, rows, 7, k, cfg.cap, 2, algo=algo), ref, f"{name} {algo}")
        hs = wmh.Hasher(layout, 7, k, cfg.cap)
        check(hs.hash(rows), ref, f"{name} hasher")
    # uint16 weights (f1) and the quantiser / scale objective
    cfg, data = datagen.make("c2", n_rows=128)
    xf = torch.from_numpy(datagen.gen_c2_real_rows(cfg.data_seed, 0, 128, cfg.dim)).cuda()
    scale = wmh.choose_scale(wmh.Rows.from_dense(xf), [1.0, 2.0, 4.0])
    q = wmh.quantize(xf, scale)
    rq = wmh.Rows.from_dense(q)
    lq = wmh.prepare(rq)
    qn = q.view(torch.int16).cpu().numpy().view(np.uint16)
    Lq = oracle.Layout(oracle.colmax_dense(qn))
    refq = Lq.hash_dense(qn, 7, 64, 65535)
    for algo in ("index", "simple"):
        check(wmh.hash(lq, rq, 7, 64, 65535, 2, algo=algo), refq, f"uint16 {algo}")
    # collide, collide2, LSH, host e2e
    sig5 = wmh.hash(layout5, rows5, 7, 128, 65535, 2)
    pairs = torch.from_numpy(datagen.random_pairs(3, 200, 500)).cuda()
    m, _ = wmh.collide(sig5, pairs)
    a = wmh.sketch(layout5, rows5, 7, 128, 65535)
    m2, _ = wmh.collide_sketches(a, a, pairs[:, 0].contiguous(), pairs[:, 1].contiguous())
    assert torch.equal(m, m2)
    print("ok collide / collide2", flush=True)
    idx = wmh.LSH(sig5, K=4, L=8)
    idx.query(sig5[:20], max_out=16)
    print("ok lsh", flush=True)
    hx = torch.from_numpy(np.ascontiguousarray(data5.x)).pin_memory()
    out = wmh.hash_host(layout5, wmh.Rows.from_dense(hx), 7, 128, 65535, 2)
    assert torch.equal(out.view(torch.int16), sig5.cpu().view(torch.int16))
    print("ok hash_host", flush=True)
    wmh.empty_launch()
    torch.cuda.synchronize()
    print("all kernels ran", flush=True)


if __name__ == "__main__":
    main()
