"""f3 measurement: build a (K, L) banding LSH index over c2's 10^5 x 500 signatures
and query 10^4 rows (CUDA events).  Prints one JSON line."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402
import paper_1602_08393_b200 as wmh  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        out = fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps, out


def main(K=5, L=20, n_q=10000):
    cfg, data = datagen.make("c2")
    rows = wmh.Rows.from_dense(torch.from_numpy(data.x).cuda())
    layout = wmh.prepare(rows)
    sig = wmh.hash(layout, rows, cfg.seed, cfg.k, cfg.cap)
    build_ms, ix = timed(lambda: wmh.LSH(sig, K, L))
    q = sig[:n_q]
    query_ms, (counts, _) = timed(lambda: ix.query(q, max_out=64))
    c = counts.to(torch.int64)
    print(json.dumps({"what": "f3 banding LSH over c2 signatures", "n_rows": sig.shape[0], "k": sig.shape[1],
                      "K": K, "L": L, "build_ms": build_ms, "n_queries": n_q, "query_ms": query_ms,
                      "queries_per_s": n_q / (query_ms / 1e3), "mean_candidates": float(c.float().mean()),
                      "max_candidates": int(c.max())}))


if __name__ == "__main__":
    main()
