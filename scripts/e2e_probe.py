"""PCIe bounds for the e2e leg: pinned H2D / D2H bandwidth alone and both at once,
then wmh_hash_host on c2 (chunk count from WMH_E2E_CHUNKS)."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import datagen
import paper_1602_08393_b200 as wmh


def bw():
    n = 100 << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = {}
    for name, fn in [("h2d", lambda: d.copy_(h, non_blocking=True)),
                     ("d2h", lambda: h2.copy_(d2, non_blocking=True))]:
        fn(); torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        out[name + "_gbs"] = 5 * n / (time.perf_counter() - t) / 1e9
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    out["both_gbs_each"] = 5 * n / (time.perf_counter() - t) / 1e9
    return out


def e2e():
    cfg, data = datagen.make("c2")
    hx = torch.from_numpy(data.x).pin_memory()
    rows = wmh.Rows.from_dense(hx)
    layout = wmh.prepare(wmh.Rows.from_dense(hx.cuda()))
    out = torch.empty((hx.shape[0], cfg.k), dtype=torch.uint16).pin_memory()
    for _ in range(2):
        wmh.hash_host(layout, rows, cfg.seed, cfg.k, cfg.cap, 2, out=out)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        wmh.hash_host(layout, rows, cfg.seed, cfg.k, cfg.cap, 2, out=out)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 5
    return {"e2e_ms": dt * 1e3, "hashes_per_s": hx.shape[0] * cfg.k / dt}


if __name__ == "__main__":
    r = e2e()
    if "--bw" in sys.argv:
        r.update(bw())
    print(json.dumps(r))
