"""Scratch edge probes (GPU): large M through the index (direct-build fallback),
uint16 weights through wmh_hash_host, k at the index limit through the hasher."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import datagen, oracle
import paper_1602_08393_b200 as wmh
from tests.helpers import oracle_hash

def csr(dense):
    rp = np.concatenate([[0], np.cumsum((dense > 0).sum(1))]).astype(np.int64)
    col = np.concatenate([np.nonzero(r)[0] for r in dense]).astype(np.int32)
    val = np.concatenate([r[r > 0] for r in dense]).astype(dense.dtype)
    return rp, col, val

rng = np.random.default_rng(5)
# 1. M = 2^20 * 255 = 2.7e8 through AUTO (index) on 6 CSR rows
D = 1 << 20
rows_np = np.zeros((6, D), np.uint8)
for r in range(6):
    idx = rng.choice(D, 3000, replace=False)
    rows_np[r, idx] = rng.integers(1, 256, 3000)
rp, col, val = csr(rows_np)
rows = wmh.Rows.from_csr(torch.from_numpy(rp).cuda(), torch.from_numpy(col).cuda(), torch.from_numpy(val).cuda(), D)
layout = wmh.prepare(rows, bounds=torch.full((D,), 255, dtype=torch.uint32, device="cuda"))
layout_big = layout
t = time.time()
sig = wmh.hash(layout, rows, 9, 32, 65535).cpu().numpy().astype(np.uint32)
print("bigM algo", wmh.last_algo, "%.2fs" % (time.time() - t), flush=True)
L = oracle.Layout(np.full(D, 255, np.uint32))
ref = oracle_hash(L, datagen.CSR(rp, col, val, D), 9, 32, 65535)
print("bigM parity", np.array_equal(sig, ref), flush=True)
t = time.time()
sigi = wmh.hash(layout, rows, 9, 32, 65535, algo="index").cpu().numpy().astype(np.uint32)
print("bigM index %.2fs" % (time.time() - t), "horizon", wmh.last_horizon, "parity", np.array_equal(sigi, ref), flush=True)
# 2. uint16 dense weights through wmh_hash_host
x = (rng.integers(0, 3000, (300, 256)) * (rng.random((300, 256)) < 0.4)).astype(np.uint16)
dev_rows = wmh.Rows.from_dense(torch.from_numpy(x.view(np.int16)).cuda().view(torch.uint16))
layout = wmh.prepare(dev_rows)
d = wmh.hash(layout, dev_rows, 3, 40, 65535).cpu()
h = wmh.hash_host(layout, wmh.Rows.from_dense(torch.from_numpy(x.view(np.int16)).view(torch.uint16).pin_memory()), 3, 40, 65535)
print("u16 host==dev", torch.equal(d, h), flush=True)
# 3. the hasher at k = 50000
rows_np = ((rng.random((4, 512)) < 0.5) * rng.integers(1, 16, (4, 512))).astype(np.uint8)
rp, col, val = csr(rows_np)
rows = wmh.Rows.from_csr(torch.from_numpy(rp).cuda(), torch.from_numpy(col).cuda(), torch.from_numpy(val).cuda(), 512)
layout = wmh.prepare(rows)
hs = wmh.Hasher(layout, 2, 50000, 65535)
a = hs.hash(rows).cpu()
b = wmh.hash(layout, rows, 2, 50000, 65535, algo="simple").cpu()
print("hasher k=50000", torch.equal(a, b), flush=True)
try:
    wmh.Hasher(layout, 2, 65536, 65535)
    print("hasher k=65536: accepted?!")
except wmh.WmhError as e:
    print("hasher k=65536 rejected:", str(e)[:80])
print("post-error call ok", torch.equal(wmh.hash(layout, rows, 2, 16, 65535, algo="simple").cpu(), wmh.hash(layout, rows, 2, 16, 65535, algo="index").cpu()))
