"""Shared helpers for the GPU parity tests: move datagen inputs to the device and
run the oracle on the same inputs."""
import numpy as np
import torch

import datagen
import oracle


def to_rows(data, device="cuda"):
    import paper_1602_08393_b200 as wmh
    if isinstance(data, datagen.Dense):
        return wmh.Rows.from_dense(torch.from_numpy(np.ascontiguousarray(data.x)).to(device))
    return wmh.Rows.from_csr(torch.from_numpy(data.row_ptr).to(device), torch.from_numpy(data.col).to(device),
                             torch.from_numpy(data.val).to(device), data.dim)


def oracle_bounds(data, fixed_bound=None):
    if fixed_bound is not None:
        return np.full(data.dim, fixed_bound, np.uint32)
    if isinstance(data, datagen.Dense):
        return oracle.colmax_dense(data.x)
    return oracle.colmax_csr(data.row_ptr, data.col, data.val, data.dim)


def oracle_hash(L: "oracle.Layout", data, seed, k, cap, rows=None):
    """Oracle signatures (uint32) of all rows, or of the listed rows."""
    if isinstance(data, datagen.Dense):
        x = data.x if rows is None else data.x[rows]
        return L.hash_dense(x, seed, k, cap)
    sub = data if rows is None else data.take(rows)
    return L.hash_csr(sub.row_ptr, sub.col, sub.val, seed, k, cap)
