"""World-size-2 gloo tests (CPU) of the multi-GPU host logic: the row sharding and
the a2 max exchange that makes M -- hence every draw -- identical on every rank
(P:190), so signatures do not depend on how rows are sharded."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_rows, dim):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import datagen
        import oracle
        import paper_1602_08393_b200 as wmh

        # every rank regenerates only its shard (counter-based rows)
        lo, hi = wmh.shard(n_rows, rank, world)
        x_local = datagen.gen_counter_c5_rows(1005, np.arange(lo, hi), dim)
        # shards tile [0, n) exactly
        spans = [None] * world
        dist.all_gather_object(spans, (lo, hi))
        assert spans[0][0] == 0 and spans[-1][1] == n_rows
        assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))

        local_m = torch.from_numpy(oracle.colmax_dense(x_local))
        b = wmh.reduce_bounds(local_m.clone())            # default group (initialised, world > 1)
        x_all = datagen.gen_counter_c5_rows(1005, np.arange(n_rows), dim)
        global_m = oracle.colmax_dense(x_all)
        assert np.array_equal(b.numpy(), global_m), "all-reduce(MAX) must give the global column max"
        assert np.array_equal(wmh.reduce_bounds(local_m.clone(), group=False).numpy(), local_m.numpy())

        # signature invariance across sharding on the oracle side
        L = oracle.Layout(b.numpy())
        sig_shard = L.hash_dense(x_local, 1, 24, 65535, threads=1)
        sig_all = L.hash_dense(x_all, 1, 24, 65535, threads=1)
        assert np.array_equal(sig_shard, sig_all[lo:hi])
        gathered = [None] * world
        dist.all_gather_object(gathered, sig_shard)
        assert np.array_equal(np.concatenate(gathered), sig_all)
        # the binding's optional signature exchange (all-gather, unequal shards)
        full = wmh.gather_signatures(torch.from_numpy(sig_shard.astype(np.int16)).view(torch.uint16))
        assert np.array_equal(full.view(torch.int16).numpy().astype(np.uint16).astype(np.uint32), sig_all)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_rows", [101, 64])
def test_gloo_world2_sharding_and_max_exchange(n_rows):
    mp.spawn(_worker, args=(2, _free_port(), n_rows, 96), nprocs=2, join=True)


def test_shard_arithmetic():
    import paper_1602_08393_b200 as wmh
    for n in (0, 1, 7, 100, 1001):
        for w in (1, 2, 3, 8):
            spans = [wmh.shard(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        wmh.shard(10, 2, 2)
