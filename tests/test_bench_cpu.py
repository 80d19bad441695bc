"""Host logic of bench.py (no GPU): the strong-scaling shards, the roofline's
required work (Theorem 2's capped expectation and the expected maximum over a
32-row group), and the reference arm's lazy c5 data."""
import numpy as np
import pytest

import bench


@pytest.mark.parametrize("N,G", [(16_000_000, 1), (16_000_000, 8), (1000, 3), (7, 8), (1, 2)])
def test_shards_partition_the_rows(N, G):
    import paper_1602_08393_b200 as wmh
    parts = [bench.shard(N, r, G) for r in range(G)]
    assert parts == [wmh.shard(N, r, G) for r in range(G)]
    assert parts[0][0] == 0 and parts[-1][1] == N
    assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
    sizes = [b - a for a, b in parts]
    assert max(sizes) - min(sizes) <= 1


def test_expected_draws_matches_theorem2():
    """E[min(G, cap)] = (1 - (1 - s)^cap) / s for G ~ Geom(s) (reading R9)."""
    M, k, cap = 1000, 3, 50
    x_sum = np.array([0, 10, 250, 1000])
    s = x_sum / M
    want = 0.0
    for si in s:
        want += k * (cap if si == 0 else (1 - (1 - si) ** cap) / si)
    assert bench.expected_draws(x_sum, M, k, cap) == pytest.approx(want, rel=1e-12)


def test_group_expected_max_against_simulation():
    """E[max_r min(G_r, cap)] over a 32-row group, against a seeded simulation of
    the geometric first-green draws; all-zero rows contribute nothing."""
    rng = np.random.default_rng(3)
    M, cap = 10_000, 65535
    x_sum = np.concatenate([rng.integers(200, 600, size=60), [0, 0, 0, 0]]).astype(np.int64)
    rng.shuffle(x_sum)
    got, sampled = bench.group_expected_max(x_sum, M, cap)
    assert sampled == 2
    s = x_sum / M
    T = 200_000
    tot = 0.0
    for g in range(2):
        sg = s[32 * g:32 * g + 32]
        sg = sg[sg > 0]
        draws = rng.geometric(sg[None, :], size=(T, len(sg)))
        tot += np.minimum(draws, cap).max(axis=1).mean()
    assert got == pytest.approx(tot, rel=5e-3)


def test_group_expected_max_single_row_is_theorem2():
    """A group with one live row: the maximum is that row's own capped geometric."""
    M, cap = 100, 30
    x_sum = np.zeros(32, np.int64)
    x_sum[5] = 7
    got, _ = bench.group_expected_max(x_sum, M, cap)
    s = 7 / M
    assert got == pytest.approx((1 - (1 - s) ** cap) / s, rel=1e-9)


def test_reference_data_is_lazy_for_c5():
    import datagen
    cfg, data = bench.reference_data("c5", 16_000_000)
    assert isinstance(data, datagen.CounterRows) and data.n_rows == 16_000_000
    x = data.rows(np.array([0, 15_999_999]))
    assert x.shape == (2, 4096)
    assert np.array_equal(x, datagen.gen_counter_c5_rows(cfg.data_seed, np.array([0, 15_999_999]), 4096))


def test_group_expected_max_64_row_tiles_against_simulation():
    """The same expectation over the 64-row tiles of the bit-sliced kernel (G = 2)."""
    rng = np.random.default_rng(4)
    M, cap = 10_000, 65535
    x_sum = rng.integers(200, 600, size=128).astype(np.int64)
    got, sampled = bench.group_expected_max(x_sum, M, cap, rows=64)
    assert sampled == 2
    s = x_sum / M
    T = 100_000
    tot = 0.0
    for g in range(2):
        draws = rng.geometric(s[64 * g:64 * g + 64][None, :], size=(T, 64))
        tot += np.minimum(draws, cap).max(axis=1).mean()
    assert got == pytest.approx(tot, rel=5e-3)


def test_tile_need_rate_is_the_mean_tile_column_max_over_M():
    """q per tile = sum_c max over the tile's rows of x[r][c] / M (a draw can only
    be green where its offset is below that maximum); ragged last tile included."""
    import datagen
    rng = np.random.default_rng(6)
    x = rng.integers(0, 9, size=(130, 8)).astype(np.uint8)
    M = int(x.max(axis=0).astype(np.int64).sum())
    want = np.mean([x[a:a + 64].max(axis=0).astype(np.int64).sum() / M for a in (0, 64, 128)])
    got = bench.tile_need_rate(None, datagen.Dense(x), 130, 64, M)
    assert got == pytest.approx(want, rel=1e-12)


def test_index_cf_mirrors_kernel_warp_choice():
    """bench.py's INDEX floor recomputes the kernel's own per-row plan, so it must
    use the kernel's fallback cost: 2 for dense rows, 64 for CSR rows hashed with
    2-4 warps (c3: k = 1000), with 8 warps (c4: k = 4000) 6 when the row's column
    bitmap fits shared memory (dim <= ~66,000), else 24."""
    import bench
    assert bench.index_cf(1000, False) == 64.0
    assert bench.index_cf(4000, False) == 24.0                       # dim too wide for the bitmap
    assert bench.index_cf(4000, False, 65536) == 6.0                 # c4: the bitmap
    assert bench.index_cf(4000, False, 66240) == 6.0 and bench.index_cf(4000, False, 66241) == 24.0
    assert bench.index_cf(4000, True) == 2.0
    assert bench.index_cf(1024, False) == 64.0 and bench.index_cf(1025, False) == 64.0   # 4 warps
    assert bench.index_cf(2049, False) == 24.0 and bench.index_cf(2049, False, 1000) == 6.0
