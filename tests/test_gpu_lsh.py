"""f3 GPU parity: the banding LSH index through the C ABI against the oracle --
exact candidate sets and counts, truncation, uint8 and uint16 signatures, and
the index built from real signatures of the hash path."""
import numpy as np
import pytest
import torch

import datagen
import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def wmh():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1602_08393_b200 as w
    return w


def _to_dev(a):
    if a.dtype == np.uint16:
        return torch.from_numpy(a.astype(np.int32)).to(torch.uint16).cuda()
    return torch.from_numpy(a).cuda()


@pytest.mark.parametrize("dt,K,L", [(np.uint16, 4, 8), (np.uint8, 2, 16), (np.uint16, 1, 3)])
def test_lsh_matches_oracle(wmh, dt, K, L):
    rng = np.random.default_rng(K * 100 + L)
    n, k = 3000, 64
    sig = rng.integers(1, 5, size=(n, k)).astype(dt)
    sig[10] = sig[20]
    q = np.concatenate([sig[:200], rng.integers(1, 5, size=(300, k)).astype(dt)])
    ix = wmh.LSH(_to_dev(sig), K, L)
    counts, rows = ix.query(_to_dev(q), max_out=3000)
    ref = oracle.lsh_candidates(sig, K, L, q)
    counts = counts.cpu().numpy().astype(np.int64)
    rows = rows.cpu().numpy()
    for i, r in enumerate(ref):
        assert counts[i] == len(r), i
        assert np.array_equal(np.sort(rows[i, :counts[i]]), r), i
        assert np.all(rows[i, counts[i]:] == -1)
    # truncated output: exact counts, a subset of the true candidates
    c2, r2 = ix.query(_to_dev(q), max_out=3)
    c2 = c2.cpu().numpy().astype(np.int64)
    r2 = r2.cpu().numpy()
    assert np.array_equal(c2, counts)
    for i, r in enumerate(ref):
        got = r2[i][r2[i] >= 0]
        assert len(got) == min(3, len(r)) and set(got.tolist()) <= set(r.tolist())


def test_lsh_on_hash_signatures(wmh):
    """Signatures of c2 rows from the hash path; near-duplicates planted by copying
    rows (identical rows collide in every band)."""
    cfg, data = datagen.make("c2", n_rows=2000)
    x = data.x.copy()
    x[1000:1010] = x[0:10]
    rows = wmh.Rows.from_dense(torch.from_numpy(x).cuda())
    layout = wmh.prepare(rows)
    sig = wmh.hash(layout, rows, 1, 100, 65535)
    ix = wmh.LSH(sig, 5, 20)
    counts, cand = ix.query(sig[:10], max_out=64)
    sig_np = sig.view(torch.int16).cpu().numpy().view(np.uint16)
    ref = oracle.lsh_candidates(sig_np, 5, 20, sig_np[:10])
    for i in range(10):
        assert int(counts[i]) == len(ref[i])
        assert np.array_equal(np.sort(cand[i, :int(counts[i])].cpu().numpy()), ref[i])
        assert 1000 + i in ref[i]
