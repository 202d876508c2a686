"""Exact top-k under value ties on the tensor-core path (R13: ties -> lower index).

The tcgen05 epilogue walks a 32-column chunk's candidates in the candidate
mask's bit order, which is not column order (bit 8i + r <-> column 4r + i).
A candidate whose value equals the list's k-th value but whose index is lower
must still displace the k-th key, so the own-list test compares full keys
(VERDICT r1 "What's weak" 2).  These cases force exactly that pattern:

* the round-1 reproducer (n = 256, M = 16, one query, k = 1): row 0 sums to
  96, rows 1 and 4 to 48, all others to 160 -- the mask order visits row 4
  before row 1, and the answer is row 1;
* three-level tables (each row's codes all 0, 1 or 2, so every sum is one of
  three values) over several 256-vector tiles and row partitions: about a
  third of the rows tie at the best value and the top-k is the lowest-index
  ones; for k = 100 the lists of 32 and group thresholds (pair tiles);
* constant tables: every sum equal, top-k = the k lowest indices.

Both tile modes run: single-CTA 128-query tiles (nq <= 128, k <= 32) and CTA
pairs (nq > 128, or k > 32), for both metrics.  Every key is compared with
the oracle (O8) bit for bit.
"""
import numpy as np
import pytest
import torch

from synth import generators as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bolt():
    import paper_1706_10283_b200 as bolt
    assert torch.cuda.is_available(), "GPU tests need a B200"
    bolt._lib.load()
    return bolt


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def three_level_tables(nq, m, metric):
    """Entry 1 is the best code, 2 the middle, 0 the worst (per metric)."""
    ql = np.zeros((nq, m, 16), np.uint8)
    if metric == 0:
        ql[:, :, 0], ql[:, :, 1], ql[:, :, 2] = 10, 3, 6
    else:
        ql[:, :, 0], ql[:, :, 1], ql[:, :, 2] = 3, 10, 6
    return ql


def rows_of_levels(levels, m):
    """Each row's M codes all equal its level (0, 1 or 2)."""
    return np.repeat(np.asarray(levels, np.uint8)[:, None], m, axis=1)


def _check(bolt, orc, flat, ql, k, metric, nq_mode, index_base=0, variant=None):
    n = flat.shape[0]
    codes = bolt.pack_codes(dev(flat))
    variant = bolt.VARIANT_TC if variant is None else variant
    got = host(bolt.topk(codes, n, dev(ql), k, metric, index_base=index_base, variant=variant))
    ref = orc.topk(flat, ql, k, metric, index_base=index_base)
    np.testing.assert_array_equal(got, ref, err_msg=f"mode {nq_mode}, k {k}, metric {metric}")
    return got


# nq = 1 and 64: single-CTA tiles; 130 and 257: CTA pairs (two query tiles)
MODES = [("single", 1), ("single", 64), ("pair", 130), ("pair", 257)]


@pytest.mark.parametrize("metric", [0, 1])
@pytest.mark.parametrize("mode,nq", MODES)
def test_round1_reproducer(bolt, orc, metric, mode, nq):
    m, n = 16, 256
    levels = np.zeros(n, np.int64)          # sum 160 (L2) / 48 (dot): worst
    levels[0] = 2                           # 96: middle
    levels[[1, 4]] = 1                      # 48 (L2) / 160 (dot): best, tied
    flat = rows_of_levels(levels, m)
    ql = three_level_tables(nq, m, metric)
    got = _check(bolt, orc, flat, ql, 1, metric, mode)
    v, idx = bolt.keys_split(dev(got), metric)
    assert (host(idx)[:, 0] == 1).all()
    if mode == "single":
        assert bolt.topk_plan(n, m, nq, 1, bolt.VARIANT_TC)[0] == "tc"


@pytest.mark.parametrize("metric", [0, 1])
@pytest.mark.parametrize("k", [1, 10, 32, 100])
@pytest.mark.parametrize("mode,nq", MODES)
@pytest.mark.parametrize("n", [256, 3001, 70_001])
def test_three_level_ties(bolt, orc, metric, k, mode, nq, n):
    m = 16
    levels = np.random.default_rng(n + k).integers(0, 3, n)
    flat = rows_of_levels(levels, m)
    ql = three_level_tables(nq, m, metric)
    got = _check(bolt, orc, flat, ql, k, metric, mode, index_base=11)
    best = np.flatnonzero(levels == 1)[:k] + 11
    _, idx = bolt.keys_split(dev(got), metric)
    np.testing.assert_array_equal(host(idx)[0, :len(best)], best)


@pytest.mark.parametrize("metric", [0, 1])
@pytest.mark.parametrize("k", [1, 10, 32, 100])
@pytest.mark.parametrize("m", [8, 16, 32])
def test_constant_tables_tc(bolt, orc, metric, k, m):
    """Every sum equal: the k lowest indices, in order, for single-CTA tiles
    (nq = 40) and pairs (nq = 200); M = 32 always runs pairs."""
    n = 20_000
    flat = G.random_codes(n, m, 5 + m)
    for nq in (40, 200):
        ql = np.full((nq, m, 16), 7, np.uint8)
        got = _check(bolt, orc, flat, ql, k, metric, f"nq={nq}")
        _, idx = bolt.keys_split(dev(got), metric)
        assert (host(idx) == np.arange(k)[None]).all()


@pytest.mark.parametrize("metric", [0, 1])
@pytest.mark.parametrize("m", [8, 16, 32])
def test_binary_tables_random_codes(bolt, orc, metric, m):
    """Entries in {0, 1}: sums take at most M + 1 values, ties straddle the
    k-th position in every list; several partitions and a ragged tail."""
    n = 100_003
    flat = G.random_codes(n, m, 40 + m)
    for nq, k in ((100, 10), (300, 32), (150, 100)):
        ql = G.random_qluts(nq, m, 41 + nq, hi=2)
        _check(bolt, orc, flat, ql, k, metric, f"nq={nq}")


@pytest.mark.parametrize("metric", [0, 1])
@pytest.mark.parametrize("k", [1, 10, 16, 32])
@pytest.mark.parametrize("nq", [1, 224, 300])
@pytest.mark.parametrize("n", [256, 3001, 70_001])
def test_three_level_ties_sparse(bolt, orc, metric, k, nq, n):
    """The same tie patterns through the 2:4-sparse kernel (BOLT_VARIANT_SP),
    whose lists take candidates in vector order per query."""
    m = 16
    levels = np.random.default_rng(n + k).integers(0, 3, n)
    flat = rows_of_levels(levels, m)
    ql = three_level_tables(nq, m, metric)
    got = _check(bolt, orc, flat, ql, k, metric, "sp", index_base=11, variant=bolt.VARIANT_SP)
    best = np.flatnonzero(levels == 1)[:k] + 11
    _, idx = bolt.keys_split(dev(got), metric)
    np.testing.assert_array_equal(host(idx)[0, :len(best)], best)


@pytest.mark.parametrize("metric", [0, 1])
@pytest.mark.parametrize("m,k", [(8, 32), (16, 10), (32, 16)])
def test_constant_and_binary_tables_sparse(bolt, orc, metric, m, k):
    n = 50_001
    flat = G.random_codes(n, m, 5 + m)
    ql = np.full((250, m, 16), 7, np.uint8)
    got = _check(bolt, orc, flat, ql, k, metric, "sp", variant=bolt.VARIANT_SP)
    _, idx = bolt.keys_split(dev(got), metric)
    assert (host(idx) == np.arange(k)[None]).all()
    ql = G.random_qluts(230, m, 41 + m, hi=2)
    _check(bolt, orc, flat, ql, k, metric, "sp", variant=bolt.VARIANT_SP)
