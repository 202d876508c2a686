"""Pins of the fp64 CPU oracle against things other than itself (CPU only).

Each test names the PAPER.md passage it checks (P:Lx) and what it is pinned to:
a hand-derived worked example (tests/golden/), a closed form or identity, a
special case that reduces to a library routine (scipy / numpy), or brute force
on tiny inputs.  Chosen so a dropped term, wrong sign/index or transposed
operand in any oracle function fails at least one test.
"""
import json
import os

import numpy as np
import pytest
from scipy.cluster.vq import kmeans2, vq

from synth import generators as G

HERE = os.path.dirname(os.path.abspath(__file__))


def centroid_bank(M, L, seed, scale=1.0):
    return G.random_floats((M, 16, L), seed, scale)


def one_hot(codes, K=16):
    n, M = codes.shape
    oh = np.zeros((n, M, K), np.int64)
    oh[np.arange(n)[:, None], np.arange(M)[None, :], codes.astype(np.int64)] = 1
    return oh.reshape(n, M * K)


# --------------------------------------------------------------- worked example
def test_worked_example_golden(orc):
    """Hand-derived example (tests/golden/worked_example.json): pins layout v1
    unpack, encode, LUT, quantize, scan, top-k keys/ties and dequant at once."""
    g = json.load(open(os.path.join(HERE, "golden", "worked_example.json")))
    M, J = g["M"], g["J"]
    C = np.zeros((M, 16, 1), np.float32)
    C[:, :, 0] = np.arange(16, dtype=np.float32)
    X = np.array(g["rows"], np.float32)
    codes = orc.encode(X, C)
    np.testing.assert_array_equal(codes, np.array(g["codes"]))
    words = np.array(g["layout_v1_words"], np.uint32)
    np.testing.assert_array_equal(orc.unpack_v1(words, len(X), M), codes)
    b = np.array(g["b"], np.float32)

    D = orc.luts(np.array([g["l2_query"]], np.float32), C, orc.L2SQ)
    beta = orc.quantize(D, g["a"], b)
    np.testing.assert_array_equal(beta[0, 0], g["l2_beta_row_m0"])
    acc = orc.scan(codes, beta)[:, 0]
    np.testing.assert_array_equal(acc, g["l2_acc"])
    keys = orc.topk(codes, beta, 2, orc.L2SQ)
    assert [int(x) for x in keys[0]] == [int(s) for s in g["l2_top2_keys"]]
    keys9 = orc.topk(codes, beta, 9, orc.L2SQ)
    assert int(keys9[0, -1]) == int(g["l2_top9_last_key"])

    Dd = orc.luts(np.array([g["dot_query"]], np.float32), C, orc.DOT)
    betad = orc.quantize(Dd, g["a"], b)
    accd = orc.scan(codes, betad)[:, 0]
    np.testing.assert_array_equal(accd, g["dot_acc"])
    assert int(orc.topk(codes, betad, 1, orc.DOT)[0, 0]) == int(g["dot_top1_key"])
    np.testing.assert_array_equal(orc.dequant(accd, g["a"], b), g["dot_dequant"])


# ------------------------------------------------------------------- encode O3
@pytest.mark.parametrize("M,L", [(1, 1), (2, 3), (4, 4), (8, 2), (16, 8)])
def test_encode_matches_scipy_vq(orc, M, L):
    """per subspace the code is the nearest centroid -- the special
    case scipy.cluster.vq.vq computes (a library routine, lowest index on ties)."""
    X = G.random_floats((300, M * L), 10 + M)
    C = centroid_bank(M, L, 20 + M)
    codes = orc.encode(X, C)
    for m in range(M):
        ref, _ = vq(X[:, m * L:(m + 1) * L].astype(np.float64), C[m].astype(np.float64))
        np.testing.assert_array_equal(codes[:, m], ref)


def test_encode_centroid_identity_and_ties(orc):
    """A vector assembled from centroids encodes to their indices (BJ identity);
    duplicated centroids resolve to the lowest index (R9)."""
    M, L = 8, 4
    C = centroid_bank(M, L, 31)
    rng = np.random.default_rng(1)
    idx = rng.integers(0, 16, (200, M))
    X = np.concatenate([C[m][idx[:, m]] for m in range(M)], axis=1)
    np.testing.assert_array_equal(orc.encode(X, C), idx)
    C2 = C.copy()
    C2[:, 9] = C2[:, 4]          # centroid 9 duplicates centroid 4
    X2 = np.concatenate([C2[m][np.full(5, 9)] for m in range(M)], axis=1)
    assert (orc.encode(X2, C2) == 4).all()


def test_encode_gap(orc):
    M, L = 4, 2
    C = centroid_bank(M, L, 5)
    X = G.random_floats((100, M * L), 6)
    codes, gap = orc.encode(X, C, with_gap=True)
    assert (gap >= 0).all() and (gap <= 1).all()
    C2 = C.copy()
    C2[:, 3] = C2[:, 2]
    _, gap2 = orc.encode(np.concatenate([C2[m][[2]] for m in range(M)], 1), C2, with_gap=True)
    assert (gap2 == 0).all()


# --------------------------------------------------------------------- LUT O4
@pytest.mark.parametrize("metric", [0, 1])
def test_lut_additivity_reconstruction(orc, metric):
    """P:L206-209 additivity + P:L329-331 reconstruction: summing the exact
    tables over a vector's codes equals the full-vector reduction of its
    reconstruction x_hat, computed densely with numpy (BJ identity)."""
    M, L = 8, 4
    C = centroid_bank(M, L, 41)
    X = G.random_floats((64, M * L), 42)
    Q = G.random_floats((5, M * L), 43)
    codes = orc.encode(X, C)
    D = orc.luts(Q, C, metric)
    xhat = np.concatenate([C[m][codes[:, m]] for m in range(M)], axis=1).astype(np.float64)
    approx = np.einsum("qmk,nmk->qn", D, one_hot(codes).reshape(-1, M, 16).astype(np.float64))
    Q64 = Q.astype(np.float64)
    if metric == 0:
        dense = ((Q64[:, None, :] - xhat[None]) ** 2).sum(-1)
    else:
        dense = Q64 @ xhat.T
    np.testing.assert_allclose(approx, dense, rtol=1e-12, atol=1e-12)


def test_lut_special_cases(orc):
    """dot with q=0 is all zero; L2 with q^(m)=c_7 gives D[m][7]=0
    while every other entry is the squared distance between the two centroids."""
    M, L = 4, 3
    C = centroid_bank(M, L, 51)
    assert (orc.luts(np.zeros((2, M * L), np.float32), C, orc.DOT) == 0).all()
    q = np.concatenate([C[m][7] for m in range(M)])[None]
    D = orc.luts(q, C, orc.L2SQ)
    assert (D[0, :, 7] == 0).all()
    assert (D[0, :, np.arange(16) != 7] > 0).all()
    # transposition check: entry (m, k) depends on codebook m's centroid k only
    C2 = C.copy()
    C2[2, 5] += 1.0
    D2 = orc.luts(q, C2, orc.L2SQ)
    diff = D2 != D
    assert diff[0, 2, 5] and diff.sum() == 1


# ------------------------------------------------------------------ quantize O6
def test_quantize_spec_examples(orc):
    """P:L279 beta = clamp(floor(a(y - b)), 0, 255) (R1); SPEC S:L236-238 examples."""
    def q1(y, a, b):
        D = np.full((1, 1, 16), y, np.float64)
        return int(orc.quantize(D, a, np.array([b], np.float32))[0, 0, 0])
    assert q1(100.7, 1.0, 0.0) == 100
    assert q1(-3.0, 1.0, 0.0) == 0
    assert q1(1e6, 1.0, 0.0) == 255
    assert q1(255.999, 1.0, 0.0) == 255
    assert q1(3.0, 2.0, 1.5) == 3
    assert q1(1.5, 2.0, 1.5) == 0


def test_quantize_monotone_and_lemma1(orc):
    """Monotone in y; Lemma 1 with the 1/a step (R5):
    in range, |y - yhat| < 1/a with yhat = beta/a + b."""
    rng = np.random.default_rng(3)
    M = 4
    D = np.sort(rng.uniform(-5, 40, (50, M, 16)), axis=None).reshape(50, M, 16)
    a, b = np.float32(6.3), np.array([0.5, -1.0, 2.0, 0.0], np.float32)
    beta = orc.quantize(D, a, b)
    for m in range(M):
        col = beta[:, m, :].ravel()
        assert (np.diff(col.astype(int)) >= 0).all()
    yhat = beta / np.float64(a) + b.astype(np.float64)[None, :, None]
    lo = b.astype(np.float64)[None, :, None]
    inr = (D >= lo) & (D < lo + 255.0 / np.float64(a))
    assert inr.sum() > 1000
    err = np.abs(D - yhat)[inr]
    assert (err < 1.0 / np.float64(a)).all()


# ----------------------------------------------------------------- calibrate O5
def test_calibrate_nearest_rank_matches_numpy(orc):
    """P:L289 b = F^-1(alpha): the empirical inverse CDF is numpy's
    'inverted_cdf' quantile (library routine); a = 255 / F^-1(1-alpha) of the
    pooled residuals (R2); the returned alpha is the grid argmin."""
    rng = np.random.default_rng(7)
    nq, M = 40, 4
    D = rng.gamma(2.0, 3.0, (nq, M, 16)) + np.arange(M)[None, :, None] * 10
    a, b, alpha, mse = orc.calibrate(D)
    grid = [0, .001, .002, .005, .01, .02, .05, .1]
    assert alpha == grid[int(np.argmin(mse))]
    for m in range(M):
        assert b[m] == np.quantile(D[:, m, :].ravel(), alpha, method="inverted_cdf")
    resid = (D - b[None, :, None]).ravel()
    assert a == pytest.approx(255.0 / np.quantile(resid, 1 - alpha, method="inverted_cdf"), rel=1e-15)
    # the reported error is the reconstruction MSE of P:L283-286 for the chosen (a, b)
    beta = np.clip(np.floor(a * (D - b[None, :, None])), 0, 255)
    yhat = beta / a + b[None, :, None]
    assert mse[grid.index(alpha)] == pytest.approx(((yhat - D) ** 2).mean(), rel=1e-12)


def _nearest_rank_checks(orc, D):
    """Every grid alpha (not only the winner): b_m = F_m^-1(alpha) and
    a = 255 / F^-1(1 - alpha) of the pooled residuals, both numpy's
    'inverted_cdf' quantile (library routine), and the grid error recomputed
    from P:L283-286."""
    ag, bg, mse = orc.calibrate_grid(D)
    M = D.shape[1]
    for g, alpha in enumerate(orc.ALPHA_GRID):
        for m in range(M):
            assert bg[g, m] == np.quantile(D[:, m, :].ravel(), alpha, method="inverted_cdf"), (alpha, m)
        resid = (D - bg[g][None, :, None]).ravel()
        assert ag[g] == 255.0 / np.quantile(resid, 1 - alpha, method="inverted_cdf"), alpha
        beta = np.clip(np.floor(ag[g] * (D - bg[g][None, :, None])), 0, 255)
        yhat = beta / ag[g] + bg[g][None, :, None]
        assert mse[g] == pytest.approx(((yhat - D) ** 2).mean(), rel=1e-12)
    return ag, bg, mse


def test_calibrate_every_alpha_tail_heavy(orc):
    """P:L289 at alpha > 0: a bulk on [0, 1) with one far outlier above it and
    one below, 200,000 entries per table, so alpha n is an integer at every
    grid point (0.001 n = 200): the nearest rank max(ceil(p n) - 1, 0) and
    floor(p n) pick different entries there, and only the former is numpy's
    inverted CDF.  Clipping the two outliers costs (256^2 + 200^2) / 400,000
    in MSE, less than alpha = 0's resolution loss (step ~1), so the winner is
    alpha = 0.001 (R4), and the returned (a, b) are that grid point's."""
    rng = np.random.default_rng(7)
    D = rng.uniform(0.0, 1.0, (12_500, 2, 16))
    D[17, 0, 3], D[5, 1, 1] = 256.0, -200.0
    ag, bg, mse = _nearest_rank_checks(orc, D)
    a, b, alpha, mse2 = orc.calibrate(D)
    assert alpha == 0.001 and int(np.argmin(mse)) == 1
    assert a == ag[1] and (b == bg[1]).all()
    np.testing.assert_array_equal(mse, mse2)
    # the two picks differ by one rank here (a continuous sample has no ties)
    s0 = np.sort(D[:, 0, :].ravel())
    assert bg[1, 0] == s0[199] != s0[200]


def test_calibrate_every_alpha_gamma(orc):
    """Same per-alpha checks on the gamma tables where alpha = 0 wins, with
    n = 40 x 16 = 640 per table (alpha n not an integer: ceil - 1 = floor)."""
    rng = np.random.default_rng(7)
    D = rng.gamma(2.0, 3.0, (40, 4, 16)) + np.arange(4)[None, :, None] * 10
    _nearest_rank_checks(orc, D)


def test_calibrate_constant_and_uniform(orc):
    """Constant tables: b = c, beta = 0, MSE 0.  Uniform entries:
    floor quantization error is U[0, 1/a), so MSE = (1/a)^2 / 3 (R5/R17)."""
    D = np.full((10, 3, 16), 4.25)
    a, b, alpha, mse = orc.calibrate(D)
    assert (b == 4.25).all() and mse.min() == 0.0
    rng = np.random.default_rng(11)
    D = rng.uniform(0, 100, (400, 2, 16))
    a, b, alpha, mse = orc.calibrate(D)
    b0 = D.min(axis=(0, 2))                       # alpha = 0: b_m = table minimum
    a0 = 255.0 / (D - b0[None, :, None]).max()    # a = 255 / max pooled residual
    assert mse[0] == pytest.approx((1 / a0) ** 2 / 3, rel=0.05)
    assert mse[[0, 1, 2]].min() == mse.min()      # small alphas win on light tails


# --------------------------------------------------------------------- scan O7
def test_scan_equals_onehot_matmul(orc):
    """P:L224-231 running total == one-hot(codes) x table contraction (numpy matmul)."""
    for n, M, nq in [(1, 1, 1), (37, 3, 5), (200, 16, 7), (64, 64, 3)]:
        codes = G.random_codes(n, M, n + M)
        ql = G.random_qluts(nq, M, nq + M)
        ref = one_hot(codes) @ ql.reshape(nq, M * 16).astype(np.int64).T
        np.testing.assert_array_equal(orc.scan(codes, ql), ref)


def test_scan_single_entry_and_spec(orc):
    """A table with one nonzero entry (q=1, m=2, k=5) pins the q/m/k indexing;
    S:L293: M=2, codes (1,2), tables 10 and 20 -> 30."""
    codes = G.random_codes(100, 4, 3)
    ql = np.zeros((3, 4, 16), np.uint8)
    ql[1, 2, 5] = 200
    out = orc.scan(codes, ql)
    np.testing.assert_array_equal(out[:, 1], np.where(codes[:, 2] == 5, 200, 0))
    assert (out[:, [0, 2]] == 0).all()
    ql2 = np.zeros((1, 2, 16), np.uint8)
    ql2[0, 0, 1], ql2[0, 1, 2] = 10, 20
    assert orc.scan(np.array([[1, 2]], np.uint8), ql2)[0, 0] == 30
    full = np.full((1, 64, 16), 255, np.uint8)
    assert orc.scan(G.random_codes(3, 64, 9), full).max() == 255 * 64


# --------------------------------------------------------------- topk O8 / O9
def _sorted_keys(acc, metric, base=0):
    v = acc.astype(np.uint64) if metric == 0 else (0xFFFF - acc.astype(np.int64)).astype(np.uint64)
    idx = np.arange(len(acc), dtype=np.uint64) + np.uint64(base)
    return np.sort((v << np.uint64(48)) | idx)


@pytest.mark.parametrize("metric", [0, 1])
def test_topk_matches_full_sort(orc, metric):
    """Top-k = prefix of the fully sorted keys (numpy sort), ties by lower index;
    k = n gives the argsort; k > n pads with UINT64_MAX."""
    n, M, nq = 500, 4, 6
    codes = G.random_codes(n, M, 70)
    ql = G.random_qluts(nq, M, 71, hi=8)          # heavy ties
    acc = orc.scan(codes, ql)
    for k in (1, 10, n):
        keys = orc.topk(codes, ql, k, metric, index_base=1000)
        for q in range(nq):
            np.testing.assert_array_equal(keys[q], _sorted_keys(acc[:, q], metric, 1000)[:k])
    kk = orc.topk(codes[:3], ql, 5, metric)
    assert (kk[:, 3:] == np.uint64(2**64 - 1)).all()
    v, idx = orc.keys_split(orc.topk(codes, ql, n, metric), metric)
    order = np.lexsort((np.arange(n), acc[:, 0] if metric == 0 else -acc[:, 0].astype(int)))
    np.testing.assert_array_equal(idx[0], order)
    np.testing.assert_array_equal(v[0], acc[order, 0])


def test_merge_of_partition_equals_whole(orc):
    n, M, nq, k = 1000, 8, 4, 10
    codes = G.random_codes(n, M, 80)
    ql = G.random_qluts(nq, M, 81, hi=16)
    whole = orc.topk(codes, ql, k, 0)
    bounds = [0, 8, 400, 401, 1000]
    parts = np.stack([orc.topk(codes[lo:hi], ql, k, 0, index_base=lo)
                      for lo, hi in zip(bounds[:-1], bounds[1:])])
    np.testing.assert_array_equal(orc.merge(parts), whole)


# ------------------------------------------------------------------ dequant O10
def test_dequant_is_sum_of_reconstructions(orc):
    """P:L286 + P:L291: the sum over tables of yhat = beta/a + b_m equals acc/a + sum b."""
    M, nq, n = 8, 3, 50
    codes = G.random_codes(n, M, 90)
    ql = G.random_qluts(nq, M, 91)
    a, b = np.float32(3.7), G.random_floats(M, 92)
    acc = orc.scan(codes, ql)
    per_entry = ql.astype(np.float64) / np.float64(a) + b.astype(np.float64)[None, :, None]
    ref = np.einsum("qmk,nmk->nq", per_entry, one_hot(codes).reshape(n, M, 16).astype(np.float64))
    np.testing.assert_allclose(orc.dequant(acc, a, b), ref, rtol=1e-12, atol=1e-10)


# -------------------------------------------------------------------- kmeans O2
def test_kmeans_exact_structure(orc):
    """16 tight, separated blobs seeded one per blob: k-means converges to the
    blob means (numpy mean), and 16 distinct points repeated give the points."""
    rng = np.random.default_rng(5)
    L, per = 3, 40
    centers = np.arange(16)[:, None] * 10.0 + np.zeros((16, L))
    pts = (centers[:, None, :] + rng.uniform(-1, 1, (16, per, L))).reshape(-1, L).astype(np.float32)
    init = np.arange(16)[None] * per
    C = orc.kmeans(pts, 1, init, iters=5)
    np.testing.assert_allclose(C[0], pts.reshape(16, per, L).astype(np.float64).mean(1), rtol=1e-12)
    rep = np.repeat(centers.astype(np.float32), 10, axis=0)
    C2 = orc.kmeans(rep, 1, (np.arange(16) * 10)[None], iters=3)
    np.testing.assert_array_equal(C2[0], centers)


def test_kmeans_matches_scipy_lloyd_and_monotone(orc):
    """Without empty clusters, 16 Lloyd iterations equal scipy kmeans2 with the
    same initial centroids (library routine); inertia is non-increasing."""
    X = G.rows(1, 1, 3000)
    M = 8
    L = 4
    init = G.kmeans_init_all(G.CONFIGS["c1"], len(X))
    C, inertia = orc.kmeans(X, M, init, iters=16, with_inertia=True)
    for m in range(M):
        sub = X[:, m * L:(m + 1) * L].astype(np.float64)
        ref, _ = kmeans2(sub, sub[init[m]].copy(), iter=16, minit="matrix", missing="raise")
        np.testing.assert_allclose(C[m], ref, rtol=1e-9, atol=1e-9)
        assert (np.diff(inertia[m]) <= 1e-9 * inertia[m][0]).all()


def test_kmeans_empty_cluster_takes_farthest(orc):
    """R8: an empty cluster takes the point farthest from its centroid."""
    pts = np.array([[0.0], [0.1], [0.2], [50.0]] + [[100.0 + i] for i in range(14)], np.float32)
    # centroids 0 and 1 both start at row 0 -> ties go to centroid 0, centroid 1
    # is empty; row 3 (50, equidistant from 0 and 100 -> centroid 0) is farthest
    init = np.array([[0, 0] + list(range(4, 18))])
    C = orc.kmeans(pts, 1, init, iters=1)
    assert C[0, 1, 0] == 50.0
    assert C[0, 0, 0] == pytest.approx((0.0 + float(np.float32(0.1)) + float(np.float32(0.2)) + 50.0) / 4, rel=1e-15)
    np.testing.assert_array_equal(C[0, 2:, 0], pts[4:, 0])


def test_kmeans_two_empty_clusters_take_distinct_rows(orc):
    """R8 with two clusters empty in one iteration: centroids 0, 1, 2 all
    start at row 0, so assignment ties give every nearby point to centroid 0
    and leave 1 and 2 empty.  In ascending k, centroid 1 takes the farthest
    point (row 3, 50: equidistant from 0 and 100, so assigned to centroid 0,
    distance 2500) and centroid 2 the farthest row NOT already taken this
    iteration (row 4, 30: distance 900) -- never row 3 twice."""
    vals = [0.0, 0.1, 0.2, 50.0, 30.0] + [100.0 + i for i in range(13)]
    pts = np.array(vals, np.float32)[:, None]
    init = np.array([[0, 0, 0] + list(range(5, 18))])
    C = orc.kmeans(pts, 1, init, iters=1)
    assert C[0, 1, 0] == 50.0 and C[0, 2, 0] == 30.0
    f = [float(np.float32(v)) for v in vals[:5]]
    assert C[0, 0, 0] == ((((f[0] + f[1]) + f[2]) + f[3]) + f[4]) / 5  # row-order sum (R8)
    np.testing.assert_array_equal(C[0, 3:, 0], pts[5:, 0])


# ------------------------------------------------------------ Lemmas 3 / 4
def test_lemmas_3_4(orc):
    """P:L319-325 with x_hat from the oracle encoder: zero violations over 1e4 pairs."""
    M, L = 8, 4
    C = centroid_bank(M, L, 61)
    X = G.random_floats((100, M * L), 62)
    Q = G.random_floats((100, M * L), 63)
    codes = orc.encode(X, C)
    xh = np.concatenate([C[m][codes[:, m]] for m in range(M)], axis=1).astype(np.float64)
    X64, Q64 = X.astype(np.float64), Q.astype(np.float64)
    r = np.linalg.norm(X64 - xh, axis=1)
    dots = np.abs(Q64 @ X64.T - Q64 @ xh.T)
    assert (dots <= np.linalg.norm(Q64, axis=1)[:, None] * r[None] + 1e-12).all()
    d1 = np.linalg.norm(Q64[:, None] - X64[None], axis=2)
    d2 = np.linalg.norm(Q64[:, None] - xh[None], axis=2)
    assert (np.abs(d1 - d2) <= r[None] + 1e-12).all()


# ------------------------------------------------- Bolt No Quantize (f3, O13/O14)
@pytest.mark.parametrize("metric", [0, 1])
def test_scan_f32_within_summation_bound_and_reconstruction(orc, metric):
    """O13 against the mathematics: the fp32 running sum of M fp32 table
    entries differs from the exact (fp64) sum of the same entries by at most
    (M - 1) u sum|entries| (u = 2^-24, recursive summation bound); and with
    the exact tables rounded to fp32, the scan of a vector's codes is its
    reconstruction's dense distance within that bound plus the rounding of
    the M entries."""
    M, L = 8, 4
    C = centroid_bank(M, L, 141)
    X = G.random_floats((64, M * L), 142)
    Q = G.random_floats((5, M * L), 143)
    codes = orc.encode(X, C)
    D64 = orc.luts(Q, C, metric)
    D32 = D64.astype(np.float32)
    got = orc.scan_f32(codes, D32).astype(np.float64)
    terms = np.stack([D32[:, m, :][:, codes[:, m]] for m in range(M)]).astype(np.float64)  # [M][nq][n]
    exact = terms.sum(0).T
    bound = (M - 1) * 2.0**-24 * np.abs(terms).sum(0).T
    assert (np.abs(got - exact) <= bound + 1e-30).all()
    xhat = np.concatenate([C[m][codes[:, m]] for m in range(M)], axis=1).astype(np.float64)
    Q64 = Q.astype(np.float64)
    dense = (((Q64[:, None, :] - xhat[None]) ** 2).sum(-1) if metric == 0 else Q64 @ xhat.T).T
    round_err = 2.0**-24 * np.abs(np.stack([D64[:, m, :][:, codes[:, m]] for m in range(M)])).sum(0).T
    assert (np.abs(got - dense) <= bound + round_err + 1e-12).all()


@pytest.mark.parametrize("metric", [0, 1])
def test_topk_f32_reduces_to_quantized_topk(orc, metric):
    """O14 against O8: with integer tables (exact in fp32, sums <= 255 M exact)
    the fp32 top-k ranks exactly as the u8 top-k -- same indices, same values
    -- including the heavy ties of small tables (lower index first)."""
    n, M, nq = 700, 8, 6
    codes = G.random_codes(n, M, 170)
    for hi in (4, 256):
        ql = G.random_qluts(nq, M, 171 + hi, hi=hi)
        for k in (1, 10, n, n + 5):
            ref_v, ref_i = orc.keys_split(orc.topk(codes, ql, k, metric, index_base=33), metric)
            v, i = orc.keys_split_f32(orc.topk_f32(codes, ql.astype(np.float32), k, metric, index_base=33), metric)
            np.testing.assert_array_equal(i, ref_i)
            ok = ref_i >= 0
            np.testing.assert_array_equal(v[ok], ref_v[ok].astype(np.float32))


def test_topk_f32_order_on_signed_values(orc):
    """R18 on negative / mixed-sign sums (dot tables): the keys sort as the
    floats do -- checked against numpy's stable argsort of the O13 sums."""
    n, M, nq = 300, 4, 3
    codes = G.random_codes(n, M, 180)
    luts = G.random_floats((nq, M, 16), 181, 3.0)
    s = orc.scan_f32(codes, luts)
    for metric in (0, 1):
        v, idx = orc.keys_split_f32(orc.topk_f32(codes, luts, n, metric), metric)
        for q in range(nq):
            order = np.argsort(s[:, q] if metric == 0 else -s[:, q], kind="stable")
            np.testing.assert_array_equal(idx[q], order)
            np.testing.assert_array_equal(v[q], s[order, q])
