"""GPU parity: the CUDA path (through the C ABI) against the fp64 CPU oracle on
identical seeded inputs.  Contract (SURVEY 8(c) / BASELINE.json north_star):
  * scan u16 sums, top-k keys (values, indices, order, lower-index ties), merge,
    pack/unpack: bit-exact;
  * fp32 tables: |gpu - oracle| <= 1e-4 * max|D(q)| per query;
  * quantized tables and codes: exact except near-ties (|t - rint(t)| < 1e-3, or
    relative centroid-distance gap < 1e-5), counted, cap 0.01 %;
  * dequant: |gpu - oracle| <= 2^-21 (|acc/a| + |sum b|).
"""
import numpy as np
import pytest
import torch

from synth import generators as G

pytestmark = pytest.mark.gpu

NEAR_TIE_CAP = 1e-4  # 0.01 %


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


def pack_on_gpu(bolt, flat):
    return bolt.pack_codes(dev(flat.astype(np.uint8)))


# --------------------------------------------------------------------- layout
@pytest.mark.parametrize("n,m", [(1, 1), (7, 3), (8, 16), (9, 16), (1001, 8), (4097, 64)])
def test_pack_unpack_layout_v1(bolt, orc, n, m):
    flat = G.random_codes(n, m, n * 7 + m)
    words = host(pack_on_gpu(bolt, flat))
    assert words.size == bolt.codes_words(n, m)
    np.testing.assert_array_equal(orc.unpack_v1(words, n, m), flat)      # O12 reads GPU layout
    np.testing.assert_array_equal(host(bolt.unpack_codes(dev(words), n, m)), flat)


# --------------------------------------------------------------------- encode
def _encode_check(bolt, orc, X, C):
    n = X.shape[0]
    m = C.shape[0]
    words = host(bolt.encode(dev(X), dev(C)))
    got = orc.unpack_v1(words, n, m)
    ref, gap = orc.encode(X, C, with_gap=True)
    diff = got != ref
    exempt = diff & (gap < 1e-5)
    assert (diff == exempt).all(), f"{(diff & ~exempt).sum()} non-tie code mismatches"
    assert exempt.sum() <= NEAR_TIE_CAP * diff.size + 1e-9, f"near-ties {exempt.sum()} over cap"
    return exempt.sum()


@pytest.mark.parametrize("n,m,L", [(1, 1, 1), (9, 2, 3), (513, 4, 4), (1000, 8, 4), (4099, 16, 8),
                                   (777, 32, 16), (300, 64, 2), (100, 5, 7)])
def test_encode_random(bolt, orc, n, m, L):
    X = G.random_floats((n, m * L), 1000 + n)
    C = G.random_floats((m, 16, L), 2000 + m)
    _encode_check(bolt, orc, X, C)


def test_encode_centroid_identity(bolt, orc):
    m, L = 16, 8
    C = G.random_floats((m, 16, L), 5)
    idx = np.random.default_rng(0).integers(0, 16, (1000, m))
    X = np.ascontiguousarray(np.concatenate([C[c][idx[:, c]] for c in range(m)], axis=1))
    got = orc.unpack_v1(host(bolt.encode(dev(X), dev(C))), 1000, m)
    np.testing.assert_array_equal(got, idx)


@pytest.mark.parametrize("seed,m,L", [(0, 16, 8), (1, 16, 8), (2, 16, 8),   # J = 128: 4 slabs per stage
                                       (0, 32, 8),                           # J = 256 (c4): 2 slabs
                                       (0, 32, 16), (1, 64, 8),              # J = 512 (c3): 2 column parts
                                       (0, 8, 16)])                          # J/M = 16 in one 128-float part
def test_encode_fast_equals_direct_near_ties(bolt, orc, seed, m, L):
    """The TMA-staged expanded-distance encoder (ENCODE_EXPANDED: ||c||^2 - 2 x.c ranking,
    rounding bound, direct fallback) returns the direct-difference kernel's
    codes bit for bit, on rows built at or near midpoints of centroid pairs
    (exact fp32 ties, 1e-5 .. 0.5 offsets) with c2-sized coordinates (0..255,
    where the expansion's rounding is largest), duplicated centroids and rows
    equal to centroids; and both agree with the oracle up to near-ties."""
    n = 60_000
    rng = np.random.default_rng(seed + 100 * m + L)
    C = rng.uniform(0, 255, (m, 16, L)).astype(np.float32)
    C[:4, 9] = C[:4, 4]                       # exact duplicate centroids in 4 codebooks
    C[m - 1, 15] = C[m - 1, 0]                # ... and in the last codebook (the last column part)
    a = rng.integers(0, 16, (n, m))
    b = rng.integers(0, 16, (n, m))
    mid = (C[np.arange(m)[None, :], a] + C[np.arange(m)[None, :], b]) / np.float32(2)
    scale = rng.choice(np.array([0, 0, 1e-5, 1e-3, 0.5], np.float32), size=(n, m, 1))
    X = (mid + scale * rng.standard_normal((n, m, L)).astype(np.float32)).astype(np.float32)
    X[: n // 10] = C[np.arange(m)[None, :], a[: n // 10]]  # rows on centroids
    X = np.ascontiguousarray(X.reshape(n, m * L))
    Xd, Cd = dev(X), dev(C)
    fast = host(bolt.encode(Xd, Cd, variant=bolt.ENCODE_EXPANDED))
    direct = host(bolt.encode(Xd, Cd, variant=bolt.ENCODE_DIRECT))
    np.testing.assert_array_equal(host(bolt.encode(Xd, Cd)), direct)
    # ragged row counts (partial TMA row blocks, partial groups)
    for nn in (1, 7, 63, 65, 511, 513, 4099):
        np.testing.assert_array_equal(host(bolt.encode(Xd[:nn], Cd, variant=bolt.ENCODE_EXPANDED)),
                                      host(bolt.encode(Xd[:nn], Cd, variant=bolt.ENCODE_DIRECT)))
    np.testing.assert_array_equal(fast, direct)
    _encode_check(bolt, orc, X[:5000], C)


# ------------------------------------------------------------------------ LUT
@pytest.mark.parametrize("metric", [0, 1])
@pytest.mark.parametrize("nq,m,L", [(1, 1, 1), (16, 8, 4), (33, 16, 8), (7, 32, 16), (5, 64, 3)])
def test_luts(bolt, orc, metric, nq, m, L):
    Q = G.random_floats((nq, m * L), 3000 + nq, scale=3.0)
    C = G.random_floats((m, 16, L), 4000 + m)
    ref = orc.luts(Q, C, metric)
    d64 = host(bolt.build_luts(dev(Q), dev(C), metric, f64=True))
    np.testing.assert_array_equal(d64, ref)       # same fp64 operations in the same order
    d32 = host(bolt.build_luts(dev(Q), dev(C), metric))
    tol = 1e-4 * np.abs(ref).reshape(nq, -1).max(axis=1)
    assert (np.abs(d32 - ref).reshape(nq, -1) <= tol[:, None]).all()


def _quant_params(m, seed, lo=-1.0, hi=1.0):
    rng = np.random.default_rng(seed)
    return np.float32(rng.uniform(3, 40)), rng.uniform(lo, hi, m).astype(np.float32)


@pytest.mark.parametrize("metric", [0, 1])
def test_quantize_fused_and_standalone(bolt, orc, metric):
    nq, m, L = 64, 16, 8
    Q = G.random_floats((nq, m * L), 11)
    C = G.random_floats((m, 16, L), 12)
    a, b = _quant_params(m, 13, *((-1, 5) if metric == 0 else (-3, 0)))
    D = orc.luts(Q, C, metric)
    ref, t = orc.quantize(D, a, b, with_t=True)
    got, f32 = bolt.build_quantized_luts(dev(Q), dev(C), metric, float(a), dev(b), return_f32=True)
    got = host(got)
    diff = got != ref
    near = np.abs(t - np.rint(t)) < 1e-3
    assert (diff <= near).all()
    assert diff.sum() <= NEAR_TIE_CAP * diff.size
    assert (0 < ref).any() and (ref < 255).any() and (ref == 0).any()
    # standalone quantize of the GPU fp32 tables: oracle promotes the same fp32 values
    d32 = host(f32)
    ref2 = orc.quantize(d32.astype(np.float64), a, b)
    np.testing.assert_array_equal(host(bolt.quantize_luts(dev(d32), float(a), dev(b))), ref2)


# ----------------------------------------------------------------------- scan
SCAN_SHAPES = [(1, 1, 1), (7, 2, 3), (8, 16, 1), (9, 16, 2), (1000, 8, 16), (4097, 16, 9),
               (1234, 17, 5), (513, 32, 8), (333, 33, 4), (2049, 64, 17), (100, 3, 8), (64, 4, 1)]


@pytest.mark.parametrize("n,m,nq", SCAN_SHAPES)
def test_scan_bitexact(bolt, orc, n, m, nq):
    flat = G.random_codes(n, m, n + 17 * m)
    ql = G.random_qluts(nq, m, nq + 31 * m)
    ref = orc.scan(flat, ql)
    got = host(bolt.scan(pack_on_gpu(bolt, flat), n, dev(ql)))
    np.testing.assert_array_equal(got, ref)


def test_scan_extremes(bolt, orc):
    n, m, nq = 999, 64, 3
    flat = G.random_codes(n, m, 1)
    ql = np.full((nq, m, 16), 255, np.uint8)
    ql[1] = 0
    ql[2, :, 15] = 255
    ql[2, :, :15] = 128
    got = host(bolt.scan(pack_on_gpu(bolt, flat), n, dev(ql)))
    np.testing.assert_array_equal(got, orc.scan(flat, ql))
    assert got[:, 0].max() == 255 * 64


def test_scan_dequant(bolt, orc):
    n, m, nq = 2001, 32, 40
    flat = G.random_codes(n, m, 2)
    ql = G.random_qluts(nq, m, 3)
    a, b = _quant_params(m, 4, -2, 1)
    acc = orc.scan(flat, ql)
    ref = orc.dequant(acc, a, b)
    bsum = float(np.sum(b.astype(np.float64)))
    got = host(bolt.scan_dequant(pack_on_gpu(bolt, flat), n, dev(ql), float(a), np.float32(bsum)))
    tol = 2.0 ** -21 * (np.abs(acc / np.float64(a)) + abs(bsum))
    assert (np.abs(got - ref) <= tol).all()


# tcgen05 full-output scan (one-hot x table contraction, all sums stored):
# ragged n (several 256-vector tiles + tail), nq across 256-query tiles
TC_SCAN_SHAPES = [(1, 8, 1), (300, 16, 70), (2049, 32, 257), (5000, 8, 513), (777, 16, 64), (70000, 16, 300)]


@pytest.mark.parametrize("n,m,nq", TC_SCAN_SHAPES)
def test_scan_tc_bitexact(bolt, orc, n, m, nq):
    flat = G.random_codes(n, m, n + 5 * m)
    ql = G.random_qluts(nq, m, nq + 7 * m)
    codes = pack_on_gpu(bolt, flat)
    got = host(bolt.scan(codes, n, dev(ql), variant=bolt.VARIANT_TC))
    np.testing.assert_array_equal(got, orc.scan(flat, ql))


def test_scan_dequant_tc(bolt, orc):
    n, m, nq = 3001, 32, 200
    flat = G.random_codes(n, m, 21)
    ql = G.random_qluts(nq, m, 22)
    a, b = _quant_params(m, 23, -2, 1)
    acc = orc.scan(flat, ql)
    ref = orc.dequant(acc, a, b)
    bsum = np.float32(np.sum(b.astype(np.float64)))
    codes = pack_on_gpu(bolt, flat)
    got = host(bolt.scan_dequant(codes, n, dev(ql), float(a), bsum, variant=bolt.VARIANT_TC))
    tol = 2.0 ** -21 * (np.abs(acc / np.float64(a)) + abs(float(bsum)))
    assert (np.abs(got - ref) <= tol).all()
    # same fmaf in both variants: bit-identical
    prmt = host(bolt.scan_dequant(codes, n, dev(ql), float(a), bsum, variant=bolt.VARIANT_PRMT))
    np.testing.assert_array_equal(got.view(np.uint32), prmt.view(np.uint32))


def test_scan_tc_strided_out(bolt, orc):
    """ldo > nq: only the first nq columns of each output row are written."""
    import torch
    n, m, nq, ldo = 1500, 16, 100, 130
    flat = G.random_codes(n, m, 31)
    ql = G.random_qluts(nq, m, 32)
    buf = torch.full((n, ldo), 0xBEEF, dtype=torch.uint16, device="cuda")
    codes, qd = pack_on_gpu(bolt, flat), dev(ql)
    # the binding takes a contiguous out; call the C ABI directly for a strided one
    bolt._lib.call("bolt_scan_ex", codes.data_ptr(), n, m, qd.data_ptr(), nq,
                   buf.data_ptr(), ldo, bolt.VARIANT_TC, torch.cuda.current_stream().cuda_stream)
    got = host(buf)
    np.testing.assert_array_equal(got[:, :nq], orc.scan(flat, ql))
    assert (got[:, nq:] == 0xBEEF).all()


# ---------------------------------------------------------------------- top-k
TOPK_CASES = [
    # n, m, nq, k, lut_hi (small -> many ties), index_base
    (1, 1, 1, 1, 256, 0),
    (5, 4, 3, 10, 256, 0),            # k > n: padding
    (100, 8, 16, 10, 4, 0),
    (1000, 16, 9, 1, 256, 5),
    (4097, 16, 33, 10, 16, 0),
    (2500, 8, 20, 32, 8, 123456),
    (3000, 32, 7, 33, 256, 0),
    (5000, 16, 5, 100, 32, 0),
    (20000, 16, 8, 128, 256, 2**40),
    (65537, 16, 3, 10, 8, 0),
    (10000, 64, 4, 64, 256, 0),
    # small-batch query tiles of 2 and 4 (several tiles), the batched PRMT
    # kernel (nq >= 64), an index base at the top of the 48-bit range
    (30001, 16, 6, 10, 16, 0),
    (30001, 16, 10, 7, 256, 0),
    (12345, 8, 12, 20, 256, 0),
    (9000, 16, 70, 10, 8, 0),
    (4000, 32, 11, 10, 256, 2**48 - 4001),
]


@pytest.mark.parametrize("metric", [0, 1])
@pytest.mark.parametrize("n,m,nq,k,hi,base", TOPK_CASES)
def test_topk_prmt_bitexact(bolt, orc, metric, n, m, nq, k, hi, base):
    flat = G.random_codes(n, m, n + m + k)
    ql = G.random_qluts(nq, m, nq + k, hi=hi)
    ref = orc.topk(flat, ql, k, metric, index_base=base)
    got = host(bolt.topk(pack_on_gpu(bolt, flat), n, dev(ql), k, metric, index_base=base,
                         variant=bolt.VARIANT_PRMT))
    np.testing.assert_array_equal(got, ref)


TC_CASES = [
    # n, m, nq, k, lut_hi, index_base -- tcgen05 variant: m in {8, 16, 32}, k <= 32
    (1, 16, 1, 1, 256, 0),
    (5, 8, 3, 10, 256, 0),
    (300, 16, 129, 10, 4, 7),          # two query tiles, heavy ties, ragged tile
    (4097, 16, 33, 10, 16, 0),
    (2500, 8, 200, 32, 8, 123456),
    (3000, 32, 7, 17, 256, 0),
    (65537, 16, 130, 10, 8, 0),        # several row partitions + tail
    (20000, 32, 64, 30, 256, 2**40),
    (20000, 16, 64, 32, 256, 2**40),
    (100000, 16, 300, 10, 256, 0),
    # single-CTA 128-query tiles (nq <= 128, m <= 16, k <= 32)
    (65537, 8, 128, 12, 8, 0),
    (1_000_000, 16, 100, 10, 256, 5),
    (777, 16, 24, 4, 3, 0),
]


@pytest.mark.parametrize("metric", [0, 1])
@pytest.mark.parametrize("n,m,nq,k,hi,base", TC_CASES)
def test_topk_tc_bitexact(bolt, orc, metric, n, m, nq, k, hi, base):
    """tcgen05 one-hot x table contraction: same integers, same keys."""
    flat = G.random_codes(n, m, n + m + k + 1)
    ql = G.random_qluts(nq, m, nq + k + 1, hi=hi)
    ref = orc.topk(flat, ql, k, metric, index_base=base)
    got = host(bolt.topk(pack_on_gpu(bolt, flat), n, dev(ql), k, metric, index_base=base,
                         variant=bolt.VARIANT_TC))
    np.testing.assert_array_equal(got, ref)


# 2:4-sparse tcgen05 (f2): vectors on M (compressed one-hot + TMEM metadata),
# 224 queries per tile on N; k <= 32 (k <= 16 for m = 32)
SP_CASES = [
    # n, m, nq, k, lut_hi, index_base
    (1, 16, 1, 1, 256, 0),
    (5, 8, 3, 10, 256, 0),              # k > n: padding
    (300, 16, 225, 10, 4, 7),           # two query tiles, heavy ties, ragged tile
    (4097, 16, 33, 10, 16, 0),
    (2500, 8, 200, 32, 8, 123456),
    (3000, 32, 7, 16, 256, 0),
    (65537, 16, 449, 10, 8, 0),         # several row partitions + tail, three query tiles
    (20000, 32, 64, 12, 256, 2**40),
    (20000, 16, 230, 32, 256, 2**40),
    (100000, 16, 700, 10, 256, 0),
    (1_000_000, 16, 300, 10, 256, 5),
    (777, 8, 24, 4, 3, 0),
    (1_000_003, 32, 250, 10, 256, 0),
]


@pytest.mark.parametrize("metric", [0, 1])
@pytest.mark.parametrize("n,m,nq,k,hi,base", SP_CASES)
def test_topk_sp_bitexact(bolt, orc, metric, n, m, nq, k, hi, base):
    """Sparse one-hot x table contraction: same integers, same keys."""
    flat = G.random_codes(n, m, n + m + k + 3)
    ql = G.random_qluts(nq, m, nq + k + 3, hi=hi)
    ref = orc.topk(flat, ql, k, metric, index_base=base)
    got = host(bolt.topk(pack_on_gpu(bolt, flat), n, dev(ql), k, metric, index_base=base,
                         variant=bolt.VARIANT_SP))
    np.testing.assert_array_equal(got, ref)


# 32 < k <= 128 on the tensor cores: lists of 32 merged, verified, and the
# flagged queries redone exactly (the constant-table and few-partition cases
# force the fallback; the large random case mostly does not)
# (n, m, nq, k, table max): 1M rows give 488 lists of 32 per query (more
# lists than k: the merge's heads bound), the others fewer lists than k
TC_LARGE_K = [(3000, 16, 40, 100, 256), (70_000, 16, 30, 64, 256), (5000, 8, 33, 128, 4), (200_000, 32, 25, 100, 256),
              (1_000_000, 16, 24, 100, 256), (1_000_000, 16, 26, 40, 16)]


@pytest.mark.parametrize("metric", [0, 1])
@pytest.mark.parametrize("n,m,nq,k,hi", TC_LARGE_K)
def test_topk_tc_large_k(bolt, orc, metric, n, m, nq, k, hi):
    flat = G.random_codes(n, m, n + k)
    ql = G.random_qluts(nq, m, nq + k, hi=hi)
    got = host(bolt.topk(pack_on_gpu(bolt, flat), n, dev(ql), k, metric, index_base=7, variant=bolt.VARIANT_TC))
    np.testing.assert_array_equal(got, orc.topk(flat, ql, k, metric, index_base=7))


def test_topk_tc_large_k_all_ties(bolt, orc):
    n, m, nq, k = 20_000, 16, 26, 100
    flat = G.random_codes(n, m, 3)
    ql = np.full((nq, m, 16), 9, np.uint8)
    got = host(bolt.topk(pack_on_gpu(bolt, flat), n, dev(ql), k, 0, variant=bolt.VARIANT_TC))
    np.testing.assert_array_equal(got, orc.topk(flat, ql, k, 0))


def test_topk_constant_tables_all_ties(bolt, orc):
    """Every distance equal: the answer is the k lowest indices."""
    n, m, nq, k = 3001, 16, 4, 50
    flat = G.random_codes(n, m, 9)
    ql = np.full((nq, m, 16), 7, np.uint8)
    for metric in (0, 1):
        got = host(bolt.topk(pack_on_gpu(bolt, flat), n, dev(ql), k, metric, variant=bolt.VARIANT_PRMT))
        np.testing.assert_array_equal(got, orc.topk(flat, ql, k, metric))
        v, idx = bolt.keys_split(dev(got), metric)
        np.testing.assert_array_equal(host(idx)[0], np.arange(k))


@pytest.mark.parametrize("w,nq,k", [(1, 3, 10), (5, 7, 10), (36, 50, 10), (40, 3, 128), (160, 20, 10),
                                     (256, 4, 12), (257, 4, 5), (300, 2, 32)])
def test_merge_matches_sorted_union(bolt, w, nq, k):
    """bolt_topk_merge = the k smallest keys of the union of the w sorted lists
    (warp-per-query kernel for w <= 256, block tournament above), with padded
    list tails, a fully padded list and a query whose lists are all padding."""
    r = np.random.default_rng([7, w, nq, k])
    keys = np.sort(r.integers(0, 2**62, (w, nq, k), dtype=np.int64), axis=2).view(np.uint64)
    mx = np.iinfo(np.uint64).max
    keys[0, :, k // 2:] = mx
    keys[w - 1, 0, :] = mx
    keys[:, nq - 1, :] = mx if nq > 1 else keys[:, nq - 1, :]
    got = host(bolt.topk_merge(dev(keys)))
    exp = np.sort(keys.transpose(1, 0, 2).reshape(nq, -1), axis=1)[:, :k]
    np.testing.assert_array_equal(got, exp)


def test_merge_and_split(bolt, orc):
    n, m, nq, k = 6000, 8, 12, 20
    flat = G.random_codes(n, m, 21)
    ql = G.random_qluts(nq, m, 22, hi=16)
    bounds = [0, 8, 1600, 1608, 4000, 6000]
    parts = []
    for lo, hi_ in zip(bounds[:-1], bounds[1:]):
        codes = pack_on_gpu(bolt, flat[lo:hi_])
        parts.append(bolt.topk(codes, hi_ - lo, dev(ql), k, 0, index_base=lo))
    merged = host(bolt.topk_merge(torch.stack(parts)))
    np.testing.assert_array_equal(merged, orc.topk(flat, ql, k, 0))
    np.testing.assert_array_equal(merged, orc.merge(np.stack([host(p) for p in parts])))
    for metric in (0, 1):
        keys = orc.topk(flat, ql, k, metric)
        v, idx = bolt.keys_split(dev(keys), metric)
        rv, ridx = orc.keys_split(keys, metric)
        np.testing.assert_array_equal(host(v), rv)
        np.testing.assert_array_equal(host(idx), ridx)


# ------------------------------------------------------------ configs (c1)
@pytest.fixture(scope="module")
def c1_model(orc):
    cfg = G.CONFIGS["c1"]
    X = G.database(cfg)
    init = G.kmeans_init_all(cfg, len(X))
    C = orc.fit(X, cfg.m, init, cfg.kmeans_iters)
    calib = G.calibration(cfg, X)
    params = {mt: orc.fit_quantizer(calib, C, mt) for mt in cfg.metrics}
    return cfg, X, C, params


@pytest.mark.parametrize("metric", [0, 1])
def test_c1_end_to_end(bolt, orc, c1_model, metric):
    """BASELINE c1: encode, fused tables, full N x Q u16 output, top-10."""
    cfg, X, C, params = c1_model
    a, b, _ = params[metric]
    Q = G.queries(cfg)
    codes = bolt.encode(dev(X), dev(C))
    _encode_check(bolt, orc, X, C)
    gcodes = orc.unpack_v1(host(codes), cfg.n, cfg.m)
    D = orc.luts(Q, C, metric)
    ref_q, t = orc.quantize(D, a, b, with_t=True)
    ql = host(bolt.build_quantized_luts(dev(Q), dev(C), metric, float(a), dev(b)))
    assert ((ql != ref_q) <= (np.abs(t - np.rint(t)) < 1e-3)).all()
    out = host(bolt.scan(codes, cfg.n, dev(ql)))
    np.testing.assert_array_equal(out, orc.scan(gcodes, ql))
    keys = host(bolt.topk(codes, cfg.n, dev(ql), 10, metric))
    np.testing.assert_array_equal(keys, orc.topk(gcodes, ql, 10, metric))


def test_search_host_matches_device_path(bolt, orc, c1_model):
    cfg, X, C, params = c1_model
    a, b, _ = params[0]
    Q = G.queries(cfg)
    hs = bolt.HostSearch(cfg.n, cfg.j, cfg.m, cfg.nq, 10)
    keys_h = torch.empty((cfg.nq, 10), dtype=torch.uint64).pin_memory()
    hs(torch.from_numpy(X).pin_memory(), torch.from_numpy(Q).pin_memory(), dev(C), 0, float(a), dev(b), keys_h)
    torch.cuda.synchronize()
    codes = bolt.encode(dev(X), dev(C))
    ql = bolt.build_quantized_luts(dev(Q), dev(C), 0, float(a), dev(b))
    np.testing.assert_array_equal(keys_h.numpy(), host(bolt.topk(codes, cfg.n, ql, 10, 0)))


@pytest.mark.parametrize("chunks", [2, 3, 7])
def test_host_search_pipelined(bolt, orc, c1_model, chunks):
    """The copy/compute-overlapped host search returns the same keys as the
    single-stream one (block top-k lists merged; ragged last block)."""
    cfg, X, C, params = c1_model
    a, b, _ = params[0]
    Q = G.queries(cfg)
    Xh, Qh = torch.from_numpy(X).pin_memory(), torch.from_numpy(Q).pin_memory()
    k1 = torch.empty((cfg.nq, 10), dtype=torch.uint64).pin_memory()
    k2 = torch.empty((cfg.nq, 10), dtype=torch.uint64).pin_memory()
    bolt.HostSearch(cfg.n, cfg.j, cfg.m, cfg.nq, 10)(Xh, Qh, dev(C), 0, float(a), dev(b), k1)
    hs = bolt.HostSearch(cfg.n, cfg.j, cfg.m, cfg.nq, 10, chunks=chunks)
    for _ in range(2):  # back to back: the second call's copies must wait for the first's compute
        hs(Xh, Qh, dev(C), 0, float(a), dev(b), k2)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(k2.numpy(), k1.numpy())
    codes = bolt.encode(dev(X), dev(C))
    ql = bolt.build_quantized_luts(dev(Q), dev(C), 0, float(a), dev(b))
    np.testing.assert_array_equal(k1.numpy(), orc.topk(orc.unpack_v1(host(codes), cfg.n, cfg.m), host(ql), 10, 0))


# ------------------------------------------- c2 / c3 at full size (all queries)
def _e2e_trace(orc, X, Q, C, a, b, metric, gcodes, qlg, keys_g, k):
    """End-to-end parity from raw X and Q (SURVEY 8(c) last contract row):
    the oracle's own pipeline -- O3 encode, O4 tables, O6 quantize, O8 top-k
    -- against the GPU's keys.  Every difference must trace to an exempted
    near-tie upstream: a query whose tables differ (|t - rint t| < 1e-3), or a
    row whose code differs (relative centroid gap < 1e-5) inside one of the
    two lists.  Returns (key overlap, queries differing, table near-ties,
    code near-ties)."""
    ocodes, gap = orc.encode(X, C, with_gap=True)
    dcode = gcodes != ocodes
    assert (dcode <= (gap < 1e-5)).all(), "code mismatch that is not a near-tie"
    assert dcode.sum() <= NEAR_TIE_CAP * dcode.size
    D = orc.luts(Q, C, metric)
    qlo, t = orc.quantize(D, a, b, with_t=True)
    dtab = qlg != qlo
    assert (dtab <= (np.abs(t - np.rint(t)) < 1e-3)).all(), "table mismatch that is not a near-tie"
    assert dtab.sum() <= NEAR_TIE_CAP * dtab.size
    keys_o = orc.topk(ocodes, qlo, k, metric)            # the oracle alone, from X and Q
    keys_mid = orc.topk(ocodes, qlg, k, metric)          # oracle codes, GPU tables
    qtab = dtab.reshape(len(Q), -1).any(axis=1)
    a_diff = (keys_o != keys_mid).any(axis=1)
    assert (a_diff <= qtab).all(), "a top-k difference with identical tables and codes"
    rows_bad = set(np.flatnonzero(dcode.any(axis=1)).tolist())
    _, i_mid = orc.keys_split(keys_mid, metric)
    _, i_g = orc.keys_split(keys_g, metric)
    for q in np.flatnonzero((keys_mid != keys_g).any(axis=1)):
        involved = set(i_mid[q].tolist()) | set(i_g[q].tolist())
        assert involved & rows_bad, f"query {q}: differs with no near-tie code in either list"
    _, i_o = orc.keys_split(keys_o, metric)
    overlap = np.mean([len(set(i_o[q]) & set(i_g[q])) / k for q in range(len(Q))])
    ndiff = int((keys_o != keys_g).any(axis=1).sum())
    print(f"e2e: key overlap {overlap:.6f}, {ndiff} of {len(Q)} queries differ; near-ties: "
          f"{int(dtab.sum())} table entries, {int(dcode.sum())} codes")
    return overlap, ndiff, int(dtab.sum()), int(dcode.sum())


@pytest.mark.slow
def test_c2_full_size_all_queries(bolt, orc):
    """BASELINE c2 (N=1M, J=128, M=16, Q=10k, top-10) in the launch configuration
    bench.py times: ALL 10,000 queries' keys bit-exact against the oracle's
    scan of the full GPU code set (read with O12), plus the end-to-end trace
    from raw X and Q."""
    cfg = G.CONFIGS["c2"]
    X = G.database(cfg)
    train = G.training(cfg, 20_000)
    init = G.kmeans_init_all(cfg, len(train))
    C = orc.fit(train, cfg.m, init, 4)
    a, b, _ = orc.fit_quantizer(G.calibration(cfg, train)[:200], C, 0)
    Q = G.queries(cfg)
    Xd, Qd = dev(X), dev(Q)
    codes = bolt.encode(Xd, dev(C))
    ql = bolt.build_quantized_luts(Qd, dev(C), 0, float(a), dev(b))
    assert bolt.topk_plan(cfg.n, cfg.m, cfg.nq, cfg.k)[0] == "tc"
    keys = host(bolt.topk(codes, cfg.n, ql, cfg.k, 0))
    gcodes = orc.unpack_v1(host(codes), cfg.n, cfg.m)
    qlh = host(ql)
    np.testing.assert_array_equal(keys, orc.topk(gcodes, qlh, cfg.k, 0))
    _e2e_trace(orc, X, Q, C, a, b, 0, gcodes, qlh, keys, cfg.k)


@pytest.mark.slow
def test_c3_full_size_all_queries(bolt, orc):
    """BASELINE c3 (N=1M, J=512, M=32, Q=1k, dot product, top-10 MIPS) in the
    bench launch configuration: all 1,000 queries bit-exact against the
    oracle over the full GPU code set, plus the end-to-end trace."""
    cfg = G.CONFIGS["c3"]
    X = G.database(cfg)
    train = G.training(cfg, 10_000)
    C = orc.fit(train, cfg.m, G.kmeans_init_all(cfg, len(train)), 3)
    a, b, _ = orc.fit_quantizer(G.calibration(cfg, train)[:200], C, 1)
    Q = G.queries(cfg)
    codes = bolt.encode(dev(X), dev(C))
    ql = bolt.build_quantized_luts(dev(Q), dev(C), 1, float(a), dev(b))
    assert bolt.topk_plan(cfg.n, cfg.m, cfg.nq, cfg.k)[0] == "tc"
    keys = host(bolt.topk(codes, cfg.n, ql, cfg.k, 1))
    gcodes = orc.unpack_v1(host(codes), cfg.n, cfg.m)
    qlh = host(ql)
    np.testing.assert_array_equal(keys, orc.topk(gcodes, qlh, cfg.k, 1))
    _e2e_trace(orc, X, Q, C, a, b, 1, gcodes, qlh, keys, cfg.k)


@pytest.mark.slow
def test_c4_full_size_sampled(bolt, orc):
    """BASELINE c4 (A 100k x 256 encoded, B 256 x 1024 as queries, fused
    dequantised fp32 output [100k][1024]) in the bench launch configuration
    (tcgen05 full output, TMA stores): the whole u16 sum matrix is exact and
    sampled rows of the fp32 output match the oracle's dequantisation."""
    cfg = G.CONFIGS["c4"]
    X = G.database(cfg)
    Q = G.queries(cfg)
    C = orc.fit(X[:20_000], cfg.m, G.kmeans_init_all(cfg, 20_000), 3)
    a, b, _ = orc.fit_quantizer(G.calibration(cfg, X)[:200], C, 1)
    codes = bolt.encode(dev(X), dev(C))
    ql = bolt.build_quantized_luts(dev(Q), dev(C), 1, float(a), dev(b))
    gcodes = orc.unpack_v1(host(codes), cfg.n, cfg.m)
    qlh = host(ql)
    acc = host(bolt.scan(codes, cfg.n, ql))
    np.testing.assert_array_equal(acc, orc.scan(gcodes, qlh))
    bsum = float(np.sum(b.astype(np.float64)))
    out = host(bolt.scan_dequant(codes, cfg.n, ql, float(a), np.float32(bsum)))
    rows = np.random.default_rng(5).choice(cfg.n, 2000, replace=False)
    ref = orc.dequant(acc[rows], float(a), b)
    tol = 2.0**-21 * (np.abs(acc[rows] / np.float64(a)) + abs(bsum))
    assert (np.abs(out[rows] - ref) <= tol).all()


# ------------------------------------- c5 / sweep: device-generated database
def test_c5_device_rows_sampled(bolt, orc):
    """c5's rows come from the GPU generator (synth/gen_gpu.cu); a slice far
    into the 1e8-row database is copied to the host, where the oracle encodes
    it and scans it for small query batches (the small-batch kernel, several
    partial lists) and a tcgen05-sized batch."""
    import torch
    from synth import gpu as sg
    cfg2 = G.CONFIGS["c2"]
    r0, n = 99_900_000, 100_000  # 1e5 rows re-encoded by the oracle
    X = torch.empty((n, 128), dtype=torch.float32, device="cuda")
    sg.c5_rows(r0, n, dev(G.c5_means()), X)
    Xh = host(X)
    assert Xh.min() >= 0 and Xh.max() <= 255 and (Xh == np.rint(Xh)).all()
    assert 40 < Xh.mean() < 90 and len(np.unique(Xh[:, 0])) > 100  # mixture of clipped normals
    train = G.training(cfg2, 20_000)
    C = orc.fit(train, cfg2.m, G.kmeans_init_all(cfg2, len(train)), 3)
    a, b, _ = orc.fit_quantizer(G.calibration(cfg2, train)[:200], C, 0)
    codes = bolt.encode(X, dev(C))
    gcodes = orc.unpack_v1(host(codes), n, cfg2.m)
    ref, gap = orc.encode(Xh, C, with_gap=True)
    d = gcodes != ref
    assert (d <= (gap < 1e-5)).all() and d.sum() <= NEAR_TIE_CAP * d.size
    Q = G.queries(G.CONFIGS["c5"], 70)
    for nq, variant in ((1, bolt.VARIANT_AUTO), (5, bolt.VARIANT_AUTO), (70, bolt.VARIANT_TC)):
        ql = bolt.build_quantized_luts(dev(Q[:nq]), dev(C), 0, float(a), dev(b))
        keys = host(bolt.topk(codes, n, ql, 10, 0, index_base=r0, variant=variant))
        np.testing.assert_array_equal(keys, orc.topk(gcodes, host(ql), 10, 0, index_base=r0))


@pytest.mark.slow
def test_c5_full_size_sampled(bolt, orc):
    """BASELINE c5 on one GPU in bench.py's launch configuration: the 1e8-row
    device-generated database encoded in 1M-row chunks, Q = 65,536, top-100
    (tcgen05 lists of 32 over 382 partitions, merged and verified); the oracle
    checks 64 sampled queries over the full 800 MB of GPU codes (read with O12)."""
    import torch
    from synth import gpu as sg
    cfg2, cfg5 = G.CONFIGS["c2"], G.CONFIGS["c5"]
    n, m = cfg5.n, cfg2.m
    train = G.training(cfg2, 20_000)
    C = orc.fit(train, m, G.kmeans_init_all(cfg2, len(train)), 3)
    a, b, _ = orc.fit_quantizer(G.calibration(cfg2, train)[:200], C, 0)
    Cd, mu = dev(C), dev(G.c5_means())
    codes = torch.empty(bolt.codes_words(n, m), dtype=torch.uint32, device="cuda")
    chunk = 1 << 20
    X = torch.empty((chunk, 128), dtype=torch.float32, device="cuda")
    for r0 in range(0, n, chunk):
        rows = min(chunk, n - r0)
        sg.c5_rows(r0, rows, mu, X[:rows])
        w0 = r0 // 8 * m
        bolt.encode(X[:rows], Cd, out=codes[w0:w0 + bolt.codes_words(rows, m)])
    del X
    ql = bolt.build_quantized_luts(dev(G.queries(cfg5)), Cd, 0, float(a), dev(b))
    assert bolt.topk_plan(n, m, cfg5.nq, cfg5.k)[0] == "tc"
    keys = host(bolt.topk(codes, n, ql, cfg5.k, 0))
    qs = np.random.default_rng(5).choice(cfg5.nq, 64, replace=False)  # 64 sampled queries
    qlh = host(ql[torch.from_numpy(qs).cuda()])
    gcodes = orc.unpack_v1(host(codes), n, m)
    np.testing.assert_array_equal(keys[qs], orc.topk(gcodes, qlh, cfg5.k, 0))


# ------------------------------- swapped tcgen05 top-k (small query batches)
TCS_SHAPES = [(3000, 16, 1, 10), (70_000, 16, 24, 10), (5003, 8, 33, 32), (20_000, 32, 64, 5), (9000, 16, 100, 1),
              (130_001, 16, 128, 16), (257, 8, 65, 20), (1, 16, 3, 4)]


@pytest.mark.parametrize("metric", [0, 1])
@pytest.mark.parametrize("n,m,nq,k", TCS_SHAPES)
def test_topk_tcs_bit_exact(bolt, orc, metric, n, m, nq, k):
    """Vectors on the MMA's M side, queries on N (32/64/128): bit-exact keys
    for ragged n (partial tiles, several partitions), nq inside a query tile,
    k up to 32, both metrics."""
    flat = G.random_codes(n, m, 500 + n)
    ql = G.random_qluts(nq, m, 501 + nq)
    got = host(bolt.topk(pack_on_gpu(bolt, flat), n, dev(ql), k, metric, index_base=5, variant=bolt.VARIANT_TCS))
    np.testing.assert_array_equal(got, orc.topk(flat, ql, k, metric, index_base=5))


def test_topk_tcs_ties_and_model_tables(bolt, orc):
    n, m, nq = 40_000, 16, 20
    flat = G.random_codes(n, m, 77)
    for hi in (2, 16):
        ql = G.random_qluts(nq, m, 78 + hi, hi=hi)
        for metric in (0, 1):
            got = host(bolt.topk(pack_on_gpu(bolt, flat), n, dev(ql), 32, metric, variant=bolt.VARIANT_TCS))
            np.testing.assert_array_equal(got, orc.topk(flat, ql, 32, metric))
    cfg = G.CONFIGS["c2"]
    X = G.database(cfg, 50_000)
    train = G.training(cfg, 4000)
    C = orc.fit(train, cfg.m, G.kmeans_init_all(cfg, len(train)), 2)
    a, b, _ = orc.fit_quantizer(G.calibration(cfg, train)[:100], C, 0)
    codes = bolt.encode(dev(X), dev(C))
    ql = bolt.build_quantized_luts(dev(G.queries(cfg, 40)), dev(C), 0, float(a), dev(b))
    got = host(bolt.topk(codes, 50_000, ql, 10, 0, variant=bolt.VARIANT_TCS))
    np.testing.assert_array_equal(got, orc.topk(orc.unpack_v1(host(codes), 50_000, cfg.m), host(ql), 10, 0))


# --------------------------------------------- Bolt No Quantize (f3, O13/O14)
F32_SHAPES = [(1, 1, 1), (300, 8, 5), (1001, 16, 33), (4099, 32, 64), (257, 64, 7), (5000, 5, 40)]


@pytest.mark.parametrize("n,m,nq", F32_SHAPES)
def test_scan_f32_bit_exact(bolt, orc, n, m, nq):
    """Same fp32 tables and codes: fp32 totals bit-identical to O13 (fp32,
    ascending m); ragged n (partial groups), nq (partial query tiles), odd m."""
    flat = G.random_codes(n, m, 300 + n)
    luts = G.random_floats((nq, m, 16), 301 + nq, 10.0)
    got = host(bolt.scan_f32(pack_on_gpu(bolt, flat), n, dev(luts)))
    np.testing.assert_array_equal(got, orc.scan_f32(flat, luts))


@pytest.mark.parametrize("n,m,nq", [(5000, 16, 40), (3001, 64, 7), (999, 5, 33)])
def test_scan_f32_within_fp64_bound(bolt, n, m, nq):
    """The GPU's No-Quantize sums against the exact (fp64) sum of the same fp32
    entries -- not against O13's fp32 order: the recursive-summation bound
    |fl(sum) - sum| <= gamma_{M-1} sum|entries|, gamma_j = j u / (1 - j u),
    u = 2^-24 (M terms summed from 0.0f, the first addition exact)."""
    flat = G.random_codes(n, m, 600 + n)
    luts = G.random_floats((nq, m, 16), 601 + nq, 10.0)
    got = host(bolt.scan_f32(pack_on_gpu(bolt, flat), n, dev(luts))).astype(np.float64)
    terms = np.stack([luts[:, c, :][:, flat[:, c]] for c in range(m)]).astype(np.float64)  # [M][nq][n]
    exact = terms.sum(0).T
    u = 2.0 ** -24
    gamma = (m - 1) * u / (1 - (m - 1) * u)
    bound = gamma * np.abs(terms).sum(0).T
    assert (np.abs(got - exact) <= bound).all()
    assert (got != exact).any()  # fp32 rounding is really exercised


@pytest.mark.parametrize("metric", [0, 1])
@pytest.mark.parametrize("n,m,nq,k", [(5000, 16, 40, 10), (777, 8, 3, 32), (20, 4, 70, 30), (100_000, 16, 33, 1),
                                      (3, 8, 2, 10)])
def test_topk_f32_bit_exact(bolt, orc, metric, n, m, nq, k):
    flat = G.random_codes(n, m, 400 + n)
    luts = G.random_floats((nq, m, 16), 401 + nq, 10.0)
    if metric == 0:
        luts = np.abs(luts)  # distances
    keys = bolt.topk_f32(pack_on_gpu(bolt, flat), n, dev(luts), k, metric, index_base=9)
    ref = orc.topk_f32(flat, luts, k, metric, index_base=9)
    np.testing.assert_array_equal(host(keys), ref)
    v, i = bolt.keys_split_f32(keys, metric)
    rv, ri = orc.keys_split_f32(ref, metric)
    np.testing.assert_array_equal(host(i), ri)
    np.testing.assert_array_equal(host(v)[ri >= 0], rv[ri >= 0])


def test_topk_f32_ties_and_tables_from_model(bolt, orc):
    """Integer tables (heavy ties; lower index first) and the model's own fp32
    tables (build_luts) fed to both sides."""
    n, m, nq = 3000, 16, 12
    flat = G.random_codes(n, m, 17)
    luts = G.random_qluts(nq, m, 18, hi=3).astype(np.float32)
    np.testing.assert_array_equal(host(bolt.topk_f32(pack_on_gpu(bolt, flat), n, dev(luts), 20, 0)),
                                  orc.topk_f32(flat, luts, 20, 0))
    cfg = G.CONFIGS["c2"]
    X = G.database(cfg, 5000)
    train = G.training(cfg, 4000)
    C = orc.fit(train, cfg.m, G.kmeans_init_all(cfg, len(train)), 2)
    codes = bolt.encode(dev(X), dev(C))
    D = bolt.build_luts(dev(G.queries(cfg, 9)), dev(C), 0)
    np.testing.assert_array_equal(host(bolt.topk_f32(codes, 5000, D, 10, 0)),
                                  orc.topk_f32(orc.unpack_v1(host(codes), 5000, cfg.m), host(D), 10, 0))


# ------------------------------------------- streaming encode-on-write (f4)
@pytest.mark.parametrize("pieces", [[1, 7, 8, 3, 500, 1, 2000, 9, 13], [8, 8, 16], [5], [3, 3, 3, 3, 3, 3, 3, 3, 3]])
def test_encode_append_equals_encode(bolt, orc, pieces):
    """Appending rows in pieces (partial layout-v1 groups included) gives the
    codes of encoding all rows at once, bit for bit, and those match the
    oracle up to near-ties."""
    import torch
    cfg = G.CONFIGS["c2"]
    n = sum(pieces)
    X = G.database(cfg, n, start=11)
    train = G.training(cfg, 4000)
    C = orc.fit(train, cfg.m, G.kmeans_init_all(cfg, len(train)), 2)
    whole = host(bolt.encode(dev(X), dev(C)))
    buf = torch.full((bolt.codes_words(n, cfg.m),), 0xFFFFFFFF, dtype=torch.int64).to(torch.uint32).cuda()
    n_old = 0
    for p in pieces:
        bolt.encode_append(dev(X[n_old:n_old + p]), dev(C), buf, n_old)
        n_old += p
    got = host(buf)
    # words of the last group past row n: encode writes zero nibbles there
    np.testing.assert_array_equal(got, whole)
    _encode_check(bolt, orc, X, C)


def test_code_buffer_grows_and_searches(bolt, orc):
    import torch
    cfg = G.CONFIGS["c2"]
    X = G.database(cfg, 3001, start=5)
    train = G.training(cfg, 4000)
    C = orc.fit(train, cfg.m, G.kmeans_init_all(cfg, len(train)), 2)
    a, b, _ = orc.fit_quantizer(G.calibration(cfg, train)[:100], C, 0)
    cb = bolt.CodeBuffer(cfg.m, torch.device("cuda"), capacity=64)
    for r0 in range(0, 3001, 777):
        cb.append(dev(X[r0:r0 + 777]), dev(C))
    assert cb.n == 3001
    np.testing.assert_array_equal(host(cb.codes), host(bolt.encode(dev(X), dev(C))))
    ql = bolt.build_quantized_luts(dev(G.queries(cfg, 7)), dev(C), 0, float(a), dev(b))
    keys = host(bolt.topk(cb.codes, cb.n, ql, 10, 0))
    np.testing.assert_array_equal(keys, orc.topk(orc.unpack_v1(host(cb.codes), 3001, cfg.m), host(ql), 10, 0))


# ------------------------------------------------------------ empty inputs
def test_empty_inputs(bolt):
    """n = 0 or nq = 0 through every entry point: no launch faults, top-k lists
    all padding (UINT64_MAX), empty outputs stay empty."""
    import torch
    m = 16
    C = dev(G.random_floats((m, 16, 8), 5))
    codes0 = bolt.encode(torch.empty((0, 128), dtype=torch.float32, device="cuda"), C)
    assert codes0.numel() == 0
    codes = bolt.pack_codes(dev(G.random_codes(100, m, 6)))
    ql = dev(G.random_qluts(3, m, 7))
    pad = np.full((3, 10), np.uint64(2**64 - 1))
    for v in (bolt.VARIANT_AUTO, bolt.VARIANT_PRMT, bolt.VARIANT_TC):
        np.testing.assert_array_equal(host(bolt.topk(codes, 0, ql, 10, 0, variant=v)), pad)
    assert host(bolt.topk(codes, 100, ql[:0], 10, 0)).shape == (0, 10)
    assert host(bolt.scan(codes, 0, ql)).shape == (0, 3)
    assert host(bolt.scan(codes, 100, ql[:0])).shape == (100, 0)
    luts = dev(G.random_floats((3, m, 16), 8))
    np.testing.assert_array_equal(host(bolt.topk_f32(codes, 0, luts, 10, 0)), pad)
    assert host(bolt.scan_f32(codes, 0, luts)).shape == (0, 3)
    buf = torch.zeros(bolt.codes_words(8, m), dtype=torch.uint32, device="cuda")
    bolt.encode_append(torch.empty((0, 128), dtype=torch.float32, device="cuda"), C, buf, 0)
    assert int(host(buf).sum()) == 0


# ------------------------------------------------------- offline fit (f1)
@pytest.mark.parametrize("cfg_name,n", [("c1", 10_000), ("c2", 20_000), ("c4", 5_000)])
def test_kmeans_gpu_equals_oracle(bolt, orc, cfg_name, n):
    """GPU k-means follows the oracle's fp64 operation order exactly (R8), so
    the fp32 codebooks agree bit for bit."""
    cfg = G.CONFIGS[cfg_name]
    train = G.training(cfg, n)
    init = G.kmeans_init_all(cfg, n)
    ref = orc.fit(train, cfg.m, init, 6)
    got = host(bolt.kmeans(dev(train), cfg.m, dev(init), 6))
    np.testing.assert_array_equal(got, ref)


def test_kmeans_gpu_empty_cluster(bolt, orc):
    pts = np.array([[0.0], [0.1], [0.2], [50.0]] + [[100.0 + i] for i in range(14)], np.float32)
    init = np.array([[0, 0] + list(range(4, 18))])
    np.testing.assert_array_equal(host(bolt.kmeans(dev(pts), 1, dev(init), 3)), orc.fit(pts, 1, init, 3))


@pytest.mark.parametrize("metric", [0, 1])
@pytest.mark.parametrize("cfg_name", ["c1", "c2", "c3"])
def test_calibrate_gpu_equals_oracle(bolt, orc, cfg_name, metric):
    cfg = G.CONFIGS[cfg_name]
    train = G.training(cfg, 4000)
    C = orc.fit(train, cfg.m, G.kmeans_init_all(cfg, len(train)), 3)
    calib = G.calibration(cfg, train)[:300]
    D = orc.luts(calib, C, metric)
    a_ref, b_ref, alpha_ref, mse_ref = orc.calibrate(D)
    a, b, am = bolt.calibrate(dev(D))
    am = host(am)
    np.testing.assert_array_equal(am[1:], mse_ref)
    assert am[0] == alpha_ref
    assert host(a)[0] == np.float32(a_ref)
    np.testing.assert_array_equal(host(b), b_ref.astype(np.float32))


def test_calibrate_gpu_alpha_above_zero(bolt, orc):
    """The tail-heavy tables of the oracle pin (tests/test_oracle_pins.py)
    where alpha = 0.001 wins: the GPU picks the same alpha, (a, b) and grid
    errors, bit for bit."""
    rng = np.random.default_rng(7)
    D = rng.uniform(0.0, 1.0, (12_500, 2, 16))
    D[17, 0, 3], D[5, 1, 1] = 256.0, -200.0
    a_ref, b_ref, alpha_ref, mse_ref = orc.calibrate(D)
    assert alpha_ref == 0.001
    a, b, am = bolt.calibrate(dev(D))
    am = host(am)
    assert am[0] == alpha_ref
    np.testing.assert_array_equal(am[1:], mse_ref)
    assert host(a)[0] == np.float32(a_ref)
    np.testing.assert_array_equal(host(b), b_ref.astype(np.float32))


def test_model_fit_on_gpu(bolt, orc):
    cfg = G.CONFIGS["c1"]
    X = G.database(cfg)
    init = G.kmeans_init_all(cfg, len(X))
    calib = G.calibration(cfg, X)
    model = bolt.BoltModel.fit(dev(X), cfg.m, dev(init), dev(calib), 0, iters=cfg.kmeans_iters)
    C = orc.fit(X, cfg.m, init, cfg.kmeans_iters)
    np.testing.assert_array_equal(host(model.C), C)
    a, b, alpha = orc.fit_quantizer(calib, C, 0)
    assert model.a == float(a) and model.alpha == alpha
    np.testing.assert_array_equal(host(model.b), b)
