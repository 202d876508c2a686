"""Out-of-bounds write checks (GPU): every output and workspace buffer is a
window into a larger allocation pre-filled with a byte pattern; after the call
the bytes around the window — and, for strided outputs (ldo > nq), the padding
columns between rows — must still hold the pattern, and the results must equal
those of the same call on plain allocations.  Stands in for a memcheck run
(compute-sanitizer is not available on the GPU pool): ragged sizes, odd M,
every scan / top-k variant including the TMA-store full output and k > 32.
"""
import numpy as np
import pytest
import torch

from synth import generators as G

pytestmark = pytest.mark.gpu

PAT = 0xA5
PAD = 4096  # guard bytes on each side (keeps every view 4 KB aligned)


@pytest.fixture(scope="module")
def bolt():
    import paper_1706_10283_b200 as bolt
    assert torch.cuda.is_available(), "GPU tests need a B200"
    bolt._lib.load()
    return bolt


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


class Guarded:
    """nbytes of device memory with PAD pattern bytes before and after."""

    def __init__(self, nbytes: int):
        self.n = int(nbytes)
        self.buf = torch.full((PAD + self.n + PAD,), PAT, dtype=torch.uint8, device="cuda")

    def view(self, dtype, shape):
        return self.buf[PAD:PAD + self.n].view(dtype).view(shape)

    def check(self, what: str):
        torch.cuda.synchronize()
        b = self.buf.cpu().numpy()
        bad_pre = np.flatnonzero(b[:PAD] != PAT)
        bad_post = np.flatnonzero(b[PAD + self.n:] != PAT)
        assert bad_pre.size == 0, f"{what}: {bad_pre.size} bytes written before the buffer (first at -{PAD - bad_pre[0]})"
        assert bad_post.size == 0, f"{what}: {bad_post.size} bytes written past the end (first at +{bad_post[0]})"


def _rows(g: Guarded, n: int, ldo: int, es: int) -> np.ndarray:
    """The [n][ldo] element window as bytes [n][ldo * es] (host copy; uint8
    only, so no uint16/uint64 tensor ops are needed)."""
    torch.cuda.synchronize()
    return g.buf[PAD:PAD + n * ldo * es].view(n, ldo * es).cpu().numpy()


def _check_strided(g: Guarded, n: int, ldo: int, nq: int, es: int, ref: torch.Tensor, what: str):
    """Columns nq..ldo still hold the pattern; columns < nq equal `ref` bytewise."""
    g.check(what)
    raw = _rows(g, n, ldo, es)
    pad = raw[:, nq * es:]
    assert (pad == PAT).all(), f"{what}: {(pad != PAT).sum()} padding bytes between rows written"
    want = ref.contiguous().view(torch.uint8).view(n, nq * es).cpu().numpy()
    np.testing.assert_array_equal(raw[:, :nq * es], want)


@pytest.mark.parametrize("n,m,L", [(4099, 16, 8), (777, 32, 16), (100, 5, 7), (1, 8, 8)])
def test_encode_guard(bolt, n, m, L):
    X = dev(G.random_floats((n, m * L), 70 + n))
    C = dev(G.random_floats((m, 16, L), 71 + m))
    words = bolt.codes_words(n, m)
    g = Guarded(4 * words)
    out = bolt.encode(X, C, out=g.view(torch.uint32, (words,)))
    g.check("bolt_encode")
    assert torch.equal(out.view(torch.int32), bolt.encode(X, C).view(torch.int32))


def test_build_quantized_luts_guard(bolt):
    nq, m, L = 33, 16, 8
    Q = dev(G.random_floats((nq, m * L), 72, scale=2.0))
    C = dev(G.random_floats((m, 16, L), 73))
    b = dev(np.linspace(-1, 1, m).astype(np.float32))
    g = Guarded(nq * m * 16)
    out = bolt.build_quantized_luts(Q, C, 0, 9.0, b, out=g.view(torch.uint8, (nq, m, 16)))
    g.check("bolt_build_quantized_luts")
    assert torch.equal(out, bolt.build_quantized_luts(Q, C, 0, 9.0, b))


SCAN_CASES = [  # n, m, nq, variant
    (3001, 16, 64, 0), (3001, 16, 200, 0), (1025, 32, 72, 0), (999, 8, 96, 0),
    (3001, 16, 200, 1), (517, 12, 10, 0), (2049, 16, 8, 0)]


@pytest.mark.parametrize("n,m,nq,variant", SCAN_CASES)
def test_scan_guard_strided(bolt, n, m, nq, variant):
    codes = bolt.pack_codes(dev(G.random_codes(n, m, 74 + n)))
    ql = dev(G.random_qluts(nq, m, 75 + nq))
    ldo = nq + 8
    g = Guarded(n * ldo * 2)
    out = g.view(torch.uint16, (n, ldo))[:, :nq]
    bolt.scan(codes, n, ql, out=out, variant=variant)
    _check_strided(g, n, ldo, nq, 2, bolt.scan(codes, n, ql, variant=variant), "bolt_scan_ex")


@pytest.mark.parametrize("n,m,nq,variant", SCAN_CASES)
def test_scan_dequant_guard_strided(bolt, n, m, nq, variant):
    codes = bolt.pack_codes(dev(G.random_codes(n, m, 76 + n)))
    ql = dev(G.random_qluts(nq, m, 77 + nq))
    ldo = nq + 4
    g = Guarded(n * ldo * 4)
    out = g.view(torch.float32, (n, ldo))[:, :nq]
    bolt.scan_dequant(codes, n, ql, 7.5, -3.25, out=out, variant=variant)
    _check_strided(g, n, ldo, nq, 4, bolt.scan_dequant(codes, n, ql, 7.5, -3.25, variant=variant),
                   "bolt_scan_dequant_ex")


TOPK_CASES = [  # n, m, nq, k, variant (0 auto, 1 PRMT, 2 tcgen05, 3 swapped tcgen05)
    (5000, 16, 3, 10, 0), (5000, 12, 70, 10, 1), (20000, 16, 40, 10, 2), (20000, 16, 300, 32, 2),
    (20000, 16, 100, 100, 2), (20000, 16, 50, 10, 3), (9001, 32, 130, 5, 2), (9001, 8, 20, 1, 0),
    (7, 16, 5, 10, 0), (7, 16, 200, 10, 2)]


@pytest.mark.parametrize("n,m,nq,k,variant", TOPK_CASES)
def test_topk_guard(bolt, n, m, nq, k, variant):
    codes = bolt.pack_codes(dev(G.random_codes(n, m, 78 + n)))
    ql = dev(G.random_qluts(nq, m, 79 + nq))
    wsb = bolt.topk_workspace_bytes(n, m, nq, k, variant)
    gw = Guarded(max(wsb, 8))
    go = Guarded(nq * k * 8)
    out = bolt.topk(codes, n, ql, k, 0, index_base=11, variant=variant,
                    out=go.view(torch.uint64, (nq, k)), workspace=gw.view(torch.uint8, (max(wsb, 8),)))
    go.check("bolt_topk_ex keys")
    gw.check("bolt_topk_ex workspace")
    ref = bolt.topk(codes, n, ql, k, 0, index_base=11, variant=variant)
    assert torch.equal(out.view(torch.int64), ref.view(torch.int64))


@pytest.mark.parametrize("w,nq,k", [(5, 7, 10), (40, 3, 10), (300, 2, 32), (2, 5, 128)])
def test_merge_guard(bolt, w, nq, k):
    r = np.random.default_rng([5, w, nq, k])
    keys = np.sort(r.integers(0, 2**62, (w, nq, k), dtype=np.int64), axis=2).view(np.uint64)
    keys[0, :, k // 2:] = np.iinfo(np.uint64).max  # padded list tails
    kd = dev(keys)
    g = Guarded(nq * k * 8)
    out = bolt.topk_merge(kd, out=g.view(torch.uint64, (nq, k)))
    g.check("bolt_topk_merge")
    assert torch.equal(out.view(torch.int64), bolt.topk_merge(kd).view(torch.int64))


@pytest.mark.parametrize("n,m,nq,k", [(3001, 16, 9, 10), (517, 8, 40, 32), (65, 32, 3, 1)])
def test_f32_guard(bolt, n, m, nq, k):
    codes = bolt.pack_codes(dev(G.random_codes(n, m, 80 + n)))
    luts = dev(G.random_floats((nq, m, 16), 81 + nq))
    ldo = nq + 3
    g = Guarded(n * ldo * 4)
    out = g.view(torch.float32, (n, ldo))[:, :nq]
    bolt.scan_f32(codes, n, luts, out=out)
    _check_strided(g, n, ldo, nq, 4, bolt.scan_f32(codes, n, luts), "bolt_scan_f32")
    go = Guarded(nq * k * 8)
    keys = bolt.topk_f32(codes, n, luts, k, 0, out=go.view(torch.uint64, (nq, k)))
    go.check("bolt_topk_f32")
    assert torch.equal(keys.view(torch.int64), bolt.topk_f32(codes, n, luts, k, 0).view(torch.int64))
