"""Bolt (arXiv 1706.10283) read-side hot path on B200 (sm_100a).

Thin Python binding of the C ABI in include/bolt.h: every function below only
checks tensors and marshals pointers; all computation runs in the CUDA kernels
of libbolt.so on the caller's current CUDA stream.  PyTorch provides device
memory and streams only.  There is no CPU fallback.

Names follow the paper: h = ``encode``, g = ``build_luts`` +
``quantize_luts``, d^ = ``scan`` / ``topk``
(P:L224-231, L264), k closest = ``topk``.
"""
from __future__ import annotations

import dataclasses

import torch

from . import _lib
from ._lib import BoltError  # noqa: F401

L2SQ, DOT = 0, 1
VARIANT_AUTO, VARIANT_PRMT, VARIANT_TC, VARIANT_TCS, VARIANT_SP = 0, 1, 2, 3, 4
K = 16
_METRICS = {"l2": L2SQ, "l2sq": L2SQ, "euclidean": L2SQ, "dot": DOT, "mips": DOT}


def _metric(metric) -> int:
    if isinstance(metric, str):
        return _METRICS[metric.lower()]
    if metric not in (L2SQ, DOT):
        raise ValueError(f"metric must be L2SQ (0) or DOT (1), got {metric!r}")
    return int(metric)


def _stream(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _cuda(t: torch.Tensor, name: str, dtype=None) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t


def _ptr(t):
    return None if t is None else t.data_ptr()


def version() -> str:
    return _lib.load().bolt_version().decode()


def codes_words(n: int, m: int) -> int:
    return int(_lib.load().bolt_codes_words(n, m))


# ------------------------------------------------------------------ h (encode)
ENCODE_AUTO, ENCODE_DIRECT, ENCODE_EXPANDED = 0, 1, 2


def encode(X: torch.Tensor, C: torch.Tensor, out: torch.Tensor | None = None,
           variant: int = ENCODE_AUTO) -> torch.Tensor:
    """X fp32 [n][J], C fp32 [M][16][J/M] -> layout-v1 codes, uint32 [ceil(n/8)*M].
    variant: ENCODE_AUTO / ENCODE_DIRECT (direct differences) or ENCODE_EXPANDED
    (expanded distances + exact fallback); all return the same codes bit for bit."""
    _cuda(X, "X", torch.float32)
    _cuda(C, "C", torch.float32)
    n, j = X.shape
    m = C.shape[0]
    if out is None:
        out = torch.empty(codes_words(n, m), dtype=torch.uint32, device=X.device)
    _lib.call("bolt_encode_ex", X.data_ptr(), n, j, j, C.data_ptr(), m, out.data_ptr(), int(variant),
              _stream(X.device))
    return out


def encode_append(X: torch.Tensor, C: torch.Tensor, codes: torch.Tensor, n_old: int) -> torch.Tensor:
    """Encode-on-write: append the rows of X (fp32 [n_new][J]) to `codes`, which
    holds n_old rows and has room for codes_words(n_old + n_new, M) words;
    afterwards codes == encode(all rows) bit for bit (bolt_encode_append)."""
    _cuda(X, "X", torch.float32)
    _cuda(C, "C", torch.float32)
    _cuda(codes, "codes", torch.uint32)
    n_new, j = X.shape
    m = C.shape[0]
    if codes.numel() < codes_words(n_old + n_new, m):
        raise ValueError(f"codes holds {codes.numel()} words, {codes_words(n_old + n_new, m)} needed")
    _lib.call("bolt_encode_append", X.data_ptr(), n_new, j, j, C.data_ptr(), m, codes.data_ptr(), n_old,
              _stream(X.device))
    return codes


class CodeBuffer:
    """A live, growable layout-v1 code store for streaming encode-on-write
    (SURVEY 8(f4)): append() encodes new rows straight into the buffer
    (capacity doubles when full); `codes` / `n` feed topk / scan directly."""

    def __init__(self, m: int, device, capacity: int = 1 << 16):
        self.m, self.n = m, 0
        self._buf = torch.zeros(codes_words(max(capacity, 8), m), dtype=torch.uint32, device=device)

    @property
    def codes(self) -> torch.Tensor:
        return self._buf[:codes_words(self.n, self.m)]

    def append(self, X: torch.Tensor, C: torch.Tensor) -> None:
        need = codes_words(self.n + X.shape[0], self.m)
        if need > self._buf.numel():
            grown = torch.zeros(max(need, 2 * self._buf.numel()), dtype=torch.uint32, device=self._buf.device)
            grown[:self._buf.numel()] = self._buf
            self._buf = grown
        encode_append(X, C, self._buf, self.n)
        self.n += X.shape[0]


def pack_codes(flat: torch.Tensor) -> torch.Tensor:
    _cuda(flat, "flat", torch.uint8)
    n, m = flat.shape
    out = torch.empty(codes_words(n, m), dtype=torch.uint32, device=flat.device)
    _lib.call("bolt_pack_codes", flat.data_ptr(), n, m, out.data_ptr(), _stream(flat.device))
    return out


def unpack_codes(codes: torch.Tensor, n: int, m: int) -> torch.Tensor:
    _cuda(codes, "codes", torch.uint32)
    out = torch.empty((n, m), dtype=torch.uint8, device=codes.device)
    _lib.call("bolt_unpack_codes", codes.data_ptr(), n, m, out.data_ptr(), _stream(codes.device))
    return out


# ------------------------------------------------------------------- g (LUTs)
def build_luts(Q: torch.Tensor, C: torch.Tensor, metric, f64: bool = False) -> torch.Tensor:
    """Q fp32 [nq][J] -> D [nq][M][16] (fp32, or fp64 with f64=True)."""
    _cuda(Q, "Q", torch.float32)
    _cuda(C, "C", torch.float32)
    nq, j = Q.shape
    m = C.shape[0]
    out = torch.empty((nq, m, K), dtype=torch.float64 if f64 else torch.float32, device=Q.device)
    fn = "bolt_build_luts_f64" if f64 else "bolt_build_luts"
    _lib.call(fn, Q.data_ptr(), nq, j, j, C.data_ptr(), m, _metric(metric), out.data_ptr(), _stream(Q.device))
    return out


def quantize_luts(luts: torch.Tensor, a: float, b: torch.Tensor) -> torch.Tensor:
    """fp32 [nq][M][16] -> u8 beta = clamp(floor(a (y - b_m)), 0, 255)."""
    _cuda(luts, "luts", torch.float32)
    _cuda(b, "b", torch.float32)
    nq, m, _ = luts.shape
    out = torch.empty((nq, m, K), dtype=torch.uint8, device=luts.device)
    _lib.call("bolt_quantize_luts", luts.data_ptr(), nq, m, float(a), b.data_ptr(), out.data_ptr(),
              _stream(luts.device))
    return out


def build_quantized_luts(Q: torch.Tensor, C: torch.Tensor, metric, a: float, b: torch.Tensor,
                         return_f32: bool = False, out: torch.Tensor | None = None):
    """Fused g: fp64 tables quantized to u8 [nq][M][16] (+ fp32 tables)."""
    _cuda(Q, "Q", torch.float32)
    _cuda(C, "C", torch.float32)
    _cuda(b, "b", torch.float32)
    nq, j = Q.shape
    m = C.shape[0]
    if out is None:
        out = torch.empty((nq, m, K), dtype=torch.uint8, device=Q.device)
    f32 = torch.empty((nq, m, K), dtype=torch.float32, device=Q.device) if return_f32 else None
    _lib.call("bolt_build_quantized_luts", Q.data_ptr(), nq, j, j, C.data_ptr(), m, _metric(metric),
              float(a), b.data_ptr(), out.data_ptr(), _ptr(f32), _stream(Q.device))
    return (out, f32) if return_f32 else out


# ------------------------------------------------------------------- d^ (scan)
def scan(codes: torch.Tensor, n: int, qluts: torch.Tensor, out: torch.Tensor | None = None,
         variant: int = VARIANT_AUTO) -> torch.Tensor:
    """Exact u16 sums [n][nq] (row = database vector)."""
    _cuda(codes, "codes", torch.uint32)
    _cuda(qluts, "qluts", torch.uint8)
    nq, m, _ = qluts.shape
    if out is None:
        out = torch.empty((n, nq), dtype=torch.uint16, device=codes.device)
    _lib.call("bolt_scan_ex", codes.data_ptr(), n, m, qluts.data_ptr(), nq, out.data_ptr(), out.stride(0),
              int(variant), _stream(codes.device))
    return out


def scan_dequant(codes: torch.Tensor, n: int, qluts: torch.Tensor, a: float, b_sum: float,
                 out: torch.Tensor | None = None, variant: int = VARIANT_AUTO) -> torch.Tensor:
    """fp32 [n][nq] = acc / a + sum_m b_m (approximate A.B)."""
    _cuda(codes, "codes", torch.uint32)
    _cuda(qluts, "qluts", torch.uint8)
    nq, m, _ = qluts.shape
    if out is None:
        out = torch.empty((n, nq), dtype=torch.float32, device=codes.device)
    _lib.call("bolt_scan_dequant_ex", codes.data_ptr(), n, m, qluts.data_ptr(), nq, float(a), float(b_sum),
              out.data_ptr(), out.stride(0), int(variant), _stream(codes.device))
    return out


def topk_workspace_bytes(n: int, m: int, nq: int, k: int, variant: int = VARIANT_AUTO) -> int:
    return int(_lib.load().bolt_topk_workspace_bytes_ex(n, m, nq, k, variant))


def topk_plan(n: int, m: int, nq: int, k: int, variant: int = VARIANT_AUTO):
    """-> (resolved variant name 'prmt' | 'tc' | 'tcs' | 'sp', number of merged row partitions)."""
    import ctypes
    v, p = ctypes.c_int(0), ctypes.c_int(0)
    _lib.call("bolt_topk_plan", n, m, nq, k, variant, ctypes.byref(v), ctypes.byref(p))
    return {VARIANT_PRMT: "prmt", VARIANT_TC: "tc", VARIANT_TCS: "tcs", VARIANT_SP: "sp"}[v.value], p.value


def topk(codes: torch.Tensor, n: int, qluts: torch.Tensor, k: int, metric, index_base: int = 0,
         variant: int = VARIANT_AUTO, out: torch.Tensor | None = None,
         workspace: torch.Tensor | None = None) -> torch.Tensor:
    """u64 keys [nq][k], ascending ((value << 48) | global index; R13)."""
    _cuda(codes, "codes", torch.uint32)
    _cuda(qluts, "qluts", torch.uint8)
    nq, m, _ = qluts.shape
    if out is None:
        out = torch.empty((nq, k), dtype=torch.uint64, device=codes.device)
    wsb = topk_workspace_bytes(n, m, nq, k, variant)
    if workspace is None or workspace.numel() < wsb:
        workspace = torch.empty(max(wsb, 8), dtype=torch.uint8, device=codes.device)
    _lib.call("bolt_topk_ex", codes.data_ptr(), n, m, qluts.data_ptr(), nq, int(k), _metric(metric),
              int(index_base), out.data_ptr(), workspace.data_ptr(), workspace.numel(), int(variant),
              _stream(codes.device))
    return out


def topk_merge(keys: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """[W][nq][k] sorted shard lists -> [nq][k]."""
    _cuda(keys, "keys", torch.uint64)
    w, nq, k = keys.shape
    if out is None:
        out = torch.empty((nq, k), dtype=torch.uint64, device=keys.device)
    _lib.call("bolt_topk_merge", keys.data_ptr(), w, nq, k, out.data_ptr(), _stream(keys.device))
    return out


def keys_split(keys: torch.Tensor, metric):
    """-> (values u16, global indices int64; -1 for padding)."""
    _cuda(keys, "keys", torch.uint64)
    vals = torch.empty(keys.shape, dtype=torch.uint16, device=keys.device)
    idx = torch.empty(keys.shape, dtype=torch.int64, device=keys.device)
    _lib.call("bolt_keys_split", keys.data_ptr(), keys.numel(), _metric(metric), vals.data_ptr(),
              idx.data_ptr(), _stream(keys.device))
    return vals, idx


# ------------------------------------------- Bolt No Quantize (fp32 tables)
def scan_f32(codes: torch.Tensor, n: int, luts: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """P:L390's "Bolt No Quantize": fp32 [n][nq] totals of the fp32 tables
    (build_luts) summed in fp32, ascending codebooks (bolt_scan_f32)."""
    _cuda(codes, "codes", torch.uint32)
    _cuda(luts, "luts", torch.float32)
    nq, m, _ = luts.shape
    if out is None:
        out = torch.empty((n, nq), dtype=torch.float32, device=codes.device)
    _lib.call("bolt_scan_f32", codes.data_ptr(), n, m, luts.data_ptr(), nq, out.data_ptr(), out.stride(0),
              _stream(codes.device))
    return out


def topk_f32(codes: torch.Tensor, n: int, luts: torch.Tensor, k: int, metric, index_base: int = 0,
             out: torch.Tensor | None = None) -> torch.Tensor:
    """u64 keys [nq][k] of the fp32 totals (R18), ascending; k <= 32."""
    _cuda(codes, "codes", torch.uint32)
    _cuda(luts, "luts", torch.float32)
    nq, m, _ = luts.shape
    if out is None:
        out = torch.empty((nq, k), dtype=torch.uint64, device=codes.device)
    wsb = _lib.load().bolt_topk_f32_workspace_bytes(n, m, nq, k)
    ws = torch.empty(max(int(wsb), 8), dtype=torch.uint8, device=codes.device)
    _lib.call("bolt_topk_f32", codes.data_ptr(), n, m, luts.data_ptr(), nq, k, _metric(metric), index_base,
              out.data_ptr(), ws.data_ptr(), ws.numel(), _stream(codes.device))
    return out


def keys_split_f32(keys: torch.Tensor, metric):
    """R18 keys -> (fp32 values, global indices int64; -1 for padding)."""
    _cuda(keys, "keys", torch.uint64)
    vals = torch.empty(keys.shape, dtype=torch.float32, device=keys.device)
    idx = torch.empty(keys.shape, dtype=torch.int64, device=keys.device)
    _lib.call("bolt_keys_split_f32", keys.data_ptr(), keys.numel(), _metric(metric), vals.data_ptr(),
              idx.data_ptr(), _stream(keys.device))
    return vals, idx


# --------------------------------------------------------- end-to-end (host)
class HostSearch:
    """Host-buffer search: H2D of X and Q, encode, fused tables, top-k, D2H of
    the keys.  chunks == 1: bolt_search_host, everything on one stream;
    chunks > 1: bolt_search_host_pipelined, X crossing PCIe in row blocks on a
    side stream while the current stream encodes and scans the blocks that
    have landed (same keys)."""

    def __init__(self, n: int, j: int, m: int, nq: int, k: int, device=None, chunks: int = 1):
        self.n, self.j, self.m, self.nq, self.k, self.chunks = n, j, m, nq, k, chunks
        self.device = torch.device(device or "cuda")
        if chunks > 1:
            wsb = int(_lib.load().bolt_search_host_pipelined_workspace_bytes(n, j, m, nq, k, chunks))
            self.copy_stream = torch.cuda.Stream(self.device)
        else:
            wsb = int(_lib.load().bolt_search_host_workspace_bytes(n, j, m, nq, k))
        self.workspace = torch.empty(wsb, dtype=torch.uint8, device=self.device)

    def __call__(self, X_host: torch.Tensor, Q_host: torch.Tensor, C: torch.Tensor, metric, a: float,
                 b: torch.Tensor, keys_host: torch.Tensor, index_base: int = 0) -> torch.Tensor:
        """keys_host [nq][k] u64 <- top-k of the rows of X_host, whose global
        indices start at index_base (a row shard of a larger database)."""
        for t, nm in ((X_host, "X_host"), (Q_host, "Q_host")):
            if t.is_cuda or t.dtype != torch.float32 or not t.is_contiguous():
                raise TypeError(f"{nm} must be a contiguous fp32 host tensor")
        if keys_host.is_cuda or keys_host.dtype != torch.uint64:
            raise TypeError("keys_host must be a uint64 host tensor")
        _cuda(C, "C", torch.float32)
        _cuda(b, "b", torch.float32)
        if self.chunks > 1:
            _lib.call("bolt_search_host_pipelined_ex", X_host.data_ptr(), self.n, self.j, Q_host.data_ptr(), self.nq,
                      C.data_ptr(), self.m, _metric(metric), float(a), b.data_ptr(), self.k, int(index_base),
                      keys_host.data_ptr(), self.workspace.data_ptr(), self.workspace.numel(), self.chunks,
                      _stream(self.device), self.copy_stream.cuda_stream)
        else:
            _lib.call("bolt_search_host_ex", X_host.data_ptr(), self.n, self.j, Q_host.data_ptr(), self.nq,
                      C.data_ptr(), self.m, _metric(metric), float(a), b.data_ptr(), self.k, int(index_base),
                      keys_host.data_ptr(), self.workspace.data_ptr(), self.workspace.numel(),
                      _stream(self.device))
        return keys_host


# ---------------------------------------------------------------- offline fit
def kmeans(train: torch.Tensor, m: int, init: torch.Tensor, iters: int = 16) -> torch.Tensor:
    """GPU k-means codebooks (R8), fp64 inside, -> C fp32 [M][16][J/M]."""
    _cuda(train, "train", torch.float32)
    _cuda(init, "init", torch.int64)
    n, j = train.shape
    out = torch.empty((m, K, j // m), dtype=torch.float32, device=train.device)
    wsb = int(_lib.load().bolt_kmeans_workspace_bytes(n, j, m))
    ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device=train.device)
    _lib.call("bolt_kmeans", train.data_ptr(), n, j, j, m, init.data_ptr(), int(iters), out.data_ptr(),
              ws.data_ptr(), ws.numel(), _stream(train.device))
    return out


def calibrate(luts64: torch.Tensor):
    """LUT-quantizer learning on fp64 tables -> (a fp32 [1], b fp32 [M], alpha_mse fp64 [9])."""
    _cuda(luts64, "luts64", torch.float64)
    nq, m, _ = luts64.shape
    a = torch.empty(1, dtype=torch.float32, device=luts64.device)
    b = torch.empty(m, dtype=torch.float32, device=luts64.device)
    am = torch.empty(9, dtype=torch.float64, device=luts64.device)
    wsb = int(_lib.load().bolt_calibrate_workspace_bytes(nq, m))
    ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device=luts64.device)
    _lib.call("bolt_calibrate", luts64.data_ptr(), nq, m, a.data_ptr(), b.data_ptr(), am.data_ptr(),
              ws.data_ptr(), ws.numel(), _stream(luts64.device))
    return a, b, am


@dataclasses.dataclass
class BoltModel:
    """Trained quantizer: codebooks C [M][16][J/M] fp32, LUT scale a, offsets b [M]."""
    C: torch.Tensor
    a: float
    b: torch.Tensor
    metric: int
    alpha: float = 0.0

    @property
    def m(self) -> int:
        return self.C.shape[0]

    @staticmethod
    def fit(train: torch.Tensor, m: int, init: torch.Tensor, calib_queries: torch.Tensor, metric,
            iters: int = 16) -> "BoltModel":
        """Offline phase entirely on the GPU: k-means codebooks,
        then the LUT quantizer from calibration queries' fp64 tables."""
        C = kmeans(train, m, init, iters)
        D = build_luts(calib_queries, C, metric, f64=True)
        a, b, am = calibrate(D)
        return BoltModel(C, float(a.item()), b, _metric(metric), float(am[0].item()))

    def encode(self, X):
        return encode(X, self.C)

    def luts(self, Q):
        return build_quantized_luts(Q, self.C, self.metric, self.a, self.b)

    def search(self, codes, n, Q, k, variant=VARIANT_AUTO):
        return topk(codes, n, self.luts(Q), k, self.metric, variant=variant)
