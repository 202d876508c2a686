"""ctypes binding of the fp64 CPU oracle (oracle/bolt_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs, never by the product
package.  Arguments are numpy arrays; the wrappers only marshal them.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bolt_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
L2SQ, DOT = 0, 1
K = 16

CFLAGS = ["-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-std=c11",
          "-shared", "-fPIC", "-Wall"]


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        i64, i32, f32 = ctypes.c_int64, ctypes.c_int, ctypes.c_float
        sig = {
            "oracle_num_threads": ([], i32),
            "oracle_set_threads": ([i32], None),
            "oracle_encode": ([P, i64, i32, P, i32, P, P], None),
            "oracle_luts": ([P, i64, i32, P, i32, i32, P], None),
            "oracle_quantize": ([P, i64, i32, f32, P, P, P], None),
            "oracle_calibrate": ([P, i64, i32, P, P, P, P], None),
            "oracle_calibrate_grid": ([P, i64, i32, P, P, P, P, P, P], None),
            "oracle_kmeans_subspace": ([P, i64, i32, i32, i32, P, i32, P, P], None),
            "oracle_scan": ([P, i64, i32, P, i64, P], None),
            "oracle_topk": ([P, i64, i32, P, i64, i32, i32, i64, P], None),
            "oracle_scan_f32": ([P, i64, i32, P, i64, P], None),
            "oracle_topk_f32": ([P, i64, i32, P, i64, i32, i32, i64, P], None),
            "oracle_merge": ([P, i32, i64, i32, P], None),
            "oracle_dequant": ([P, i64, f32, P, i32, P], None),
            "oracle_unpack_v1": ([P, i64, i32, P], None),
        }
        for name, (args, res) in sig.items():
            fn = getattr(_lib, name)
            fn.argtypes = args
            fn.restype = res
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"], "oracle inputs must be C-contiguous"
    return a.ctypes.data_as(ctypes.c_void_p)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def num_threads() -> int:
    return lib().oracle_num_threads()


def set_threads(n: int) -> None:
    lib().oracle_set_threads(int(n))


def encode(X, C, with_gap: bool = False):
    """O3: X [n][J] fp32, C [M][16][J/M] fp32 -> flat codes u8 [n][M] (+ gap fp64)."""
    X, C = _f32(X), _f32(C)
    n, J = X.shape
    M = C.shape[0]
    assert J % M == 0 and C.shape == (M, K, J // M)
    codes = np.empty((n, M), np.uint8)
    gap = np.empty((n, M), np.float64) if with_gap else None
    lib().oracle_encode(_p(X), n, J, _p(C), M, _p(codes), _p(gap) if with_gap else None)
    return (codes, gap) if with_gap else codes


def luts(Q, C, metric: int):
    """O4: Q [nq][J] fp32 -> D fp64 [nq][M][16]."""
    Q, C = _f32(Q), _f32(C)
    nq, J = Q.shape
    M = C.shape[0]
    D = np.empty((nq, M, K), np.float64)
    lib().oracle_luts(_p(Q), nq, J, _p(C), M, int(metric), _p(D))
    return D


def quantize(D, a32: float, b32, with_t: bool = False):
    """O6: D fp64 [nq][M][16], fp32 a, fp32 b[M] -> beta u8 (+ pre-floor t fp64)."""
    D = np.ascontiguousarray(D, dtype=np.float64)
    b32 = _f32(b32)
    nq, M, _ = D.shape
    beta = np.empty(D.shape, np.uint8)
    t = np.empty(D.shape, np.float64) if with_t else None
    lib().oracle_quantize(_p(D), nq, M, float(np.float32(a32)), _p(b32), _p(beta),
                          _p(t) if with_t else None)
    return (beta, t) if with_t else beta


def calibrate(D):
    """O5: D fp64 [nq][M][16] of calibration queries -> (a, b[M], alpha, mse[8]) in fp64."""
    D = np.ascontiguousarray(D, dtype=np.float64)
    nq, M, _ = D.shape
    a = np.zeros(1, np.float64)
    alpha = np.zeros(1, np.float64)
    b = np.zeros(M, np.float64)
    mse = np.zeros(8, np.float64)
    lib().oracle_calibrate(_p(D), nq, M, _p(a), _p(b), _p(alpha), _p(mse))
    return float(a[0]), b, float(alpha[0]), mse


def calibrate_grid(D):
    """O5 with every grid point exposed: -> (a [8], b [8][M], mse [8]) in fp64,
    row g for alpha = ALPHA_GRID[g]."""
    D = np.ascontiguousarray(D, dtype=np.float64)
    nq, M, _ = D.shape
    a, alpha = np.zeros(1), np.zeros(1)
    b = np.zeros(M)
    mse, ag, bg = np.zeros(8), np.zeros(8), np.zeros((8, M))
    lib().oracle_calibrate_grid(_p(D), nq, M, _p(a), _p(b), _p(alpha), _p(mse), _p(ag), _p(bg))
    return ag, bg, mse


ALPHA_GRID = (0.0, 0.001, 0.002, 0.005, 0.01, 0.02, 0.05, 0.1)


def kmeans(train, M: int, init, iters: int = 16, with_inertia: bool = False):
    """O2: per-subspace k-means. train [n][J] fp32, init int64 [M][16] row indices.
    Returns C64 fp64 [M][16][L] (+ inertia [M][iters])."""
    train = _f32(train)
    n, J = train.shape
    L = J // M
    init = np.ascontiguousarray(init, dtype=np.int64)
    C64 = np.empty((M, K, L), np.float64)
    inertia = np.empty((M, iters), np.float64)
    for m in range(M):
        cm = np.empty((K, L), np.float64)
        im = np.empty(iters, np.float64)
        lib().oracle_kmeans_subspace(_p(train), n, J, m * L, L, _p(np.ascontiguousarray(init[m])),
                                     iters, _p(cm), _p(im))
        C64[m] = cm
        inertia[m] = im
    return (C64, inertia) if with_inertia else C64


def scan(codes, qluts):
    """O7: flat codes u8 [n][M], qluts u8 [nq][M][16] -> u16 [n][nq]."""
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    qluts = np.ascontiguousarray(qluts, dtype=np.uint8)
    n, M = codes.shape
    nq = qluts.shape[0]
    out = np.empty((n, nq), np.uint16)
    lib().oracle_scan(_p(codes), n, M, _p(qluts), nq, _p(out))
    return out


def topk(codes, qluts, k: int, metric: int, index_base: int = 0):
    """O8: -> u64 keys [nq][k] ascending (UINT64_MAX padding when k > n)."""
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    qluts = np.ascontiguousarray(qluts, dtype=np.uint8)
    n, M = codes.shape
    nq = qluts.shape[0]
    keys = np.empty((nq, k), np.uint64)
    lib().oracle_topk(_p(codes), n, M, _p(qluts), nq, int(k), int(metric), int(index_base), _p(keys))
    return keys


def scan_f32(codes, luts32):
    """O13 (Bolt No Quantize): flat codes u8 [n][M], fp32 tables [nq][M][16] ->
    fp32 [n][nq], summed in fp32 in ascending m (R18)."""
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    luts32 = np.ascontiguousarray(luts32, dtype=np.float32)
    n, M = codes.shape
    nq = luts32.shape[0]
    out = np.empty((n, nq), np.float32)
    lib().oracle_scan_f32(_p(codes), n, M, _p(luts32), nq, _p(out))
    return out


def topk_f32(codes, luts32, k: int, metric: int, index_base: int = 0):
    """O14: -> u64 keys [nq][k] (R18: order-preserving float code << 32 | index)."""
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    luts32 = np.ascontiguousarray(luts32, dtype=np.float32)
    n, M = codes.shape
    nq = luts32.shape[0]
    keys = np.empty((nq, k), np.uint64)
    lib().oracle_topk_f32(_p(codes), n, M, _p(luts32), nq, int(k), int(metric), int(index_base), _p(keys))
    return keys


def keys_split_f32(keys, metric: int):
    """u64 keys (R18) -> (fp32 values, int64 indices; -1 for padding)."""
    keys = np.asarray(keys, dtype=np.uint64)
    ord_ = (keys >> np.uint64(32)).astype(np.uint32)
    if metric == DOT:
        ord_ = ~ord_
    u = np.where(ord_ & np.uint32(0x80000000), ord_ & np.uint32(0x7FFFFFFF), ~ord_).astype(np.uint32)
    vals = u.view(np.float32)
    idx = (keys & np.uint64(0xFFFFFFFF)).astype(np.int64)
    pad = keys == np.uint64(0xFFFFFFFFFFFFFFFF)
    idx[pad] = -1
    return vals, idx


def merge(shard_keys):
    """O9: [W][nq][k] -> [nq][k]."""
    shard_keys = np.ascontiguousarray(shard_keys, dtype=np.uint64)
    W, nq, k = shard_keys.shape
    out = np.empty((nq, k), np.uint64)
    lib().oracle_merge(_p(shard_keys), W, nq, k, _p(out))
    return out


def dequant(acc, a32: float, b32):
    """O10: acc u16 (any shape) -> acc/a + sum(b) in fp64."""
    acc = np.ascontiguousarray(acc, dtype=np.uint16)
    b32 = _f32(b32)
    out = np.empty(acc.shape, np.float64)
    lib().oracle_dequant(_p(acc), acc.size, float(np.float32(a32)), _p(b32), b32.size, _p(out))
    return out


def unpack_v1(words, n: int, M: int):
    """O12: layout-v1 u32 words -> flat codes u8 [n][M]."""
    words = np.ascontiguousarray(words, dtype=np.uint32)
    assert words.size >= ((n + 7) // 8) * M
    flat = np.empty((n, M), np.uint8)
    lib().oracle_unpack_v1(_p(words), n, M, _p(flat))
    return flat


def keys_split(keys, metric: int):
    """Split u64 keys into (u16 acc, int64 index); padding -> (0, -1)."""
    keys = np.asarray(keys, dtype=np.uint64)
    pad = keys == np.uint64(0xFFFFFFFFFFFFFFFF)
    v = (keys >> np.uint64(48)).astype(np.int64)
    if metric == DOT:
        v = 0xFFFF - v
    idx = (keys & np.uint64((1 << 48) - 1)).astype(np.int64)
    v = np.where(pad, 0, v).astype(np.uint16)
    idx = np.where(pad, -1, idx)
    return v, idx


# ------------------------------------------------------------------ fit ----
def fit(train, M: int, init, iters: int = 16):
    """Offline phase: k-means codebooks, rounded to the fp32 C32
    that every downstream step shares."""
    return kmeans(train, M, init, iters).astype(np.float32)


def fit_quantizer(calib_queries, C32, metric: int):
    """Offline LUT-quantizer learning -> (a32, b32[M], alpha)."""
    D = luts(calib_queries, C32, metric)
    a, b, alpha, _ = calibrate(D)
    return np.float32(a), b.astype(np.float32), alpha
