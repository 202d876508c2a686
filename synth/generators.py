"""Seeded generators for BASELINE.json configs c1-c5.

Every stream is numpy PCG64 keyed by ``[SEED, config, stream, ...]``:
stream 0 = distribution parameters, 1 = database, 2 = k-means training set,
3 = calibration sample, 4 = queries, 5 = k-means init (``[SEED, c, 5, m]``).
Row streams are produced in chunks of ``CHUNK`` rows, chunk ``j`` drawn from
``[SEED, c, s, j]``, so that the first ``n`` rows of a stream never depend on
how many rows were requested (tests and the CPU baseline use prefixes of the
benchmark workload).

Stand-ins (no dataset is available or fetched): c2 ~ Sift1M shape
(1M x 128, 10k queries, 100k train); c3 ~ 512-d GIST-like
(LabelMe, L372) with MNIST-like sparsity (L373), dot product; c4 = Fig. 3
bottom, 100,000 x 256 times 256 x n (L434); c5 = c2 scaled to 1e8 rows.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

SEED = 170610283
CHUNK = 65536
L2SQ, DOT = 0, 1


def rng(*key: int) -> np.random.Generator:
    return np.random.default_rng([SEED, *key])


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    cid: int
    n: int            # database rows
    j: int            # dimension J
    m: int            # codebooks M (16 centroids each)
    nq: int           # queries
    metrics: tuple    # (L2SQ,) / (DOT,) / both
    k: int            # top-k (0 = full N x Q output)
    n_train: int      # k-means training rows (0 = train on the database)
    n_calib: int      # calibration queries
    kmeans_iters: int = 16


CONFIGS = {
    "c1": Config("c1", 1, 10_000, 32, 8, 16, (L2SQ, DOT), 0, 0, 256),
    "c2": Config("c2", 2, 1_000_000, 128, 16, 10_000, (L2SQ,), 10, 100_000, 1_000),
    "c3": Config("c3", 3, 1_000_000, 512, 32, 1_000, (DOT,), 10, 100_000, 1_000),
    "c4": Config("c4", 4, 100_000, 256, 32, 1_024, (DOT,), 0, 0, 256),
    "c5": Config("c5", 5, 100_000_000, 128, 16, 65_536, (L2SQ,), 100, 100_000, 1_000),
}


# ----------------------------------------------------------------------------
# per-config row recipes: f(generator, size) -> float32 [size, J]
# ----------------------------------------------------------------------------
def _c1_mix() -> np.ndarray:
    return rng(1, 0).standard_normal((32, 32)) / math.sqrt(32.0)


def _c2_means() -> np.ndarray:
    return rng(2, 0).uniform(0.0, 128.0, (1024, 128))


def c5_means() -> np.ndarray:
    """Component means of the c2 mixture, shared by c5's device generator (synth/gen_gpu.cu)."""
    return _c2_means().astype(np.float32)


def _c3_scale() -> np.ndarray:
    return rng(3, 0).uniform(0.1, 2.0, 512)


def _rows_c1(g, size, _cache={}):
    if "w" not in _cache:
        _cache["w"] = _c1_mix()
    z = g.standard_normal((size, 32))
    return (z @ _cache["w"]).astype(np.float32)


def _rows_c2(g, size, _cache={}):
    if "mu" not in _cache:
        _cache["mu"] = _c2_means()
    comp = g.integers(0, 1024, size)
    z = g.standard_normal((size, 128))
    x = np.rint(_cache["mu"][comp] + 20.0 * z)
    return np.clip(x, 0.0, 255.0).astype(np.float32)


def _rows_c3(g, size, _cache={}):
    if "s" not in _cache:
        _cache["s"] = _c3_scale()
    nonzero = g.random((size, 512)) >= 0.5
    e = g.standard_exponential((size, 512)) * _cache["s"]
    return np.where(nonzero, e, 0.0).astype(np.float32)


def _rows_c4(g, size):
    return g.standard_normal((size, 256)).astype(np.float32)


_ROWS = {1: _rows_c1, 2: _rows_c2, 3: _rows_c3, 4: _rows_c4, 5: _rows_c2}


def rows(cid: int, stream: int, n: int, start: int = 0) -> np.ndarray:
    """Rows [start, start+n) of row-stream ``stream`` of config ``cid``."""
    fn = _ROWS[cid]
    src_cid = 2 if cid == 5 else cid
    out = np.empty((n, CONFIGS[f"c{cid}"].j), dtype=np.float32)
    pos = start
    while pos < start + n:
        j = pos // CHUNK
        lo = j * CHUNK
        chunk = fn(rng(src_cid, stream, j), CHUNK)
        a = pos - lo
        b = min(CHUNK, start + n - lo)
        out[pos - start: pos - start + (b - a)] = chunk[a:b]
        pos += b - a
    return out


def database(cfg: Config, n: int | None = None, start: int = 0) -> np.ndarray:
    if cfg.cid == 4:
        return rows(4, 1, cfg.n if n is None else n, start)
    return rows(cfg.cid, 1, cfg.n if n is None else n, start)


def queries(cfg: Config, n: int | None = None) -> np.ndarray:
    n = cfg.nq if n is None else n
    if cfg.cid == 4:
        # columns of B = rng(4,4).standard_normal((256,1024)) are the queries (L434)
        b = rng(4, 4).standard_normal((256, 1024)).astype(np.float32)
        return np.ascontiguousarray(b.T[:n])
    if cfg.cid == 5:
        return _c5_queries(n)
    return rows(cfg.cid, 4, n)


def _c5_queries(n):
    # 65,536 queries from rng(5,4) on the c2 mixture (chunked like every stream)
    out = np.empty((n, 128), dtype=np.float32)
    pos = 0
    while pos < n:
        j = pos // CHUNK
        chunk = _rows_c2(rng(5, 4, j), CHUNK)
        b = min(CHUNK, n - j * CHUNK)
        out[pos:pos + b] = chunk[:b]
        pos += b
    return out


def training(cfg: Config, n: int | None = None) -> np.ndarray:
    """k-means training rows: a separate stream for c2/c3/c5, the database itself for c1/c4."""
    if cfg.n_train == 0:
        return database(cfg, n)
    src = 2 if cfg.cid == 5 else cfg.cid
    return rows(src, 2, cfg.n_train if n is None else n)


def kmeans_init(cfg: Config, n_train: int, m: int, k: int = 16) -> np.ndarray:
    """Indices of the k training rows that seed k-means for subspace m."""
    src = 2 if cfg.cid == 5 else cfg.cid
    return rng(src, 5, m).choice(n_train, k, replace=False).astype(np.int64)


def kmeans_init_all(cfg: Config, n_train: int, k: int = 16) -> np.ndarray:
    return np.stack([kmeans_init(cfg, n_train, m, k) for m in range(cfg.m)])


def calibration(cfg: Config, train: np.ndarray | None = None) -> np.ndarray:
    """Calibration queries (reading L15): a seeded sample of the training rows
    (c2/c3/c5), of the database (c1), or of the columns of B (c4)."""
    src = 2 if cfg.cid == 5 else cfg.cid
    if cfg.cid == 4:
        q = queries(cfg)
        idx = rng(4, 3).choice(1024, cfg.n_calib, replace=False)
        return np.ascontiguousarray(q[idx])
    if train is None:
        train = training(cfg)
    idx = rng(src, 3).choice(len(train), min(cfg.n_calib, len(train)), replace=False)
    return np.ascontiguousarray(train[idx])


# ----------------------------------------------------------------------------
# generic random instances for property tests
# ----------------------------------------------------------------------------
def random_codes(n: int, m: int, seed: int, k: int = 16) -> np.ndarray:
    return np.random.default_rng([SEED, 99, seed]).integers(0, k, (n, m)).astype(np.uint8)


def random_qluts(nq: int, m: int, seed: int, hi: int = 256) -> np.ndarray:
    return np.random.default_rng([SEED, 98, seed]).integers(0, hi, (nq, m, 16)).astype(np.uint8)


def random_floats(shape, seed: int, scale: float = 1.0) -> np.ndarray:
    return (np.random.default_rng([SEED, 97, seed]).standard_normal(shape) * scale).astype(np.float32)
