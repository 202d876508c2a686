"""Multi-process (world size 2, gloo on CPU) tests of the row-sharded search glue:
shard ranges, the key all-gather, and that merging the gathered shard lists
(oracle merge here; bolt_topk_merge on GPUs) equals the unsharded top-k."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from synth import generators as G


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, m, nq, k, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle
        from paper_1706_10283_b200.dist import gather_keys, shard_range
        flat = G.random_codes(n, m, 7)
        ql = G.random_qluts(nq, m, 8, hi=16)
        r0, r1 = shard_range(n, world, rank)
        local = oracle.topk(flat[r0:r1], ql, k, 0, index_base=r0)
        gathered = gather_keys(torch.from_numpy(local)).numpy()
        np.save(os.path.join(out_dir, f"g{rank}.npy"), gathered)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [1000, 1003, 17])
def test_sharded_gather_merge_equals_whole(tmp_path, orc, n):
    world, m, nq, k = 2, 8, 5, 10
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, n, m, nq, k, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    flat = G.random_codes(n, m, 7)
    ql = G.random_qluts(nq, m, 8, hi=16)
    whole = orc.topk(flat, ql, k, 0)
    for r in range(world):
        g = np.load(tmp_path / f"g{r}.npy")
        assert g.shape == (world, nq, k)
        np.testing.assert_array_equal(orc.merge(g), whole)


def test_shard_range_properties():
    from paper_1706_10283_b200.dist import shard_range
    for n in [0, 1, 7, 8, 9, 1000, 10**8 + 3]:
        for world in [1, 2, 3, 4, 8]:
            ranges = [shard_range(n, world, r) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            for (a0, a1), (b0, b1) in zip(ranges, ranges[1:]):
                assert a1 == b0
            for r0, r1 in ranges:
                assert r0 % 8 == 0 or r0 == n
                assert r0 <= r1


def _qworker(rank, world, port, n, m, nq, k, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle
        from paper_1706_10283_b200.dist import gather_query_slices, query_range
        flat = G.random_codes(n, m, 3)
        ql = G.random_qluts(nq, m, 4, hi=16)
        q0, q1 = query_range(nq, world, rank)
        local = oracle.topk(flat, ql[q0:q1], k, 0) if q1 > q0 else np.zeros((0, k), np.uint64)
        res = gather_query_slices(torch.from_numpy(local), nq).numpy()
        np.save(os.path.join(out_dir, f"q{rank}.npy"), res)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("nq", [7, 1, 10])
def test_query_sharded_gather_equals_whole(tmp_path, orc, nq):
    """Replicated database, queries split over the ranks: the
    gathered slices equal the single-process top-k; no merge is involved."""
    world, n, m, k = 2, 900, 8, 6
    port = _free_port()
    mp.start_processes(_qworker, args=(world, port, n, m, nq, k, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    whole = orc.topk(G.random_codes(n, m, 3), G.random_qluts(nq, m, 4, hi=16), k, 0)
    for r in range(world):
        np.testing.assert_array_equal(np.load(tmp_path / f"q{r}.npy"), whole)


def test_query_range_properties():
    from paper_1706_10283_b200.dist import query_range
    for nq in [0, 1, 5, 64, 65536, 10001]:
        for world in [1, 2, 3, 8]:
            rs = [query_range(nq, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == nq
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))


def _codes_worker(rank, world, port, n, m, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1706_10283_b200.dist import gather_codes, shard_range
        words = np.random.default_rng(3).integers(0, 2**32, (n + 7) // 8 * m, dtype=np.uint64).astype(np.uint32)
        r0, r1 = shard_range(n, world, rank)
        local = torch.from_numpy(words[r0 // 8 * m:(r1 + 7) // 8 * m].copy())
        whole, n_all = gather_codes(local, r1 - r0, m)
        np.save(os.path.join(out_dir, f"c{rank}.npy"), whole.numpy())
        assert n_all == n
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,world", [(1003, 2), (16, 2), (999, 3)])
def test_gather_codes_reassembles_database(tmp_path, n, world):
    """Row shards' layout-v1 words gathered on every rank equal the whole
    database's words (the exactness check of bench.py --gpus N)."""
    m = 4
    port = _free_port()
    mp.start_processes(_codes_worker, args=(world, port, n, m, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    words = np.random.default_rng(3).integers(0, 2**32, (n + 7) // 8 * m, dtype=np.uint64).astype(np.uint32)
    for r in range(world):
        np.testing.assert_array_equal(np.load(tmp_path / f"c{r}.npy"), words)
