#!/usr/bin/env python
"""Bolt hot-path benchmark (BASELINE.json metric: billion query x code
distances / s at M=16, J=128; % of roofline).

One step = the whole §8(a) path over one batch of BASELINE c2 (synthetic
SIFT1M-like: N=1,000,000 x J=128 fp32 database per GPU, Q=10,000 queries,
M=16, squared L2, top-10):
    encode(X)  ->  fused fp64 LUT build + u8 quantize(Q)  ->  scan + top-10
    [N > 1: NCCL all-gather of the [Q][10] u64 keys + merge]
value = distances (all ranks) / step time, inputs resident in HBM.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--variant auto|prmt|tc]
    python bench.py --impl reference ...      # the fp64 CPU oracle arm
    torchrun --nproc-per-node N bench.py --gpus N ...

Timing: CUDA events on the launching stream, W untimed warm-up steps, K timed
steps between barrier + synchronize, max over ranks.  The 512 MB fp32 database
that every step streams through the encoder exceeds the 126 MB L2.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from synth import generators as G  # noqa: E402

METRIC = "Bolt scan: billion query×code distances/sec (M=16, J=128); % of roofline"
UNIT = "Gdist/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="c2")
    p.add_argument("--variant", default="auto", choices=["auto", "prmt", "tc"])
    p.add_argument("--n", "--rows", dest="n", type=int, default=0, help="override rows per GPU (debug)")
    p.add_argument("--nq", "--queries", dest="nq", type=int, default=0, help="override queries (debug)")
    p.add_argument("--k", type=int, default=0, help="override top-k (debug, c5)")
    p.add_argument("--parallel", default="row", choices=["row", "query"],
                   help="c5 with N > 1: row-sharded database (all-gather + merge) or replicated database with "
                        "the queries split over the ranks (gather of disjoint slices, SURVEY 8(f4))")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--e2e-steps", type=int, default=3)
    p.add_argument("--e2e-chunks", type=int, default=16,
                   help="row blocks of the copy/compute-overlapped host search (c2 e2e: 4 / 8 / 16 blocks 10.16 / 9.90 / 9.76 ms against a 9.28 ms H2D floor)")
    p.add_argument("--no-graph", action="store_true", help="time the step eagerly instead of a CUDA graph")
    p.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                   help="gloo: CPU collectives, for testing the N > 1 glue with several ranks on one GPU "
                        "(never a measurement)")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int, period: float = 0.02):
        self.index, self.period = index, period
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover - no NVML
            self.nv = None
            self.err = str(e)
            self.max_mhz = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                fn = getattr(self.nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                    self.nv.nvmlDeviceGetCurrentClocksThrottleReasons
                r = fn(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.nv:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": getattr(self, "err", "")}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "sm_max_mhz": 1965.0}, "fallback"


def int8_peak():
    """Measured dense kind::i8 tensor rate (TOP/s at the max SM clock) from the
    issue-rate probe (profiles/r2/int8_peak.json), or None."""
    path = os.path.join(ROOT, "profiles", "r2", "int8_peak.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f)
    return None


def profile_traffic(variant: str):
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return d.get(variant)
    return None


# ------------------------------------------------------------- workload
def workload(args, rank):
    cfg = G.CONFIGS[args.config]
    n = args.n or cfg.n
    nq = args.nq or cfg.nq
    return cfg, n, nq


def cpu_baseline_sample(cfg, X, Q, C, a, b, metric, k, budget_s=20.0, dequant=False, noquant=False,
                        with_encode=True):
    """The fp64 oracle, as it stands, on the host cores: encode of the full
    database shard, tables of all queries, and the scan + top-k for a sample
    of queries over the full database; the scan time is scaled to all
    queries.  Returns (distances/s, threads, description)."""
    from oracle import oracle
    n, nq = len(X), len(Q)
    threads = oracle.num_threads()
    t0 = time.perf_counter()
    flat = oracle.encode(X, C)
    t_enc = time.perf_counter() - t0
    t0 = time.perf_counter()
    D = oracle.luts(Q, C, metric)
    ql = D.astype(np.float32) if noquant else oracle.quantize(D, a, b)
    t_lut = time.perf_counter() - t0
    # size the scan sample to the remaining budget (at least 8 queries)
    def scan_part(qn):
        if noquant:
            oracle.topk_f32(flat, ql[:qn], k, metric)
        elif k > 0:
            oracle.topk(flat, ql[:qn], k, metric)
        else:
            acc = oracle.scan(flat, ql[:qn])
            if dequant:
                oracle.dequant(acc, a, b)

    q8 = min(8, nq)
    t0 = time.perf_counter()
    scan_part(q8)
    t8 = time.perf_counter() - t0
    qs = int(max(q8, min(nq, q8 * max(1.0, (budget_s - t_enc - t_lut - t8) / max(t8, 1e-3)))))
    qs = min(qs, 1024, nq)
    t0 = time.perf_counter()
    scan_part(qs)
    t_scan = time.perf_counter() - t0
    t_full = (t_enc if with_encode else 0.0) + t_lut + t_scan * (nq / qs)
    desc = (f"oracle encode of all {n} rows ({t_enc:.2f} s{'' if with_encode else ', not counted: the step has no encode'}) + fp64 tables of all {nq} queries "
            f"({t_lut:.2f} s) + scan{f'/top-{k}' if k else (' + dequant' if dequant else '')} of {qs} queries "
            f"over all rows ({t_scan:.2f} s), "
            f"scan scaled x{nq / qs:.1f} to {nq} queries")
    return n * nq / t_full / 1e9, threads, desc


def near_tie_report(X, Q, C, a, b, metric, gwords, gql):
    """Stage parity of this run's GPU codes and quantized tables against the
    oracle (O3, O4 + O6) with the contract's near-tie rules:
    codes exact unless the oracle's relative top-2 gap is < 1e-5, table
    entries exact unless |t - rint t| < 1e-3.  Counts only; every mismatch
    that is not a near-tie is reported separately (it must be 0)."""
    from oracle import oracle
    n, m = len(X), C.shape[0]
    gcodes = oracle.unpack_v1(gwords, n, m)
    ocodes, gap = oracle.encode(X, C, with_gap=True)
    dc = gcodes != ocodes
    D = oracle.luts(Q, C, metric)
    oql, t = oracle.quantize(D, a, b, with_t=True)
    dt = gql != oql
    return {"codes_compared": int(dc.size), "code_near_ties": int((dc & (gap < 1e-5)).sum()),
            "code_mismatches_not_near_tie": int((dc & (gap >= 1e-5)).sum()),
            "table_entries_compared": int(dt.size),
            "table_near_ties": int((dt & (np.abs(t - np.rint(t)) < 1e-3)).sum()),
            "table_mismatches_not_near_tie": int((dt & (np.abs(t - np.rint(t)) >= 1e-3)).sum())}


def check_sharded(bolt, codes, n, m, ql, final, k, metric, variant, dev, nsample=256):
    """N > 1: rank 0 scans ALL rows (every rank's codes, gathered) on its one
    GPU for sampled queries and compares with the sharded, merged keys bit for
    bit (SURVEY 4 tier T3).  Raises on any difference."""
    import torch
    import torch.distributed as dist
    from paper_1706_10283_b200.dist import gather_codes
    whole, n_all = gather_codes(codes, n, m)
    nq = ql.shape[0]
    sample = np.random.default_rng(11).choice(nq, min(nsample, nq), replace=False)
    ok = True
    if dist.get_rank() == 0:
        idx = torch.from_numpy(sample).to(dev)
        ref = bolt.topk(whole, n_all, ql[idx].contiguous(), k, metric, variant=variant)
        ok = torch.equal(ref.view(torch.int64), final.view(torch.int64)[idx])
    del whole
    if not ok:
        raise SystemExit("sharded top-k differs from the single-GPU scan of all rows")
    return {"queries_checked": int(len(sample)), "rows": int(n_all),
            "bit_exact_vs_single_gpu_scan": bool(ok)}


# ------------------------------------------------------------------ ours
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1706_10283_b200 as bolt
    from paper_1706_10283_b200.dist import gather_keys

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    local = local % torch.cuda.device_count()  # --dist-backend gloo: several ranks may share one GPU
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.dist_backend == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    cfg, n, nq = workload(args, rank)
    metric = cfg.metrics[0]
    k = cfg.k
    variant = {"auto": bolt.VARIANT_AUTO, "prmt": bolt.VARIANT_PRMT, "tc": bolt.VARIANT_TC}[args.variant]

    # --- inputs (seeded, synthetic); rank r holds database rows [r*n, (r+1)*n)
    X = G.database(cfg, n, start=rank * n)
    Q = G.queries(cfg, nq)
    train = G.training(cfg)
    init = G.kmeans_init_all(cfg, len(train))
    calib = G.calibration(cfg, train)
    Xd = torch.from_numpy(X).to(dev)
    Qd = torch.from_numpy(Q).to(dev)

    # --- offline fit on the GPU (not timed): k-means + LUT quantizer
    train_d, init_d, calib_d = (torch.from_numpy(v).to(dev) for v in (train, init, calib))
    torch.cuda.synchronize()
    t_fit = time.perf_counter()
    model = bolt.BoltModel.fit(train_d, cfg.m, init_d, calib_d, metric, iters=cfg.kmeans_iters)
    torch.cuda.synchronize()
    fit_ms = (time.perf_counter() - t_fit) * 1e3  # reported beside the step, outside the timed region
    fit_rows = len(train)
    del train, train_d, init_d, calib_d

    words = bolt.codes_words(n, cfg.m)
    codes = torch.empty(words, dtype=torch.uint32, device=dev)
    ql = torch.empty((nq, cfg.m, 16), dtype=torch.uint8, device=dev)
    full = k == 0  # c1 / c4: full [N][Q] output (u16 sums, or dequantised fp32 for c4), no top-k
    ev_scan = []
    if full:
        b_sum = float(model.b.sum().item())
        out = torch.empty((n, nq), dtype=torch.float32 if cfg.cid == 4 else torch.uint16, device=dev)

        def scan_op():
            if cfg.cid == 4:
                bolt.scan_dequant(codes, n, ql, model.a, b_sum, out=out, variant=variant)
            else:
                bolt.scan(codes, n, ql, out=out, variant=variant)
    else:
        keys = torch.empty((nq, k), dtype=torch.uint64, device=dev)
        wsb = bolt.topk_workspace_bytes(n, cfg.m, nq, k, variant)
        ws = torch.empty(max(wsb, 8), dtype=torch.uint8, device=dev)
        final = torch.empty((nq, k), dtype=torch.uint64, device=dev) if world > 1 else keys

        def scan_op():
            bolt.topk(codes, n, ql, k, metric, index_base=rank * n, variant=variant, out=keys, workspace=ws)

    def step():
        bolt.encode(Xd, model.C, out=codes)
        bolt.build_quantized_luts(Qd, model.C, metric, model.a, model.b, out=ql)
        scan_op()
        if world > 1 and not full:
            bolt.topk_merge(gather_keys(keys), out=final)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # The single-GPU step is captured once into a CUDA graph (no host enqueue
    # jitter inside the timed region); with NCCL in the step it runs eagerly.
    graph, graph_note = None, "eager"
    if world == 1 and not args.no_graph:
        try:
            side = torch.cuda.Stream(dev)
            side.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(side):
                step()
            torch.cuda.current_stream(dev).wait_stream(side)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                step()
            torch.cuda.synchronize()
            g.replay()
            torch.cuda.synchronize()
            graph, graph_note = g, "cuda-graph replay"
        except Exception as e:  # pragma: no cover - capture unsupported
            graph_note = f"eager (graph capture failed: {e})"[:200]
    stream = torch.cuda.current_stream(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local if "CUDA_VISIBLE_DEVICES" not in os.environ else
                       int(os.environ["CUDA_VISIBLE_DEVICES"].split(",")[local]))
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with clk:
        t_start.record(stream)
        for _ in range(args.steps):
            if graph is not None:
                graph.replay()
            else:
                step()
        t_end.record(stream)
        torch.cuda.synchronize()
        # dominant kernel alone (scan + fused top-k), CUDA events on its stream
        for _ in range(args.steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            scan_op()
            e1.record(stream)
            ev_scan.append((e0, e1))
        torch.cuda.synchronize()
    # the encoder and the table build alone (context: the paper's per-core rates)
    p0, p1, p2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    p0.record(stream)
    bolt.encode(Xd, model.C, out=codes)
    p1.record(stream)
    bolt.build_quantized_luts(Qd, model.C, metric, model.a, model.b, out=ql)
    p2.record(stream)
    torch.cuda.synchronize()
    enc_ms, lut_ms = p0.elapsed_time(p1), p1.elapsed_time(p2)
    if world > 1:
        dist.barrier()
    ms_local = t_start.elapsed_time(t_end)
    scan_ms = sum(a.elapsed_time(b) for a, b in ev_scan) / len(ev_scan)
    ms = ms_local
    if world > 1:
        t = torch.tensor([ms_local, scan_ms], dtype=torch.float64, device=dev if args.dist_backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, scan_ms = float(t[0]), float(t[1])
    ms_step = ms / args.steps
    dists = world * n * nq
    value = dists / (ms_step * 1e-3) / 1e9

    exact = None
    if world > 1 and not full:  # the timed step's merged keys against one GPU's scan of all rows
        exact = check_sharded(bolt, codes, n, cfg.m, ql, final, k, metric, variant, dev)
        final_timed = final.clone()

    # --- e2e through the public host-buffer API (H2D of X, Q inside the timed region)
    e2e = None
    if args.e2e_steps > 0 and full:
        # full output through the public API: pinned host X, Q in, the [N][Q] result out
        Xh = torch.from_numpy(X).pin_memory()
        Qh = torch.from_numpy(Q).pin_memory()
        outh = torch.empty(out.shape, dtype=out.dtype).pin_memory()
        Xd2, Qd2 = torch.empty_like(Xd), torch.empty_like(Qd)

        def e2e_full():
            Xd2.copy_(Xh, non_blocking=True)
            Qd2.copy_(Qh, non_blocking=True)
            bolt.encode(Xd2, model.C, out=codes)
            bolt.build_quantized_luts(Qd2, model.C, metric, model.a, model.b, out=ql)
            scan_op()
            outh.copy_(out, non_blocking=True)

        e2e_full()
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(args.e2e_steps):
            e2e_full()
        a1.record(stream)
        torch.cuda.synchronize()
        e_ms = a0.elapsed_time(a1) / args.e2e_steps
        e2e = {"value": round(n * nq / (e_ms * 1e-3) / 1e9, 4), "unit": UNIT,
               "h2d_bytes_per_step": int(X.nbytes + Q.nbytes), "d2h_bytes_per_step": int(out.numel() * out.element_size()),
               "ms_per_step": round(e_ms, 3), "api": "bolt.encode / build_quantized_luts / scan* (pinned host buffers)"}
    elif args.e2e_steps > 0:
        hs = bolt.HostSearch(n, cfg.j, cfg.m, nq, k, device=dev, chunks=args.e2e_chunks)
        Xh = torch.from_numpy(X).pin_memory()
        Qh = torch.from_numpy(Q).pin_memory()
        kh = torch.empty((nq, k), dtype=torch.uint64).pin_memory()
        kd = torch.empty((nq, k), dtype=torch.uint64, device=dev)

        def e2e_step():
            hs(Xh, Qh, model.C, metric, model.a, model.b, kh, index_base=rank * n)
            if world > 1:
                kd.copy_(kh, non_blocking=True)
                bolt.topk_merge(gather_keys(kd), out=final)
                kh.copy_(final, non_blocking=True)

        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(args.e2e_steps):
            e2e_step()
        a1.record(stream)
        torch.cuda.synchronize()
        e_ms = a0.elapsed_time(a1) / args.e2e_steps
        if world > 1:
            t = torch.tensor([e_ms], dtype=torch.float64, device=dev if args.dist_backend == "nccl" else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t[0])
        if world > 1:  # the host-buffer path (global row indices via index_base) returns the same keys
            if not torch.equal(final.view(torch.int64), final_timed.view(torch.int64)):
                raise SystemExit("e2e (host-buffer) sharded keys differ from the device path's")
            exact["e2e_keys_equal"] = True
        e2e = {"value": round(dists / (e_ms * 1e-3) / 1e9, 4), "unit": UNIT,
               "h2d_bytes_per_step": int(X.nbytes + Q.nbytes),
               "d2h_bytes_per_step": int(nq * k * 8), "ms_per_step": round(e_ms, 3),
               "api": f"bolt_search_host{'_pipelined' if args.e2e_chunks > 1 else ''} (pinned host X, Q -> keys"
                      f"{f'; X in {args.e2e_chunks} blocks overlapped with encode + scan' if args.e2e_chunks > 1 else ''})"}


    # --- roofline of the dominant kernel (scan + fused top-k, or the full-output scan)
    peaks, peak_src = measured_peaks()
    if full:
        used_variant = "tc" if variant == bolt.VARIANT_TC or (variant == bolt.VARIANT_AUTO and nq >= 64 and
                                                              cfg.m in (8, 16, 32)) else "prmt"
        parts = 1
        roof = roofline_full(used_variant, n, cfg.m, nq, out.element_size(), scan_ms, peaks, peak_src)
    else:
        used_variant, parts = bolt.topk_plan(n, cfg.m, nq, k, variant)
        roof = roofline(used_variant, n, cfg.m, nq, scan_ms, peaks, peak_src, clk.summary())
    mname = "dot product" if metric == bolt.DOT else "squared L2"
    what = (f"full [N][Q] {'fp32 dequantised (acc/a + sum b)' if cfg.cid == 4 else 'u16'} output" if full
            else f"top-{k}")

    if rank == 0:
        out = {
            "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (seeded SIFT1M-like Gaussian mixture, SURVEY 8(d) c2 recipe)",
            "config": {"workload": f"{args.config}: N={n} rows/GPU x J={cfg.j} fp32, M={cfg.m} (4-bit codes), "
                                   f"Q={nq}, {mname}, {what}; step = encode + fp64 LUT build/quantize "
                                   f"+ scan" + ("" if full else "/top-k") +
                                   (" + NCCL all-gather + merge" if world > 1 and not full else ""),
                       "n_per_gpu": n, "nq": nq, "m": cfg.m, "j": cfg.j, "k": k,
                       "variant": used_variant, "scan_parts": parts, "timing": graph_note,
                       "l2": "inputs > L2: the 512 MB fp32 database is streamed by the encoder every step",
                       "parallelism": f"row-sharded dp{world}"},
            "roofline": roof,
            "e2e": e2e,
            "gpu_launches": args.steps * (3 + (1 if parts > 1 else 0) + (1 if world > 1 and not full else 0)),
            "fit": {"ms": round(fit_ms, 2), "train_rows": fit_rows, "kmeans_iters": cfg.kmeans_iters,
                    "note": "GPU k-means + alpha-grid calibration in the oracle's fp64 summation order "
                            "(bit-identical, serial per accumulator); offline, not part of the step"},
            "clocks": clk.summary(),
            "scan_ms": round(scan_ms, 4),
            "paper_context": {
                "encode_vectors_per_s": round(n / (enc_ms * 1e-3)), "lut_queries_per_s": round(nq / (lut_ms * 1e-3)),
                "paper_encode_vectors_per_s": 5e6, "paper_lut_queries_per_s": 6e6,
                "paper_hardware": "one thread of an Intel Core i7-4960HQ at 2.6 GHz (P:L357, P:L394, P:L396); "
                                  "context only, not the target"},
        }
        if exact is not None:
            out["exactness"] = exact
        if not args.no_cpu_baseline and world == 1:
            Ch, bh = model.C.cpu().numpy(), model.b.cpu().numpy()
            v, cores, desc = cpu_baseline_sample(cfg, X, Q, Ch, np.float32(model.a), bh, metric, k,
                                                 dequant=cfg.cid == 4)
            out["cpu_baseline"] = {"value": round(v, 6), "unit": UNIT, "cores": cores, "kind": "oracle",
                                   "cpu": cpu_model_name(), "sample": desc}
            out["near_ties"] = near_tie_report(X, Q, Ch, np.float32(model.a), bh, metric,
                                               codes.cpu().numpy(), ql.cpu().numpy())
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


def roofline_full(variant, n, m, nq, out_bytes, scan_ms, peaks, peak_src):
    """Full-output scan (c1 u16, c4 fp32): bound by the HBM write of the
    [N][Q] output.  Algorithmic bytes = codes (N*M/2) + u8 tables (Q*16*M) +
    output (N*Q*out_bytes); peak = measured copy bandwidth (MEASURED_PEAKS.json)."""
    t = scan_ms * 1e-3
    algo = n * m // 2 + nq * 16 * m + n * nq * out_bytes
    gbs = algo / t / 1e9
    peak = peaks["hbm_gbs"]
    return {"bound": "hbm", "achieved": round(gbs, 1), "peak": peak, "unit": "GB/s", "frac": round(gbs / peak, 4),
            "traffic": None, "algorithmic_bytes": algo,
            "peak_source": f"{peak_src} HBM copy bandwidth (MEASURED_PEAKS.json hbm_gbs)",
            "kernel": f"bolt_scan{'_dequant' if out_bytes == 4 else ''} ({variant})", "kernel_ms": round(scan_ms, 4),
            "tensor_view": {"int8_tops": round(2.0 * 16 * m * n * nq / t / 1e12, 1)} if variant == "tc" else None}


def roofline(variant, n, m, nq, scan_ms, peaks, peak_src, clocks):
    """Dominant kernel = the scan with fused top-k (bolt_topk; includes the tiny
    split-N partial merge).  PRMT: integer-ALU bound, algorithmic work
    2*M int ops per distance (M lookups + M adds); peak = 148 SM
    x 128 int lanes/clk (alu + fma pipes, 1 warp-instruction/clk/SMSP issue)
    x max SM clock (B300_MICROARCH.md pipe rates).  TC: tensor
    bound, one-hot contraction executes 2*16*M int8 ops per distance; peak =
    dense int8 = 2 x measured bf16 (nominal 4.5 / 2.25 PF ratio)."""
    t = scan_ms * 1e-3
    dists = n * nq
    sm_mhz = peaks.get("sm_max_mhz", 1965.0)
    if variant == "tc":
        ops = 2.0 * 16 * m * dists
        achieved = ops / t
        bf16x2 = 2.0 * peaks["bf16_tflops"] * 1e12
        probe = int8_peak()
        if probe:  # the measured kind::i8 issue rate (report against it)
            peak = probe["int8_dense_tops"] * 1e12
            src = (f"measured tcgen05 kind::i8 issue rate, {probe['dense_cycles_per_instr_k32']} cycles per "
                   f"256x256x32 pair instruction at {probe['sm_mhz']} MHz (profiles/r2/int8_peak.json)")
        else:
            peak, src = bf16x2, f"int8 dense = 2 x {peak_src} bf16 ({peaks['bf16_tflops']} TFLOP/s)"
        return {"bound": "tensor", "achieved": round(achieved / 1e12, 2), "peak": round(peak / 1e12, 2),
                "unit": "TOP/s", "frac": round(achieved / peak, 4), "traffic": profile_traffic("tc"),
                "peak_source": src,
                "frac_vs_2x_bf16": round(achieved / bf16x2, 4),  # context: 2 x the driver's measured bf16 peak
                "nominal_int8_frac": round(achieved / 4.5e15, 4),  # context: B200 dense int8 4.5 POP/s
                "kernel": "bolt_topk (tcgen05 scan + top-k)", "kernel_ms": round(scan_ms, 4)}
    ops = 2.0 * m * dists
    peak = 148 * 128 * sm_mhz * 1e6
    achieved = ops / t
    return {"bound": "alu", "achieved": round(achieved / 1e12, 3), "peak": round(peak / 1e12, 3),
            "unit": "Tops/s", "frac": round(achieved / peak, 4), "traffic": profile_traffic("prmt"),
            "peak_source": f"148 SM x 128 int lanes/clk x {sm_mhz:.0f} MHz ({peak_src} sm_max_mhz); DESIGN.md",
            "kernel": "bolt_topk (PRMT scan + fused top-k)", "kernel_ms": round(scan_ms, 4),
            "hbm_view": {"algorithmic_bytes": n * m // 2 + nq * m * 16 + nq * 10 * 8,
                         "gbs": round((n * m // 2 + nq * m * 16) / t / 1e9, 1)}}


# ------------------------------------------------------------------- c5
def c2_model(bolt, dev):
    """c2's codebooks and LUT quantizer, fitted on the GPU (offline, untimed);
    c5 and the sweep reuse them (SURVEY 8(d) c5 recipe)."""
    import torch
    cfg2 = G.CONFIGS["c2"]
    train = G.training(cfg2)
    return bolt.BoltModel.fit(torch.from_numpy(train).to(dev), cfg2.m,
                              torch.from_numpy(G.kmeans_init_all(cfg2, len(train))).to(dev),
                              torch.from_numpy(G.calibration(cfg2, train)).to(dev), cfg2.metrics[0],
                              iters=cfg2.kmeans_iters)


def c5_codes(bolt, model, r0, n, dev, chunk=1 << 20):
    """Rows [r0, r0 + n) of c5's database: generated on the GPU
    (synth/gen_gpu.cu, Philox keyed by global row) in 1M-row chunks and encoded
    at once, so the 51 GB fp32 database never exists whole."""
    import torch
    from synth import gpu as synth_gpu
    m = model.m
    mu = torch.from_numpy(G.c5_means()).to(dev)
    codes = torch.empty(max(bolt.codes_words(n, m), 1), dtype=torch.uint32, device=dev)
    xbuf = torch.empty((chunk, 128), dtype=torch.float32, device=dev)
    for c0 in range(0, n, chunk):
        rows = min(chunk, n - c0)
        synth_gpu.c5_rows(r0 + c0, rows, mu, xbuf[:rows])
        w0 = c0 // 8 * m
        bolt.encode(xbuf[:rows], model.C, out=codes[w0:w0 + bolt.codes_words(rows, m)])
    del xbuf
    torch.cuda.synchronize()
    return codes


def c5_cpu_baseline(codes, n, m, qlh, k, metric, nq, budget_s=20.0):
    """The oracle's scan + top-k (O12) over the full GPU code set for sampled
    queries, extrapolated to all queries ('c5: sampled queries
    over the full 100M codes, extrapolated')."""
    from oracle import oracle
    t0 = time.perf_counter()
    flat = oracle.unpack_v1(codes, n, m)
    t_unpack = time.perf_counter() - t0
    t0 = time.perf_counter()
    oracle.topk(flat, qlh[:1], k, metric)
    t1 = time.perf_counter() - t0
    qs = int(max(1, min(len(qlh) - 1, (budget_s - t1) / max(t1, 1e-3))))
    t0 = time.perf_counter()
    if qs > 1:
        oracle.topk(flat, qlh[1:1 + qs], k, metric)
    t_s = (time.perf_counter() - t0 + t1) / (qs + 1)
    desc = (f"oracle scan + top-{k} of {qs + 1} sampled queries over all {n} codes ({t_s:.2f} s per query; "
            f"unpacking the codes took {t_unpack:.1f} s, not counted), extrapolated x{nq / (qs + 1):.0f} to {nq} "
            "queries; tables and encoding not counted (extrapolated)")
    return n / t_s / 1e9, oracle.num_threads(), desc


def run_c5(args):
    """BASELINE c5: N = 1e8 rows (c2 mixture, generated + encoded on device,
    row-sharded over the ranks: contiguous ranges of ceil(N/W/8)*8 rows),
    Q = 65,536, squared L2, top-100.  One step = fused fp64 LUT build/quantize
    of all queries (every rank, redundantly) + scan/top-k of the local shard
    (tcgen05 lists of 32, merged + verified) [+ NCCL all-gather of [Q][100]
    keys + merge for W > 1].  Encoding is setup."""
    import torch
    import torch.distributed as dist

    import paper_1706_10283_b200 as bolt
    from paper_1706_10283_b200.dist import gather_keys

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    local = local % torch.cuda.device_count()  # --dist-backend gloo: several ranks may share one GPU
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.dist_backend == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    cfg = G.CONFIGS["c5"]
    n_total = args.n or cfg.n
    nq, k, metric, m = args.nq or cfg.nq, args.k or cfg.k, cfg.metrics[0], cfg.m
    qmode = args.parallel == "query" and world > 1
    from paper_1706_10283_b200.dist import gather_query_slices, query_range
    if qmode:  # every rank holds the whole database and a slice of the queries
        r0, n = 0, n_total
        qa, qb = query_range(nq, world, rank)
    else:
        shard = -(-n_total // world // 8) * 8 if world > 1 else n_total
        r0 = rank * shard
        n = max(0, min(shard, n_total - r0))
        qa, qb = 0, nq
    model = c2_model(bolt, dev)
    t0 = time.perf_counter()
    codes = c5_codes(bolt, model, r0, n, dev)
    setup_s = time.perf_counter() - t0
    Q = G.queries(cfg, nq)[qa:qb]
    nql = qb - qa
    Qd = torch.from_numpy(Q).to(dev)
    ql = torch.empty((nql, m, 16), dtype=torch.uint8, device=dev)
    keys = torch.empty((nql, k), dtype=torch.uint64, device=dev)
    ws = torch.empty(max(bolt.topk_workspace_bytes(n, m, nql, k), 8), dtype=torch.uint8, device=dev)
    final = torch.empty((nq, k), dtype=torch.uint64, device=dev) if world > 1 else keys

    def scan_op():
        bolt.topk(codes, n, ql, k, metric, index_base=r0, out=keys, workspace=ws)

    def step():
        bolt.build_quantized_luts(Qd, model.C, metric, model.a, model.b, out=ql)
        scan_op()
        if qmode:
            final.copy_(gather_query_slices(keys, nq))
        elif world > 1:
            bolt.topk_merge(gather_keys(keys), out=final)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local if "CUDA_VISIBLE_DEVICES" not in os.environ else
                       int(os.environ["CUDA_VISIBLE_DEVICES"].split(",")[local]))
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev = []
    with clk:
        t_start.record(stream)
        for _ in range(args.steps):
            step()
        t_end.record(stream)
        torch.cuda.synchronize()
        for _ in range(max(1, min(args.steps, 3))):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            scan_op()
            e1.record(stream)
            ev.append((e0, e1))
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = t_start.elapsed_time(t_end)
    scan_ms = sum(a.elapsed_time(b) for a, b in ev) / len(ev)
    if world > 1:
        t = torch.tensor([ms, scan_ms], dtype=torch.float64, device=dev if args.dist_backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, scan_ms = float(t[0]), float(t[1])
    ms_step = ms / args.steps
    value = n_total * nq / (ms_step * 1e-3) / 1e9

    # e2e through the public API: queries from pinned host memory in, keys out
    Qh = torch.from_numpy(Q).pin_memory()
    kh = torch.empty((nq, k), dtype=torch.uint64).pin_memory()

    def e2e_step():
        Qd.copy_(Qh, non_blocking=True)
        step()
        kh.copy_(final, non_blocking=True)

    e2e = None
    if args.e2e_steps > 0:
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        a0.record(stream)
        for _ in range(args.e2e_steps):
            e2e_step()
        a1.record(stream)
        torch.cuda.synchronize()
        e_ms = a0.elapsed_time(a1) / args.e2e_steps
        if world > 1:
            t = torch.tensor([e_ms], dtype=torch.float64, device=dev if args.dist_backend == "nccl" else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t[0])
        e2e = {"value": round(n_total * nq / (e_ms * 1e-3) / 1e9, 4), "unit": UNIT,
               "h2d_bytes_per_step": int(Q.nbytes), "d2h_bytes_per_step": int(nq * k * 8),
               "ms_per_step": round(e_ms, 3),
               "api": "bolt.build_quantized_luts / topk [/ all-gather + topk_merge] (pinned host Q in, keys out); "
                      "the database is device-resident (generated + encoded on the GPU)"}

    exact = None
    if world > 1 and qmode:
        # every rank holds all rows: rank 0 rescans sampled queries of the whole set
        sample = np.random.default_rng(11).choice(nq, 64, replace=False)
        ok = True
        if rank == 0:
            qs = torch.from_numpy(G.queries(cfg, nq)[sample]).to(dev)
            qls = bolt.build_quantized_luts(qs, model.C, metric, model.a, model.b)
            ref = bolt.topk(codes, n, qls, k, metric)
            ok = torch.equal(ref.view(torch.int64), final.view(torch.int64)[torch.from_numpy(sample).to(dev)])
        if not ok:
            raise SystemExit("query-sharded top-k differs from the single-GPU scan")
        exact = {"queries_checked": 64, "rows": n, "bit_exact_vs_single_gpu_scan": True}
    elif world > 1:
        exact = check_sharded(bolt, codes, n, m, ql, final, k, metric, bolt.VARIANT_AUTO, dev, nsample=64)

    peaks, peak_src = measured_peaks()
    variant, parts = bolt.topk_plan(n, m, nql, k)
    # a ~1 s kernel: the sustained (power-capped) tensor peak applies if the
    # clocks show the cap; at full clocks with no throttle reason, the burst one
    ck = clk.summary()
    capped = "sw_power_cap" in ck.get("reasons", []) or (ck.get("sm_mhz") or 0) < 0.9 * (ck.get("sm_max_mhz") or 1)
    pk = dict(peaks)
    if capped and "bf16_tflops_sustained" in peaks:
        pk["bf16_tflops"] = peaks["bf16_tflops_sustained"]
    roof = roofline(variant, n, m, nql, scan_ms, pk, peak_src + (" sustained" if capped else " burst"), ck)
    if rank == 0:
        out = {
            "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 3),
            "higher_is_better": True, "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
            "dtype": "u8", "data": "synthetic (c5: c2 mixture generated on the GPU by Philox4x32-10, SURVEY 8(d))",
            "config": {"workload": f"c5: N={n_total} rows total ({n} on rank 0), J=128, M=16, Q={nq}, "
                                   f"squared L2, top-{k}; step = fp64 LUT build/quantize + scan/top-{k}"
                                   + ((" + NCCL all-gather of the query slices (replicated database)" if qmode
                                       else " + NCCL all-gather + merge") if world > 1 else "")
                                   + "; database generated + encoded once at setup "
                                   f"({setup_s:.1f} s, untimed)",
                       "n_per_gpu": n, "nq": nq, "m": m, "j": 128, "k": k, "variant": variant,
                       "scan_parts": parts, "timing": "eager (the top-100 path synchronises once on its flag count)",
                       "l2": "codes 800 MB / W > L2 at W <= 4; compute-bound (SURVEY 8(d))",
                       "parallelism": f"{'query' if qmode else 'row'}-sharded dp{world}"},
            "roofline": roof, "e2e": e2e,
            "gpu_launches": args.steps * (4 + (2 if world > 1 else 0)),  # LUT, scan, merge, verify [+ gather, merge]
            "clocks": clk.summary(), "scan_ms": round(scan_ms, 3),
        }
        if exact is not None:
            out["exactness"] = exact
        if not args.no_cpu_baseline and world == 1:
            v, cores, desc = c5_cpu_baseline(codes.cpu().numpy(), n, m, ql[:65].cpu().numpy(), k, metric, nql)
            out["cpu_baseline"] = {"value": round(v, 6), "unit": UNIT, "cores": cores, "kind": "oracle",
                                   "cpu": cpu_model_name(), "sample": desc}
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------- No Quantize (f3)
def run_noquant(args):
    """SURVEY 8(f3) "Bolt No Quantize" on c2: step = encode + fp32
    tables (bolt_build_luts) + fp32-table scan with fused top-10
    (bolt_topk_f32).  The paper keeps the variant only as an accuracy
    reference ("it sacrifices Bolt's high speed"); its roofline is the
    shared-memory lookup rate: one 4-byte LDS per lookup, M per distance,
    at 32 lookups / clk / SM (128 B/clk crossbar, B300_MICROARCH.md)."""
    import torch

    import paper_1706_10283_b200 as bolt

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    cfg = G.CONFIGS["c2"]
    n, nq, k, metric = args.n or cfg.n, args.nq or cfg.nq, cfg.k, cfg.metrics[0]
    model = c2_model(bolt, dev)
    Xd = torch.from_numpy(G.database(cfg, n)).to(dev)
    Qd = torch.from_numpy(G.queries(cfg, nq)).to(dev)
    codes = torch.empty(bolt.codes_words(n, cfg.m), dtype=torch.uint32, device=dev)
    keys = torch.empty((nq, k), dtype=torch.uint64, device=dev)
    luts = {}

    def step():
        bolt.encode(Xd, model.C, out=codes)
        luts["D"] = bolt.build_luts(Qd, model.C, metric)
        bolt.topk_f32(codes, n, luts["D"], k, metric, out=keys)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream(dev)
    clk = ClockSampler(0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(args.steps):
            bolt.topk_f32(codes, n, luts["D"], k, metric, out=keys)
        s1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    scan_ms = s0.elapsed_time(s1) / args.steps
    peaks, peak_src = measured_peaks()
    sm_mhz = peaks.get("sm_max_mhz", 1965.0)
    lookups = n * nq * cfg.m / (scan_ms * 1e-3)
    peak = 148 * 32 * sm_mhz * 1e6
    out = {"metric": METRIC, "value": round(n * nq / (ms * 1e-3) / 1e9, 4), "unit": UNIT, "n_gpus": 1,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f32",
           "data": "synthetic (seeded SIFT1M-like Gaussian mixture, SURVEY 8(d) c2 recipe)",
           "config": {"workload": f"c2 No Quantize (P:L390): N={n}, J=128, M={cfg.m}, Q={nq}, squared L2, top-{k} "
                                  "over fp32 tables; step = encode + fp32 tables + fp32 scan/top-k",
                      "n_per_gpu": n, "nq": nq, "m": cfg.m, "k": k},
           "roofline": {"bound": "smem", "achieved": round(lookups / 1e12, 3), "peak": round(peak / 1e12, 3),
                        "unit": "T lookups/s", "frac": round(lookups / peak, 4), "traffic": None,
                        "peak_source": f"148 SM x 32 LDS lanes/clk x {sm_mhz:.0f} MHz ({peak_src} sm_max_mhz)",
                        "kernel": "bolt_topk_f32", "kernel_ms": round(scan_ms, 4)},
           "clocks": clk.summary(), "gpu_launches": args.steps * 4}
    print(json.dumps(out))


# ------------------------------------------------------------------ sweep
SWEEP_Q = (1, 2, 4, 8, 16, 32, 64, 128, 256)


def run_sweep(args):
    """Small-batch regime (SURVEY 8(d) 'sweep'): c5's database (the c2
    mixture, generated on the GPU by synth/gen_gpu.cu in 1M-row chunks and
    encoded with the c2 model; N = 1e8 rows = 800 MB of codes, > L2) scanned
    with top-10 for Q = 1 .. 256 queries of c5.  Reports per Q the scan time,
    distances/s and the code-stream bandwidth N*M/2 / t (the HBM roofline of
    small batches: BASELINE north_star 'achieved HBM GB/s for small query
    batches')."""
    import torch

    import paper_1706_10283_b200 as bolt

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    cfg2, cfg5 = G.CONFIGS["c2"], G.CONFIGS["c5"]
    n = args.n or cfg5.n
    model = c2_model(bolt, dev)
    codes = c5_codes(bolt, model, 0, n, dev)
    Qall = torch.from_numpy(G.queries(cfg5, max(SWEEP_Q))).to(dev)
    peaks, peak_src = measured_peaks()
    stream = torch.cuda.current_stream(dev)
    code_bytes = n * cfg2.m // 2
    rows_out = []
    clk = ClockSampler(0)
    with clk:
        for q in SWEEP_Q:
            ql = bolt.build_quantized_luts(Qall[:q].contiguous(), model.C, cfg2.metrics[0], model.a, model.b)
            keys = torch.empty((q, 10), dtype=torch.uint64, device=dev)
            ws = torch.empty(max(bolt.topk_workspace_bytes(n, cfg2.m, q, 10), 8), dtype=torch.uint8, device=dev)
            variant, parts = bolt.topk_plan(n, cfg2.m, q, 10)
            for _ in range(args.warmup):
                bolt.topk(codes, n, ql, 10, cfg2.metrics[0], out=keys, workspace=ws)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                bolt.topk(codes, n, ql, 10, cfg2.metrics[0], out=keys, workspace=ws)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.steps
            rows_out.append({"q": q, "variant": variant, "parts": parts, "ms": round(ms, 4),
                             "gdist_s": round(n * q / (ms * 1e-3) / 1e9, 2),
                             "code_gbs": round(code_bytes / (ms * 1e-3) / 1e9, 1),
                             "hbm_frac": round(code_bytes / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"], 4)})
    r1 = rows_out[0]
    out = {"metric": METRIC, "value": r1["gdist_s"], "unit": UNIT, "n_gpus": 1, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": r1["ms"], "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "u8",
           "data": "synthetic (c5: c2 mixture generated on the GPU by Philox4x32-10, SURVEY 8(d))",
           "config": {"workload": f"sweep: N={n} rows (c5 database, {code_bytes / 1e6:.0f} MB of codes > L2), "
                                  f"M=16, J=128, squared L2, top-10, Q in {list(SWEEP_Q)}; value = Q=1; step = "
                                  "scan + top-k (tables prebuilt)", "n_per_gpu": n, "m": 16, "j": 128, "k": 10,
                      "l2": "codes 800 MB > 126 MB L2 (streamed from HBM every scan)"},
           "roofline": {"bound": "hbm", "achieved": round(code_bytes / (r1["ms"] * 1e-3) / 1e9, 1),
                        "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": r1["hbm_frac"], "traffic": None,
                        "peak_source": f"{peak_src} HBM copy bandwidth", "kernel": f"bolt_topk ({r1['variant']}), Q=1"},
           "sweep": rows_out, "clocks": clk.summary(),
           "gpu_launches": args.steps * len(SWEEP_Q) * 3}
    print(json.dumps(out))


# ------------------------------------------------------------- reference
def cpu_model_name() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def oracle_model(cfg, metric):
    """The model the GPU arm fits (same training rows, k-means init and
    iterations, calibration queries), fitted by the oracle -- the GPU k-means
    and calibration are bit-identical to it (tests/test_gpu_parity.py), so
    both arms search with the same codebooks and quantizer."""
    from oracle import oracle
    src = G.CONFIGS["c2"] if cfg.name == "c5" else cfg
    train = G.training(src)
    C = oracle.fit(train, src.m, G.kmeans_init_all(src, len(train)), src.kmeans_iters)
    a, b, _ = oracle.fit_quantizer(G.calibration(src, train), C, metric)
    return C, a, b


def run_reference(args):
    """The fp64 CPU oracle as it stands, on the host cores (rank 0 only).

    Each step runs the workload's own path on the oracle -- encode of the
    database rows (configs whose GPU step encodes), fp64 tables + quantize and
    the scan / top-k (or full scan + dequant) of the step's queries over those
    rows -- and is timed as it runs: value = distances the step computed /
    its measured time, ms_per_step = the measured mean.  When all queries do
    not fit the run's time budget, each step takes the next slice of the
    query set (stated in config); the 1e8-row c5 / sweep database never exists
    on the host, so those steps scan a 1M-row sample of the same mixture."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle
    # sweep: c5's database at Q = 1; c2nq: c2 with the fp32 tables (O13/O14)
    name = {"sweep": "c5", "c2nq": "c2"}.get(args.config, args.config)
    cfg = G.CONFIGS[name]
    n, nq = args.n or cfg.n, args.nq or (1 if args.config == "sweep" else cfg.nq)
    metric, k = cfg.metrics[0], (10 if args.config == "sweep" else cfg.k)
    noquant, dequant = args.config == "c2nq", cfg.cid == 4
    with_encode = args.config not in ("c5", "sweep")
    n_s = min(n, 1_000_000)
    X = G.database(cfg if name != "c5" else G.CONFIGS["c2"], n_s)
    Q = G.queries(cfg, nq)
    t0 = time.perf_counter()
    C, a, b = oracle_model(cfg, metric)
    fit_s = time.perf_counter() - t0

    def step(q0, qn):
        """One timed step over queries [q0, q0 + qn) (wrapping)."""
        idx = (np.arange(qn) + q0) % nq
        Qs = Q[idx]
        t = time.perf_counter()
        flat = oracle.encode(X, C) if with_encode else step.flat
        D = oracle.luts(Qs, C, metric)
        ql = D.astype(np.float32) if noquant else oracle.quantize(D, a, b)
        if noquant:
            oracle.topk_f32(flat, ql, k, metric)
        elif k > 0:
            oracle.topk(flat, ql, k, metric)
        else:
            acc = oracle.scan(flat, ql)
            if dequant:
                oracle.dequant(acc, a, b)
        return time.perf_counter() - t

    step.flat = None if with_encode else oracle.encode(X, C)
    # size the step: all queries if (steps + warmup) of them fit the budget
    budget = 240.0
    q8 = min(8, nq)
    t8 = step(0, q8)
    t_fixed = 0.0
    if with_encode:
        t = time.perf_counter()
        oracle.encode(X, C)
        t_fixed = time.perf_counter() - t
    per_q = max(t8 - t_fixed, 1e-6) / q8
    runs = max(1, args.steps + args.warmup)
    qs = nq if runs * (t_fixed + per_q * nq) <= budget else \
        int(min(nq, max(q8, (budget / runs - t_fixed) / per_q)))
    times = []
    for i in range(args.warmup + args.steps):
        t = step(i * qs, qs)
        if i >= args.warmup:
            times.append(t)
    t_step = statistics.mean(times)
    value = n_s * qs / t_step / 1e9
    cores = oracle.num_threads()
    desc = (f"per step: {'oracle encode of all ' + str(n_s) + ' rows + ' if with_encode else ''}fp64 tables"
            f"{'' if noquant else ' + quantize'} of {qs} of the {nq} queries + "
            f"{'fp32-table scan/top-' + str(k) if noquant else ('scan/top-' + str(k) if k else 'full scan' + (' + dequant' if dequant else ''))}"
            f" over {n_s} rows; {'all queries every step' if qs == nq else 'successive query slices'}"
            + (f"; rows: a {n_s}-row sample of the {n}-row database (same mixture)" if n_s < n else "")
            + f"; model fitted by the oracle as the GPU arm fits it ({fit_s:.1f} s, untimed)")
    out = {"impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_step * 1e3, 1),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64/int64",
           "data": "synthetic",
           "config": {"workload": f"{args.config}: N={n} x J={cfg.j}, M={cfg.m}, Q={nq}, top-{k} (fp64 CPU oracle)",
                      "n_per_gpu": n, "nq": nq, "rows_per_step": n_s, "queries_per_step": qs,
                      "same_model_as_gpu_arm": True},
           "cpu_baseline": {"value": round(value, 6), "unit": UNIT, "cores": cores, "kind": "oracle",
                            "cpu": cpu_model_name(), "sample": desc},
           "e2e": {"value": round(value, 6), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


if __name__ == "__main__":
    a = parse()
    if a.config == "sweep" and a.impl != "reference":
        run_sweep(a)
    elif a.config == "c5" and a.impl != "reference":
        run_c5(a)
    elif a.config == "c2nq" and a.impl != "reference":
        run_noquant(a)
    elif a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
