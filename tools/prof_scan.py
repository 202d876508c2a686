"""Launch the hot kernels once on c2-shaped synthetic inputs (for ncu).

    python tools/prof_scan.py [--nq 10000] [--n 1000000] [--variant prmt|tc] [--what topk|encode|full]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1706_10283_b200 as bolt
from synth import generators as G

p = argparse.ArgumentParser()
p.add_argument("--n", type=int, default=1_000_000)
p.add_argument("--nq", type=int, default=10_000)
p.add_argument("--m", type=int, default=16)
p.add_argument("--k", type=int, default=10)
p.add_argument("--variant", default="prmt")
p.add_argument("--what", default="topk")
p.add_argument("--reps", type=int, default=2)
p.add_argument("--prefill", action="store_true")
p.add_argument("--direct", action="store_true", help="encode: the direct-difference kernel")
p.add_argument("--expanded", action="store_true", help="encode: the register-loading expanded-distance kernel")
p.add_argument("--config", default="", help="use a BASELINE config's real pipeline data (c2, c3)")
a = p.parse_args()
dev = torch.device("cuda")
if a.config:
    # the bench's data: seeded config database, GPU-fitted model, encoded codes, fused tables
    cfg = G.CONFIGS[a.config]
    a.m, a.k = cfg.m, cfg.k
    a.n = min(a.n, cfg.n)
    train = G.training(cfg)
    model = bolt.BoltModel.fit(torch.from_numpy(train).to(dev), cfg.m,
                               torch.from_numpy(G.kmeans_init_all(cfg, len(train))).to(dev),
                               torch.from_numpy(G.calibration(cfg, train)).to(dev), cfg.metrics[0],
                               iters=cfg.kmeans_iters)
    codes = model.encode(torch.from_numpy(G.database(cfg, a.n)).to(dev))
    ql = model.luts(torch.from_numpy(G.queries(cfg, a.nq)).to(dev))
    metric = cfg.metrics[0]
else:
    codes = bolt.pack_codes(torch.from_numpy(G.random_codes(a.n, a.m, 1)).to(dev))
    ql = torch.from_numpy(G.random_qluts(a.nq, a.m, 2)).to(dev)
    metric = 0
v = {"prmt": bolt.VARIANT_PRMT, "tc": bolt.VARIANT_TC, "tcs": bolt.VARIANT_TCS, "sp": bolt.VARIANT_SP,
     "auto": bolt.VARIANT_AUTO}[a.variant]
if a.what == "encode":
    if a.config:  # the bench's database and GPU-fitted codebooks
        X = torch.from_numpy(G.database(cfg, a.n)).to(dev)
        C = model.C
    else:
        X = torch.from_numpy(G.database(G.CONFIGS["c2"], a.n)).to(dev)
        C = torch.from_numpy(G.random_floats((a.m, 16, 128 // a.m), 3, 50.0) + 100).to(dev)
full_out = None
if a.what in ("full", "dequant"):
    full_out = torch.empty((a.n, a.nq), dtype=torch.uint16 if a.what == "full" else torch.float32, device=dev)
ws = None
prefill = lambda: None  # noqa: E731
if a.prefill:
    # diagnostic (libbolt_x.so, BOLT_TC_XMODE & 16): shared thresholds start at
    # the exact final k-th value (the best any threshold scheme could reach)
    _, parts = bolt.topk_plan(a.n, a.m, a.nq, a.k, v)
    ws = torch.empty(bolt.topk_workspace_bytes(a.n, a.m, a.nq, a.k, v), dtype=torch.uint8, device=dev)
    keys = bolt.topk(codes, a.n, ql, a.k, metric, variant=v)
    kth = (keys[:, a.k - 1].view(torch.int64) >> 48) & 0xFFFF
    gthr = (0xFFFF - kth).to(torch.int32)
    off = parts * a.nq * a.k * 8

    def prefill():
        ws[off:off + 4 * a.nq].view(torch.int32).copy_(gthr)


def once():
    if a.what == "topk":
        bolt.topk(codes, a.n, ql, a.k, metric, variant=v, workspace=ws)
    elif a.what == "full":
        bolt.scan(codes, a.n, ql, out=full_out, variant=v)
    elif a.what == "dequant":
        bolt.scan_dequant(codes, a.n, ql, 0.5, 1.0, out=full_out, variant=v)
    elif a.what == "encode":
        bolt.encode(X, C, variant=bolt.ENCODE_DIRECT if a.direct else (bolt.ENCODE_EXPANDED if a.expanded
                                                                         else bolt.ENCODE_AUTO))


for _ in range(a.reps):
    prefill()
    once()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
tot = 0.0
for _ in range(a.reps):
    prefill()
    s.record()
    once()
    e.record()
    torch.cuda.synchronize()
    tot += s.elapsed_time(e)
print(f"{a.what} {a.variant} n={a.n} nq={a.nq} m={a.m}: {tot / a.reps:.3f} ms" + (" (prefilled thresholds)" if a.prefill else ""))

if os.environ.get("BOLT_COUNTERS"):
    import ctypes
    buf = (ctypes.c_uint64 * 24)()
    bolt._lib.load().bolt_debug_counters(ctypes.cast(buf, ctypes.c_void_p), 24)
    names = ["prod_wait_empty", "epi_wait_tfull", "epi_wait+load", "mma_wait_full", "mma_wait_tempty",
             "tiles(leader)", "cta_cycles", "ctas", "epi_proc_cycles", "slow_entries", "inserts",
             "warp_slow_chunks", "wslow_t<8", "wslow_t<64", "wslow_t<256", "wslow_t>=256", "warp_cand_iters", "lanes_no_thr_t>=1", "sum_thr_t1", "-", "-", "-", "-", "-"]
    if a.variant == "sp":
        names = names[:16] + ["sp_group_entries", "sp_query_entries", "sp_candidates", "sp_list_changes",
                              "sp_warp_tiles", "sp_groups_t<16", "sp_groups_t<128", "sp_groups_t>=128"]
    tiles = max(buf[5], 1)
    ctas = max(buf[7], 1)
    print("counters:", {n: int(buf[i]) for i, n in enumerate(names)})
    print(f"per tile: mma_wait_full={buf[3]/tiles:.0f} mma_wait_tempty={buf[4]/tiles:.0f} "
          f"cta_cycles/tile={buf[6]/ctas/(tiles/(ctas/2)):.0f} prod_wait_empty/tile={buf[0]/(tiles*2):.0f} "
          f"epi_wait_tfull/tile={buf[1]/(tiles*2):.0f} epi_wait+load/tile={buf[2]/(tiles*2):.0f} "
          f"epi_proc/warp-tile={buf[8]/(tiles*16):.0f} slow/lane-chunk={buf[9]/(tiles*16*4*32):.4f} "
          f"inserts/lane-chunk={buf[10]/(tiles*16*4*32):.4f} warp-slow/warp-chunk={buf[11]/(tiles*16*4):.4f} "
          f"cand-iters/warp-slow={buf[16]/max(buf[11],1):.2f}")
