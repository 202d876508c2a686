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
a = p.parse_args()
dev = torch.device("cuda")
codes = bolt.pack_codes(torch.from_numpy(G.random_codes(a.n, a.m, 1)).to(dev))
ql = torch.from_numpy(G.random_qluts(a.nq, a.m, 2)).to(dev)
v = {"prmt": bolt.VARIANT_PRMT, "tc": bolt.VARIANT_TC, "auto": bolt.VARIANT_AUTO}[a.variant]
if a.what == "encode":
    X = torch.from_numpy(G.database(G.CONFIGS["c2"], a.n)).to(dev)
    C = torch.from_numpy(G.random_floats((a.m, 16, 128 // a.m), 3, 50.0) + 100).to(dev)
for _ in range(a.reps):
    if a.what == "topk":
        bolt.topk(codes, a.n, ql, a.k, 0, variant=v)
    elif a.what == "full":
        bolt.scan(codes, a.n, ql)
    elif a.what == "encode":
        bolt.encode(X, C)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(a.reps):
    if a.what == "topk":
        bolt.topk(codes, a.n, ql, a.k, 0, variant=v)
    elif a.what == "full":
        bolt.scan(codes, a.n, ql)
    elif a.what == "encode":
        bolt.encode(X, C)
e.record()
torch.cuda.synchronize()
print(f"{a.what} {a.variant} n={a.n} nq={a.nq} m={a.m}: {s.elapsed_time(e) / a.reps:.3f} ms")

if os.environ.get("BOLT_COUNTERS"):
    import ctypes
    buf = (ctypes.c_uint64 * 16)()
    bolt._lib.load().bolt_debug_counters(ctypes.cast(buf, ctypes.c_void_p), 16)
    names = ["prod_wait_empty", "epi_wait_tfull", "epi_wait+load", "mma_wait_full", "mma_wait_tempty",
             "tiles(leader)", "cta_cycles", "ctas", "epi_proc_cycles", "slow_entries", "inserts"]
    tiles = max(buf[5], 1)
    ctas = max(buf[7], 1)
    print("counters:", {n: int(buf[i]) for i, n in enumerate(names)})
    print(f"per tile: mma_wait_full={buf[3]/tiles:.0f} mma_wait_tempty={buf[4]/tiles:.0f} "
          f"cta_cycles/tile={buf[6]/ctas/(tiles/(ctas/2)):.0f} prod_wait_empty/tile={buf[0]/(tiles*2):.0f} "
          f"epi_wait_tfull/tile={buf[1]/(tiles*2):.0f} epi_wait+load/tile={buf[2]/(tiles*2):.0f} "
          f"epi_proc/warp-tile={buf[8]/(tiles*16):.0f} slow/lane-chunk={buf[9]/(tiles*16*4*32):.4f} "
          f"inserts/lane-chunk={buf[10]/(tiles*16*4*32):.4f}")
