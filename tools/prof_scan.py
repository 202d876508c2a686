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
