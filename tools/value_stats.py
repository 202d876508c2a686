"""Distribution of the scan sums near the top-k threshold (ties), c2/c3 data.

    python tools/value_stats.py [--config c2] [--nq 64]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1706_10283_b200 as bolt
from synth import generators as G

p = argparse.ArgumentParser()
p.add_argument("--config", default="c2")
p.add_argument("--nq", type=int, default=64)
a = p.parse_args()
dev = torch.device("cuda")
cfg = G.CONFIGS[a.config]
train = G.training(cfg)
model = bolt.BoltModel.fit(torch.from_numpy(train).to(dev), cfg.m,
                           torch.from_numpy(G.kmeans_init_all(cfg, len(train))).to(dev),
                           torch.from_numpy(G.calibration(cfg, train)).to(dev), cfg.metrics[0],
                           iters=cfg.kmeans_iters)
codes = model.encode(torch.from_numpy(G.database(cfg, cfg.n)).to(dev))
ql = model.luts(torch.from_numpy(G.queries(cfg, a.nq)).to(dev))
acc = bolt.scan(codes, cfg.n, ql).to(torch.int32)  # [n][nq]
if cfg.metrics[0] == bolt.DOT:
    acc = 0xFFFF - acc
k = cfg.k
print(f"a={model.a:.4g} alpha={model.alpha} b_sum={float(model.b.sum()):.4g}")
for q in range(min(a.nq, 16)):
    v = acc[:, q]
    s, _ = torch.sort(v)
    T = int(s[k - 1])
    print(f"q{q}: min={int(s[0])} kth={T} n(<=T)={int((v <= T).sum())} n(==T)={int((v == T).sum())} "
          f"q1e-4={int(s[100])} q1e-3={int(s[1000])} q1e-2={int(s[10000])} median={int(s[len(s)//2])}")
