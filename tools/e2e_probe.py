"""Timeline of the pipelined host search pieces on c2 (diagnostic)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_1706_10283_b200 as bolt
from synth import generators as G
dev = torch.device("cuda")
cfg = G.CONFIGS["c2"]
X = G.database(cfg); Q = G.queries(cfg)
train = G.training(cfg)
model = bolt.BoltModel.fit(torch.from_numpy(train).to(dev), cfg.m, torch.from_numpy(G.kmeans_init_all(cfg, len(train))).to(dev),
                           torch.from_numpy(G.calibration(cfg, train)).to(dev), 0, iters=cfg.kmeans_iters)
Xd = torch.from_numpy(X).to(dev); Qd = torch.from_numpy(Q).to(dev)
codes = model.encode(Xd); ql = model.luts(Qd)
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
for ch in (1, 4, 8):
    r = cfg.n // ch
    print(f"chunks={ch}: topk over {r} rows: {t(lambda: bolt.topk(codes[: r // 8 * 16], r, ql, 10, 0)):.3f} ms, "
          f"encode: {t(lambda: bolt.encode(Xd[:r], model.C)):.3f} ms")
Xh = torch.from_numpy(X).pin_memory(); Qh = torch.from_numpy(Q).pin_memory()
kh = torch.empty((cfg.nq, 10), dtype=torch.uint64).pin_memory()
for ch in (1, 2, 4, 8):
    hs = bolt.HostSearch(cfg.n, cfg.j, cfg.m, cfg.nq, 10, chunks=ch)
    print(f"HostSearch chunks={ch}: {t(lambda: hs(Xh, Qh, model.C, 0, model.a, model.b, kh), 3):.3f} ms")

# the same pipeline driven from Python (torch streams/events), per-piece timeline
cs = torch.cuda.Stream()
ch = 8
r = cfg.n // ch
ev_copy = [torch.cuda.Event(enable_timing=True) for _ in range(ch)]
ev_comp = [torch.cuda.Event(enable_timing=True) for _ in range(ch)]
e0 = torch.cuda.Event(enable_timing=True)
Xd2 = torch.empty_like(Xd)
codes2 = torch.empty_like(codes)
torch.cuda.synchronize()
e0.record()
cs.wait_event(e0)
with torch.cuda.stream(cs):
    for i in range(ch):
        Xd2[i * r:(i + 1) * r].copy_(Xh[i * r:(i + 1) * r], non_blocking=True)
        ev_copy[i].record(cs)
for i in range(ch):
    torch.cuda.current_stream().wait_event(ev_copy[i])
    cw = codes2[i * r // 8 * 16:(i + 1) * r // 8 * 16]
    bolt.encode(Xd2[i * r:(i + 1) * r], model.C, out=cw)
    bolt.topk(cw, r, ql, 10, 0, index_base=i * r)
    ev_comp[i].record()
torch.cuda.synchronize()
print("copy done at ", [round(e0.elapsed_time(e), 2) for e in ev_copy])
print("comp done at ", [round(e0.elapsed_time(e), 2) for e in ev_comp])

s2 = torch.cuda.Stream()
for ch in (1, 8):
    hs = bolt.HostSearch(cfg.n, cfg.j, cfg.m, cfg.nq, 10, chunks=ch)
    with torch.cuda.stream(s2):
        print(f"HostSearch chunks={ch} on a non-default stream: {t(lambda: hs(Xh, Qh, model.C, 0, model.a, model.b, kh), 3):.3f} ms")
