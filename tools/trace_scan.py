"""Per-tile timeline of the tcgen05 scan, cluster 0 (libbolt_x.so, BOLT_TC_XMODE |= 64).

    BOLT_LIB=libbolt_x.so BOLT_TC_XMODE=64 python tools/trace_scan.py [--config c2]
clock64 columns per CTA rank: 0 MMA after full wait, 1 after tempty wait, 2 after
commits (rank 0 only); 3+p producer warp p empty seen, 7+p arrived; 11+w
epilogue warp w tfull seen, 19+w released, 27+w processing done.
"""
import ctypes
import os
import sys

import numpy as np

sys.argv += ["--reps", "1"] if "--reps" not in sys.argv else []
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import prof_scan  # noqa: E402,F401  (runs the scan)

import paper_1706_10283_b200 as bolt  # noqa: E402

NC, T, W = 24, 512, 40
buf = (ctypes.c_uint64 * (NC + 2 * T * W))()
bolt._lib.load().bolt_debug_counters(ctypes.cast(buf, ctypes.c_void_p), NC + 2 * T * W)
tr = np.frombuffer(buf, dtype=np.uint64)[NC:].reshape(2, T, W).astype(np.int64)
nt = int((tr[0, :, 2] > 0).sum())
if nt < 8:
    sys.exit(f"trace has {nt} tiles (need BOLT_TC_XMODE & 64 and libbolt_x.so)")
tr = tr[:, :nt]
med = lambda x: float(np.median(x))  # noqa: E731
r0 = tr[0]
commit = r0[:, 2]
print(f"tiles traced: {nt}")
print(f"MMA commit cadence          : {med(np.diff(commit)):7.0f} cyc/tile")
print(f"MMA wait full (commit->full): {med(r0[1:, 0] - commit[:-1]):7.0f}")
print(f"MMA wait tempty             : {med(r0[:, 1] - r0[:, 0]):7.0f}")
print(f"MMA issue (tempty->commit)  : {med(commit - r0[:, 1]):7.0f}")
for rk in (0, 1):
    r = tr[rk]
    pe, pa = r[:, 3:7], r[:, 7:11]
    ef, er, ed = r[:, 11:19], r[:, 19:27], r[:, 27:35]
    print(f"-- rank {rk}")
    print(f"  producer expansion (empty seen->arrive) per warp: {[round(med(pa[:, i] - pe[:, i])) for i in range(4)]}")
    print(f"  producer arrive spread (max-min over warps)     : {med(pa.max(1) - pa.min(1)):.0f}")
    print(f"  producer empty-seen spacing (per tile)          : {med(np.diff(pe[:, 0])):.0f}")
    print(f"  epi load (tfull seen->release) med warp         : {med(np.median(er - ef, 1)):.0f}")
    print(f"  epi processing med-warp / max-warp              : {med(np.median(ed - er, 1)):.0f} / {med((ed - er).max(1)):.0f}")
    print(f"  epi idle done(t)->tfull seen(t+1) med warp      : {med(np.median(ef[1:] - ed[:-1], 1)):.0f}")
    print(f"  epi tfull seen spread over warps                : {med(ef.max(1) - ef.min(1)):.0f}")
    if rk == 0:
        print(f"  commit(t)->epi tfull seen (min/max warp)        : {med(ef.min(1) - commit):.0f} / {med(ef.max(1) - commit):.0f}")
        print(f"  last release(t)->MMA tempty end(t+2)            : {med(r0[2:, 1] - er[:-2].max(1)):.0f}")
        print(f"  last producer arrive(t)->MMA full end(t)        : {med(r0[:, 0] - pa.max(1)):.0f}")
np.save(os.environ.get("TRACE_OUT", "gpurun_out/trace.npy"), tr)
