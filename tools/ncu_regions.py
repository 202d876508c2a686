"""Group an ncu SASS source page into runs of equal execution count (basic blocks).
python tools/ncu_regions.py rep.ncu-rep [min_share] [kernel-regex]"""
import collections
import csv
import io
import re
import subprocess
import sys

cmd = ["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"]
if len(sys.argv) > 3:
    cmd += ["--kernel-name", f"regex:{sys.argv[3]}", "--launch-count", "1"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr) and r[idx["Instructions Executed"]] != "Instructions Executed"]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.005
ti = sum(float(r[idx["Instructions Executed"]] or 0) for r in data)
ts = sum(float(r[idx["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
prev = None
runs = []
for r in data:
    c = float(r[idx["Instructions Executed"]] or 0)
    smp = float(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    m = re.match(r'\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)', r[1])
    o = m.group(2) if m else '?'
    if prev is None or abs(c - prev) > 0.02 * max(c, prev, 1):
        runs.append([r[0], 0, c, 0.0, 0.0, collections.Counter()])
        prev = c
    run = runs[-1]
    run[1] += 1
    run[3] += c
    run[4] += smp
    run[5][o] += 1
for a, n, c, acc, smp, ops in runs:
    if acc / ti > thr or smp / ts > thr:
        print(f"{a[-6:]} n={n:4d} execs={c:11.0f} inst={acc / ti * 100:5.1f}% samples={smp / ts * 100:5.1f}%",
              ops.most_common(5))
