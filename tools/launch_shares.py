"""Per-kernel share of the bench step from an ncu launch list (gpu__time_duration.sum CSV).
    python tools/launch_shares.py launches.csv [steps=2] [start=encode] [end=merge_kernel] > shares.json
Each of the last `steps` steps is the run of kernels from a `start` kernel to
the next `end` kernel (c5: start=build_luts end=verify_lists)."""
import collections
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID") + 1
hdr = rows[start - 1]
ix = {h: i for i, h in enumerate(hdr)}
launches = [(r[ix["Kernel Name"]], float(r[ix["Metric Value"]]), r[ix["Metric Unit"]]) for r in rows[start:]
            if len(r) == len(hdr) and r[ix["Metric Name"]] == "gpu__time_duration.sum"]
scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}
start_k = sys.argv[3] if len(sys.argv) > 3 else "encode"
end_k = sys.argv[4] if len(sys.argv) > 4 else "merge_kernel"
enc = [i for i, (k, _, _) in enumerate(launches) if start_k in k]
# complete steps only: a start kernel followed by an end kernel before the next start
# (bench.py's e2e/roofline legs launch partial sequences after the timed steps)
bounds = enc[1:] + [len(launches)]
complete = []
for e, nxt in zip(enc, bounds):
    ends = [j for j in range(e, nxt) if end_k in launches[j][0]]
    if ends:
        complete.append((e, ends[0]))
tot = collections.defaultdict(float)
for e, last in complete[-steps:]:  # one step = start kernel .. the first end kernel after it
    for k, v, u in launches[e:last + 1]:
        tot[k.split("(")[0]] += v * scale.get(u, 1e-6)
step = sum(tot.values()) / steps
print(json.dumps({"source": sys.argv[1], "steps": steps, "step_ms": round(step, 4),
                  "share": {k: round(v / steps / step, 4) for k, v in tot.items()}}, indent=1))
