#!/bin/bash
# small-batch shared-bound refresh cadence A/B on the sweep (c5 data): libbolt (every 8) vs se4/se8 (every iteration early) vs se33 (always)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for i in 1 2; do for L in libbolt.so libbolt_se4.so libbolt_se8.so libbolt_se33.so; do
  echo "$L $(BOLT_LIB=$L timeout 300 python bench.py --config sweep --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads([l for l in sys.stdin if l.startswith("{")][-1]); print(" ".join("q%d=%.3f" % (r["q"], r["ms"]) for r in d["sweep"]))')"
done; done > gpurun_out/early_times.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ties.py -q -x -k "small or prmt or ties or topk" > gpurun_out/early_tests.log 2>&1
