#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guard.py -q -x -k "lut or quant or c1 or c2 or fit or calib or host" > gpurun_out/lut_tests.log 2>&1
for i in 1 2 3; do for L in libbolt_lold.so libbolt.so; do
  echo "$L c2 $(BOLT_LIB=$L python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c 'import json,sys; d=json.loads([l for l in sys.stdin if l.startswith("{")][-1]); print(d["ms_per_step"], d["paper_context"]["lut_queries_per_s"])')"
done; done > gpurun_out/lut_times.txt 2>&1
