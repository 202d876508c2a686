#!/bin/bash
# merge A/B: warp-per-query (libbolt) vs block tournament (libbolt_mblk) + tests
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guard.py -q -x -k "merge or c2 or c3 or topk_tc" > gpurun_out/m_tests.log 2>&1
for i in 1 2; do for L in libbolt_mblk.so libbolt.so; do
  echo "$L c2 $(BOLT_LIB=$L python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c 'import json,sys; d=json.loads([l for l in sys.stdin if l.startswith("{")][-1]); print(d["ms_per_step"])')"
  echo "$L c3 $(BOLT_LIB=$L python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c 'import json,sys; d=json.loads([l for l in sys.stdin if l.startswith("{")][-1]); print(d["ms_per_step"])')"
done; done > gpurun_out/m_times.txt 2>&1
