#!/bin/bash
# same-box A/B of the e2e host search (tapered blocks in libbolt.so against libbolt_base.so)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "host or pipelined or e2e or search" > gpurun_out/e2e_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/e2e_tests.log
for i in 1 2 3; do for L in libbolt_base.so libbolt.so; do
  BOLT_LIB=$L python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 10 > gpurun_out/e2e_$L.json 2>/dev/null
  echo "$L $(python -c "import json;d=json.loads(open('gpurun_out/e2e_$L.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['e2e']['ms_per_step'],d['e2e']['value'])")"
done; done > gpurun_out/e2e_times.txt 2>&1
cat gpurun_out/e2e_times.txt
