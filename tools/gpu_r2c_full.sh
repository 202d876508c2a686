#!/bin/bash
# GPU suite + the benches of the tcgen05 top-k workloads at the working tree
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "c2 rc=$?"
python bench.py --config c3 --steps 10 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "c3 rc=$?"
python bench.py --config c5 --steps 3 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "c5 rc=$?"
tail -2 gpurun_out/gpu_tests.log
for f in c2 c3 c5; do python -c "import json;d=json.loads(open('gpurun_out/bench_$f.json').read().strip().splitlines()[-1]);print('$f',d['ms_per_step'],d['roofline']['kernel_ms'],d['roofline']['frac'])"; done
