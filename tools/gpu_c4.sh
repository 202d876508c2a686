cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "scan_tc or dequant or c4 or c1" > gpurun_out/c4_tests.log 2>&1
timeout 900 python -m pytest tests/test_gpu_guard.py -q -x > gpurun_out/guard_tests.log 2>&1
for i in 1 2; do timeout 300 python tools/prof_scan.py --variant tc --reps 10 --config c4 --nq 1024 --what dequant; done > gpurun_out/c4_times.txt 2>&1
timeout 600 python bench.py --config c4 --steps 10 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
