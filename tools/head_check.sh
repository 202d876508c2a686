cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_head.log 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2_head.json 2> gpurun_out/bench_c2_head.err
for i in 1 2; do for d in "" "--expanded"; do echo "$d $(timeout 120 python tools/prof_scan.py --what encode --reps 10 --config c2 $d | tail -1)"; done; done > gpurun_out/enc_times_head.txt 2>&1
