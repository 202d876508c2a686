#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 120 python tools/prof_scan.py --variant tc --reps 2 --config c2 > gpurun_out/c2_smoke.txt 2>&1 || { echo "hung or failed" >> gpurun_out/c2_smoke.txt; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ties.py tests/test_gpu_guard.py -q -x -k "topk_tc or ties or constant or binary or c2_full or c3_full or large_k or guard or c5" > gpurun_out/c2_tests.log 2>&1
for i in 1 2; do timeout 300 python tools/prof_scan.py --variant tc --reps 10 --config c2; done > gpurun_out/c2_times.txt 2>&1
timeout 300 python tools/prof_scan.py --variant tc --reps 5 --config c3 --nq 1000 >> gpurun_out/c2_times.txt 2>&1
timeout 300 python tools/prof_scan.py --variant tc --reps 5 --n 20000000 --nq 64 >> gpurun_out/c2_times.txt 2>&1
timeout 300 python tools/prof_scan.py --variant tc --reps 3 --n 10000000 --nq 65536 --k 100 >> gpurun_out/c2_times.txt 2>&1
timeout 300 python tools/prof_scan.py --variant tc --reps 3 --n 10000000 --nq 65536 --k 10 >> gpurun_out/c2_times.txt 2>&1
