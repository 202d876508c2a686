#!/bin/bash
# large-k (group-list) timing: c5-like and the full c5 scan
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "large_k or c5" > gpurun_out/c5k_tests.log 2>&1
timeout 300 python tools/prof_scan.py --variant tc --reps 3 --n 10000000 --nq 65536 --k 100 > gpurun_out/c5k_times.txt 2>&1
timeout 600 python tools/prof_scan.py --variant tc --reps 2 --n 100000000 --nq 65536 --k 100 >> gpurun_out/c5k_times.txt 2>&1
