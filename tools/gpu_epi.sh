#!/bin/bash
# tcgen05 top-k epilogue warps A/B (libbolt = 16 for M <= 16, libbolt_e8 = 8)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 120 python tools/prof_scan.py --variant tc --reps 2 --config c2 > gpurun_out/e_smoke.txt 2>&1 || { echo "scan hung or failed" >> gpurun_out/e_smoke.txt; exit 1; }
timeout 900 python -m pytest tests/test_gpu_ties.py tests/test_gpu_parity.py -q -x -k "tc or ties or topk or c2 or c3" > gpurun_out/e_tests.log 2>&1
for i in 1 2; do for L in libbolt.so libbolt_e8.so; do
  echo "$L c2 $(BOLT_LIB=$L timeout 60 python tools/prof_scan.py --variant tc --reps 10 --config c2 | tail -1)"
  echo "$L q64 $(BOLT_LIB=$L timeout 60 python tools/prof_scan.py --variant tc --reps 10 --n 20000000 --nq 64 | tail -1)"
  echo "$L q1k $(BOLT_LIB=$L timeout 60 python tools/prof_scan.py --variant tc --reps 10 --n 20000000 --nq 1000 | tail -1)"
  echo "$L c5k100 $(BOLT_LIB=$L timeout 60 python tools/prof_scan.py --variant tc --reps 3 --n 20000000 --nq 16384 --k 100 | tail -1)"
done; done > gpurun_out/e_times.txt 2>&1
