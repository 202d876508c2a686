#!/bin/bash
# candidate-queue A/B (libbolt_f0 = immediate inserts, f2/f8 = flush thresholds; libbolt = flush 4)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 120 python tools/prof_scan.py --variant tc --reps 2 --config c2 > gpurun_out/q_smoke.txt 2>&1 || { echo "scan hung or failed" >> gpurun_out/q_smoke.txt; exit 1; }
timeout 900 python -m pytest tests/test_gpu_ties.py tests/test_gpu_parity.py -q -x -k "tc or ties or topk or encode or c2 or c3" > gpurun_out/q_tests.log 2>&1
for i in 1 2; do for L in libbolt.so libbolt_f0.so libbolt_f2.so libbolt_f8.so; do
  echo "$L c2 $(BOLT_LIB=$L timeout 60 python tools/prof_scan.py --variant tc --reps 10 --config c2 | tail -1)"
  echo "$L c3 $(BOLT_LIB=$L timeout 60 python tools/prof_scan.py --variant tc --reps 10 --config c3 | tail -1)"
  echo "$L q64 $(BOLT_LIB=$L timeout 60 python tools/prof_scan.py --variant tc --reps 10 --n 20000000 --nq 64 | tail -1)"
done; done > gpurun_out/q_times.txt 2>&1
