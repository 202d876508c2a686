#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
BOLT_LIB=libbolt_mm.so timeout 900 python -m pytest tests/test_gpu_ties.py tests/test_gpu_parity.py -q -x -k "tc or ties or topk or c2 or c3" > gpurun_out/k10_tests.log 2>&1
for i in 1 2 3; do for L in libbolt.so libbolt_mm.so; do
  echo "$L c2 $(BOLT_LIB=$L timeout 60 python tools/prof_scan.py --variant tc --reps 10 --config c2 | tail -1)"
  echo "$L c3 $(BOLT_LIB=$L timeout 60 python tools/prof_scan.py --variant tc --reps 10 --config c3 --nq 1000 | tail -1)"
done; done > gpurun_out/k10_times.txt 2>&1
