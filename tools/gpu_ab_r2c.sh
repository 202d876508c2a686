#!/bin/bash
# same-box A/B: lone-candidate slow path (libbolt_oc.so) on c2/c3; split small-batch accumulators (ss2/ss4) on Q = 1..8
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 120 python tools/prof_scan.py --variant tc --reps 2 --config c2 > gpurun_out/ab_smoke.txt 2>&1 || { echo "scan hung or failed" >> gpurun_out/ab_smoke.txt; exit 1; }
BOLT_LIB=libbolt_oc.so timeout 900 python -m pytest tests/test_gpu_ties.py tests/test_gpu_parity.py -q -x -k "tc or ties or topk or c2 or c3" > gpurun_out/oc_tests.log 2>&1; echo "oc tests rc=$?"
BOLT_LIB=libbolt_ss2.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ties.py -q -x -k "small or prmt or sweep or ties or topk" > gpurun_out/ss_tests.log 2>&1; echo "ss2 tests rc=$?"
for i in 1 2 3; do for L in libbolt.so libbolt_oc.so; do
  echo "$L c2 $(BOLT_LIB=$L timeout 60 python tools/prof_scan.py --variant tc --reps 10 --config c2 | tail -1)"
  echo "$L c3 $(BOLT_LIB=$L timeout 60 python tools/prof_scan.py --variant tc --reps 10 --config c3 --nq 1000 | tail -1)"
done; done > gpurun_out/oc_times.txt 2>&1
for i in 1 2; do for L in libbolt.so libbolt_ss2.so libbolt_ss4.so; do for q in 1 2 4 8; do
  echo "$L q$q $(BOLT_LIB=$L timeout 60 python tools/prof_scan.py --variant prmt --reps 10 --n 100000000 --nq $q | tail -1)"
done; done; done > gpurun_out/ss_times.txt 2>&1
cat gpurun_out/oc_times.txt gpurun_out/ss_times.txt; tail -2 gpurun_out/oc_tests.log gpurun_out/ss_tests.log
