#!/bin/bash
# same-box A/B of the small-batch PRMT kernel: libbolt_sm3.so (BOLT_SMALL_IADD3: 3-input ALU adds) vs libbolt.so
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
BOLT_LIB=libbolt_sm3.so timeout 120 python tools/prof_scan.py --variant prmt --reps 2 --n 20000000 --nq 1 > gpurun_out/sm3_smoke.txt 2>&1 || { echo "scan hung or failed"; exit 1; }
BOLT_LIB=libbolt_sm3.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ties.py -q -x -k "small or prmt or sweep or ties or topk" > gpurun_out/sm3_tests.log 2>&1
tail -2 gpurun_out/sm3_tests.log
for i in 1 2 3; do for L in libbolt.so libbolt_sm3.so; do for q in 1 2 4 8; do
  echo "$L q$q $(BOLT_LIB=$L timeout 60 python tools/prof_scan.py --variant prmt --reps 10 --n 100000000 --nq $q | tail -1)"
done; done; done > gpurun_out/sm3_times.txt 2>&1
cat gpurun_out/sm3_times.txt
