#!/bin/bash
# same-box A/B of the small-batch PRMT kernel: libbolt_sxor.so (XOR selectors) vs libbolt.so
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 120 python tools/prof_scan.py --variant prmt --reps 2 --n 20000000 --nq 1 > gpurun_out/sm_smoke.txt 2>&1 || { echo "scan hung or failed" >> gpurun_out/sm_smoke.txt; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ties.py -q -x -k "small or prmt or sweep or ties or topk" > gpurun_out/sm_tests.log 2>&1
for i in 1 2; do for L in libbolt_sxor.so libbolt.so libbolt_spf4.so libbolt_spf8.so; do for q in 1 2 4 8 16; do
  echo "$L q$q $(BOLT_LIB=$L timeout 60 python tools/prof_scan.py --variant prmt --reps 10 --n 100000000 --nq $q | tail -1)"
done; done; done > gpurun_out/sm_times.txt 2>&1
for i in 1 2 3; do for L in libbolt.so libbolt_sth.so; do
  echo "$L c4 $(BOLT_LIB=$L timeout 60 python tools/prof_scan.py --variant tc --reps 10 --config c4 --nq 1024 --what dequant | tail -1)"
  echo "$L c4u16 $(BOLT_LIB=$L timeout 60 python tools/prof_scan.py --variant tc --reps 10 --config c4 --nq 1024 --what full | tail -1)"
done; done > gpurun_out/sth_times.txt 2>&1
