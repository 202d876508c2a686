#!/bin/bash
# Encoder A/B: libbolt_encl3.so (BOLT_ENC_LEAN=3: runner-up test and argmin on the FMA pipe) vs libbolt.so
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for l in libbolt_encl3.so; do
  BOLT_LIB=$l timeout 60 python tools/prof_scan.py --what encode --reps 2 --config c2 --expanded > gpurun_out/encl3_smoke.txt 2>&1 || { echo "$l hung or failed"; exit 1; }
  BOLT_LIB=$l timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "encode or c1 or host or code_buffer" > gpurun_out/encl3_tests.log 2>&1
  tail -2 gpurun_out/encl3_tests.log
done
for i in 1 2 3; do for c in c2 c3 c4; do for l in libbolt.so libbolt_encl3.so; do
  echo "$c $l $(BOLT_LIB=$l timeout 60 python tools/prof_scan.py --what encode --reps 10 --config $c --expanded | tail -1)"
done; done; done > gpurun_out/encl3.txt 2>&1
cat gpurun_out/encl3.txt
