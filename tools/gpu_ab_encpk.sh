#!/bin/bash
# Encoder A/B: libbolt_encpk.so (BOLT_ENC_PACK=1: codes staged as bytes in shared memory, packed once per stage) vs libbolt.so
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for l in libbolt_encpk.so; do
  BOLT_LIB=$l timeout 60 python tools/prof_scan.py --what encode --reps 2 --config c2 --expanded > gpurun_out/encpk_smoke.txt 2>&1 || { echo "$l hung or failed"; tail -5 gpurun_out/encpk_smoke.txt; exit 1; }
  BOLT_LIB=$l timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "encode or c1 or host or code_buffer or c2 or c3 or c4" > gpurun_out/encpk_tests.log 2>&1
  tail -3 gpurun_out/encpk_tests.log
done
for i in 1 2 3; do for c in c2 c3 c4; do for l in libbolt.so libbolt_encpk.so; do
  echo "$c $l $(BOLT_LIB=$l timeout 60 python tools/prof_scan.py --what encode --reps 10 --config $c --expanded | tail -1)"
done; done; done > gpurun_out/encpk.txt 2>&1
cat gpurun_out/encpk.txt
