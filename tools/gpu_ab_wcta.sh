#!/bin/bash
# MMA issuer's full / tempty waits at CTA scope (no per-tile L1 invalidate) vs acquire.cluster
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
BOLT_LIB=libbolt_wcta.so timeout 120 python tools/prof_scan.py --variant tc --reps 2 --config c2 > gpurun_out/w_smoke.txt 2>&1 || { echo "scan hung or failed" >> gpurun_out/w_smoke.txt; exit 1; }
cp paper_1706_10283_b200/libbolt_wcta.so /tmp/libbolt_wcta.so
for i in 1 2 3; do for L in libbolt.so libbolt_wcta.so; do
  echo "$L c2 $(BOLT_LIB=$L timeout 60 python tools/prof_scan.py --variant tc --reps 10 --config c2 | tail -1)"
  echo "$L c3 $(BOLT_LIB=$L timeout 60 python tools/prof_scan.py --variant tc --reps 10 --config c3 --nq 1000 | tail -1)"
  echo "$L c4 $(BOLT_LIB=$L timeout 60 python tools/prof_scan.py --variant tc --reps 10 --config c4 --nq 1024 --what dequant | tail -1)"
  echo "$L k100 $(BOLT_LIB=$L timeout 60 python tools/prof_scan.py --variant tc --reps 3 --n 20000000 --nq 16384 --k 100 | tail -1)"
done; done > gpurun_out/w_times.txt 2>&1
BOLT_LIB=libbolt_wcta.so timeout 900 python -m pytest tests/test_gpu_ties.py tests/test_gpu_parity.py -q -x -k "tc or ties or topk or c2 or c3 or full or dequant" > gpurun_out/w_tests.log 2>&1
