#!/bin/bash
# same-box A/B of the tcgen05 scan: libbolt_base.so (HEAD) vs the working tree, plus parity
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 120 python tools/prof_scan.py --variant tc --reps 2 --config c2 > gpurun_out/ab_smoke.txt 2>&1 || { echo "scan hung or failed" >> gpurun_out/ab_smoke.txt; exit 1; }
timeout 900 python -m pytest tests/test_gpu_ties.py tests/test_gpu_parity.py -q -x -k "tc or ties or topk or c2 or c3 or full or dequant" > gpurun_out/ab_tests.log 2>&1
for i in 1 2 3; do for L in libbolt_base.so libbolt.so; do
  echo "$L c2 $(BOLT_LIB=$L timeout 60 python tools/prof_scan.py --variant tc --reps 10 --config c2 | tail -1)"
  echo "$L q64 $(BOLT_LIB=$L timeout 60 python tools/prof_scan.py --variant tc --reps 10 --n 20000000 --nq 64 | tail -1)"
  echo "$L c4 $(BOLT_LIB=$L timeout 60 python tools/prof_scan.py --variant tc --reps 10 --config c4 --nq 1024 --what dequant | tail -1)"
done; done > gpurun_out/ab_times.txt 2>&1
