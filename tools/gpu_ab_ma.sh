#!/bin/bash
# same-box A/B of a tcgen05 top-k variant (libbolt_$V.so) against libbolt.so: parity subset, then c2 / c3 / 20M x 16k top-100
V=${1:-ma}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 120 python tools/prof_scan.py --variant tc --reps 2 --config c2 > gpurun_out/ab_smoke.txt 2>&1 || { echo "scan hung or failed" >> gpurun_out/ab_smoke.txt; exit 1; }
BOLT_LIB=libbolt_$V.so timeout 900 python -m pytest tests/test_gpu_ties.py tests/test_gpu_parity.py -q -x -k "tc or ties or topk or c2 or c3" > gpurun_out/${V}_tests.log 2>&1; echo "$V tests rc=$?"; tail -1 gpurun_out/${V}_tests.log
for i in 1 2 3; do for L in libbolt.so libbolt_$V.so; do
  echo "$L c2 $(BOLT_LIB=$L timeout 60 python tools/prof_scan.py --variant tc --reps 10 --config c2 | tail -1)"
  echo "$L c3 $(BOLT_LIB=$L timeout 60 python tools/prof_scan.py --variant tc --reps 10 --config c3 --nq 1000 | tail -1)"
  echo "$L k100 $(BOLT_LIB=$L timeout 60 python tools/prof_scan.py --variant tc --reps 5 --n 20000000 --nq 16384 --k 100 | tail -1)"
done; done > gpurun_out/${V}_times.txt 2>&1
cat gpurun_out/${V}_times.txt
