#!/bin/bash
# mbarrier suspend-time hint A/B (libbolt = no hint; mh1k/mh10k/mh100k = 1/10/100 us)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 120 BOLT_LIB=libbolt_mh10k.so python tools/prof_scan.py --variant tc --reps 2 --config c2 > gpurun_out/h_smoke.txt 2>&1
BOLT_LIB=libbolt_mh10k.so timeout 120 python tools/prof_scan.py --variant tc --reps 2 --config c2 >> gpurun_out/h_smoke.txt 2>&1 || { echo "scan hung or failed" >> gpurun_out/h_smoke.txt; exit 1; }
for i in 1 2 3; do for L in libbolt.so libbolt_mh1k.so libbolt_mh10k.so libbolt_mh100k.so; do
  echo "$L c2 $(BOLT_LIB=$L timeout 60 python tools/prof_scan.py --variant tc --reps 10 --config c2 | tail -1)"
  echo "$L q64 $(BOLT_LIB=$L timeout 60 python tools/prof_scan.py --variant tc --reps 10 --n 20000000 --nq 64 | tail -1)"
  echo "$L c4 $(BOLT_LIB=$L timeout 60 python tools/prof_scan.py --variant tc --reps 10 --config c4 --nq 1024 --what dequant | tail -1)"
  echo "$L k100 $(BOLT_LIB=$L timeout 60 python tools/prof_scan.py --variant tc --reps 3 --n 20000000 --nq 16384 --k 100 | tail -1)"
  echo "$L enc $(BOLT_LIB=$L timeout 60 python tools/prof_scan.py --what encode --reps 10 --config c2 | tail -1)"
done; done > gpurun_out/h_times.txt 2>&1
