#!/bin/bash
# production-shaped stage breakdown of the c2 scan (BOLT_XCONST builds: 2 no expansion, 3 + no filter,
# 4 filter only (no slow path), 11 MMA only); results of the variants are wrong by design
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for i in 1 2 3; do for L in libbolt.so libbolt_xc2.so libbolt_xc4.so libbolt_xc3.so libbolt_xc11.so; do
  echo "$L c2 $(BOLT_LIB=$L timeout 60 python tools/prof_scan.py --variant tc --reps 10 --config c2 | tail -1)"
done; done > gpurun_out/xc_times.txt 2>&1
