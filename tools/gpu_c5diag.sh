#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for xm in 0 4 11; do echo "c5-like xmode $xm: $(BOLT_LIB=libbolt_x.so BOLT_TC_XMODE=$xm timeout 300 python tools/prof_scan.py --variant tc --reps 2 --n 10000000 --nq 65536 --k 100 | tail -1)"; done > gpurun_out/c5diag.txt 2>&1
echo "release: $(timeout 300 python tools/prof_scan.py --variant tc --reps 2 --n 10000000 --nq 65536 --k 100 | tail -1)" >> gpurun_out/c5diag.txt
BOLT_LIB=libbolt_prof.so BOLT_COUNTERS=1 timeout 300 python tools/prof_scan.py --variant tc --reps 1 --n 10000000 --nq 65536 --k 100 >> gpurun_out/c5diag.txt 2>&1
