#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
BOLT_LIB=libbolt_prof.so BOLT_COUNTERS=1 timeout 300 python tools/prof_scan.py --variant sp --reps 1 --config c2 > gpurun_out/sp_diag.txt 2>&1
BOLT_LIB=libbolt_prof.so BOLT_COUNTERS=1 BOLT_TC_XMODE=0 timeout 300 python tools/prof_scan.py --variant sp --reps 1 --config c3 --nq 1000 >> gpurun_out/sp_diag.txt 2>&1
