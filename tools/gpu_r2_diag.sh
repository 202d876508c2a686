#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
# 1) tie tests against the round-1 kernel (expected to FAIL) and the fixed one
BOLT_LIB=libbolt_old.so timeout 600 python -m pytest tests/test_gpu_ties.py -q -x 2>&1 | tail -25 > gpurun_out/ties_old.log
# 2) e2e trace output
timeout 900 python -m pytest tests/test_gpu_parity.py -q -s -k "all_queries" 2>&1 | tail -20 > gpurun_out/e2e.log
# 3) sparse MMA probe
./tools/probe_mma_sp_bin > gpurun_out/probe_mma_sp.txt 2>&1
./tools/probe_mma_sp_bin >> gpurun_out/probe_mma_sp.txt 2>&1
# 4) issue-only / stage diagnostics and counters on c2
for xm in 0 11 3 4; do echo "xmode $xm: $(BOLT_LIB=libbolt_x.so BOLT_TC_XMODE=$xm timeout 300 python tools/prof_scan.py --variant tc --reps 5 --config c2 | tail -1)"; done > gpurun_out/xmodes.txt 2>&1
echo "prefill: $(BOLT_LIB=libbolt_x.so BOLT_TC_XMODE=16 timeout 300 python tools/prof_scan.py --variant tc --reps 5 --config c2 --prefill | tail -1)" >> gpurun_out/xmodes.txt 2>&1
BOLT_LIB=libbolt_prof.so BOLT_COUNTERS=1 timeout 300 python tools/prof_scan.py --variant tc --reps 1 --config c2 > gpurun_out/counters_c2.txt 2>&1
timeout 300 python tools/prof_scan.py --variant tc --reps 5 --config c2 >> gpurun_out/xmodes.txt 2>&1
