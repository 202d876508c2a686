#!/bin/bash
# Round-2b: whole-row TMA encoder (tests + times) and the c2 epilogue shared-word diagnostics.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 60 python tools/prof_scan.py --what encode --reps 2 --config c2 --expanded > gpurun_out/enc_smoke.txt 2>&1 || { echo "encode hung or failed" >> gpurun_out/enc_smoke.txt; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "encode or c1 or host or code_buffer" > gpurun_out/enc_tests.log 2>&1
for i in 1 2; do for d in "--direct" "--expanded"; do for c in c2 c3 c4; do echo "$c $d $(timeout 120 python tools/prof_scan.py --what encode --reps 10 --config $c $d | tail -1)"; done; done; done > gpurun_out/enc_times.txt 2>&1
for x in 0 3 4 132 128 256; do echo "xmode=$x $(BOLT_LIB=libbolt_x.so BOLT_TC_XMODE=$x timeout 60 python tools/prof_scan.py --variant tc --reps 5 --config c2 | tail -1)"; done > gpurun_out/xmode_c2.txt 2>&1
for x in 0 256; do echo "xmode=$x $(BOLT_LIB=libbolt_x.so BOLT_TC_XMODE=$x timeout 60 python tools/prof_scan.py --variant tc --reps 5 --config c2 | tail -1)"; done >> gpurun_out/xmode_c2.txt 2>&1
