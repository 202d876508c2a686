#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 60 python tools/prof_scan.py --what encode --reps 2 --config c2 > gpurun_out/enc_smoke.txt 2>&1 || { echo "encode hung or failed" >> gpurun_out/enc_smoke.txt; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "encode or c1 or host or code_buffer" > gpurun_out/enc_tests.log 2>&1
for i in 1 2; do for d in "" "--expanded"; do echo "$d $(timeout 120 python tools/prof_scan.py --what encode --reps 10 --config c2 $d | tail -1)"; done; done > gpurun_out/enc_times.txt 2>&1
for d in "" "--direct"; do echo "c4 $d $(timeout 120 python tools/prof_scan.py --what encode --reps 10 --config c4 $d | tail -1)"; done >> gpurun_out/enc_times.txt 2>&1
