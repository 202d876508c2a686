#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "encode" > gpurun_out/enc_tests.log 2>&1
for i in 1 2; do for d in "" "--direct"; do echo "$d $(timeout 300 python tools/prof_scan.py --what encode --reps 10 --config c2 $d | tail -1)"; done; done > gpurun_out/enc_times.txt 2>&1
echo "minb3 $(BOLT_LIB=libbolt_x.so BOLT_ENC_MINB3=1 timeout 300 python tools/prof_scan.py --what encode --reps 10 --config c2 | tail -1)" >> gpurun_out/enc_times.txt
echo "x-minb2 $(BOLT_LIB=libbolt_x.so timeout 300 python tools/prof_scan.py --what encode --reps 10 --config c2 | tail -1)" >> gpurun_out/enc_times.txt
for d in "" "--direct"; do echo "c4 $d $(timeout 300 python tools/prof_scan.py --what encode --reps 10 --config c4 $d | tail -1)"; done >> gpurun_out/enc_times.txt 2>&1
