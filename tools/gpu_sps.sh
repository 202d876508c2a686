#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ties.py -q -x -k "topk_sp or sparse" > gpurun_out/sps_tests.log 2>&1
for q in 8 16 32 64; do for v in prmt tc sp; do echo "q=$q $v $(timeout 300 python tools/prof_scan.py --variant $v --reps 5 --n 20000000 --nq $q | tail -1)"; done; done > gpurun_out/sps_times.txt 2>&1
for q in 32 64; do for xm in 1 3 4; do echo "q=$q sp xmode $xm $(BOLT_LIB=libbolt_x.so BOLT_TC_XMODE=$xm timeout 300 python tools/prof_scan.py --variant sp --reps 5 --n 20000000 --nq $q | tail -1)"; done; done >> gpurun_out/sps_times.txt 2>&1
