#!/bin/bash
# sparse tcgen05 top-k: correctness first, then c2 / c3 timings against the dense kernel
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "topk_sp" > gpurun_out/sp_tests.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ties.py -q -x -k "sparse" >> gpurun_out/sp_tests.log 2>&1
for v in tc sp; do timeout 300 python tools/prof_scan.py --variant $v --reps 5 --config c2; done > gpurun_out/sp_times.txt 2>&1
for v in tc sp; do timeout 300 python tools/prof_scan.py --variant $v --reps 5 --config c3 --nq 1000; done >> gpurun_out/sp_times.txt 2>&1
for xm in 1 3 4 9 0; do echo "sp xmode $xm: $(BOLT_LIB=libbolt_x.so BOLT_TC_XMODE=$xm timeout 300 python tools/prof_scan.py --variant sp --reps 3 --config c2 | tail -1)"; done >> gpurun_out/sp_times.txt 2>&1
