#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python tools/prof_scan.py --variant tc --reps 2 --config c2 > gpurun_out/p1.txt 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:topk_tc -s 2 -c 1 -o gpurun_out/tc_c2_src -f \
  python tools/prof_scan.py --variant tc --reps 2 --config c2 > gpurun_out/ncu_tc.log 2>&1
