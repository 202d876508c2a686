#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:encode -s 1 -c 1 -o gpurun_out/enc_fast -f python tools/prof_scan.py --what encode --reps 1 --config c2 > gpurun_out/ncu_enc_fast.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:encode -s 1 -c 1 -o gpurun_out/enc_direct -f python tools/prof_scan.py --what encode --reps 1 --config c2 --direct > gpurun_out/ncu_enc_direct.log 2>&1
