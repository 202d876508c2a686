#!/bin/bash
# encoder: column-part stages for J = 512 (c3) -- parity + direct vs expanded times
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 60 python tools/prof_scan.py --what encode --reps 2 --config c3 --expanded > gpurun_out/enc_smoke.txt 2>&1 || { echo "encode hung or failed" >> gpurun_out/enc_smoke.txt; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "encode or c1 or host or code_buffer or c3" > gpurun_out/enc_tests.log 2>&1
for i in 1 2; do for c in c2 c3 c4; do
  echo "$c direct $(timeout 60 python tools/prof_scan.py --what encode --reps 10 --config $c --direct | tail -1)"
  echo "$c rows $(timeout 60 python tools/prof_scan.py --what encode --reps 10 --config $c --expanded | tail -1)"
done; done > gpurun_out/enc_times.txt 2>&1
