#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:topk_small -s 3 -c 1 -o gpurun_out/small_sweep_q1 -f \
  python bench.py --config sweep --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_sweep.log 2>&1
python tools/ncu_summary.py gpurun_out/small_sweep_q1.ncu-rep > gpurun_out/small_sweep_q1.summary.txt 2>&1
python tools/ncu_regions.py gpurun_out/small_sweep_q1.ncu-rep 0.003 > gpurun_out/small_sweep_q1.regions.txt 2>&1
rm -f gpurun_out/small_sweep_q1.ncu-rep
