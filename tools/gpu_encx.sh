#!/bin/bash
# whole-row TMA encoder: parity tests + A/B (libbolt_x.so: BOLT_ENC_W8 = 8 warps x 4 slabs)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 60 python tools/prof_scan.py --what encode --reps 2 --config c2 --expanded > gpurun_out/enc_smoke.txt 2>&1 || { echo "encode hung or failed" >> gpurun_out/enc_smoke.txt; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "encode or c1 or host or code_buffer" > gpurun_out/enc_tests.log 2>&1
for i in 1 2; do for c in c2 c3 c4; do
  echo "$c direct $(timeout 60 python tools/prof_scan.py --what encode --reps 10 --config $c --direct | tail -1)"
  echo "$c rows16 $(timeout 60 python tools/prof_scan.py --what encode --reps 10 --config $c --expanded | tail -1)"
  echo "$c rows8 $(BOLT_LIB=libbolt_x.so BOLT_ENC_W8=1 timeout 60 python tools/prof_scan.py --what encode --reps 10 --config $c --expanded | tail -1)"
done; done > gpurun_out/encx.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:encode_rows -s 1 -c 1 -o gpurun_out/enc_rows16 -f python tools/prof_scan.py --what encode --reps 1 --config c2 --expanded > gpurun_out/ncu_enc_rows.log 2>&1
