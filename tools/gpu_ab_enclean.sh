#!/bin/bash
# Encoder A/B on one box (BOLT_ENC_LEAN = 2 in all but the base):
#   libbolt_encbase.so  round-2 epilogue (tags, global-memory fallback, E = 4 g A)
#   libbolt_encfbg.so   bit-group minima, global-memory fallback, E = 4 g A
#   libbolt_ence4.so    + shared-memory fallback
#   libbolt.so          + E = 2 g A
#   libbolt_x.so with BOLT_ENC_XMODE=2: no fallback at all (wrong codes; the floor)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for l in libbolt.so; do
  BOLT_LIB=$l timeout 60 python tools/prof_scan.py --what encode --reps 2 --config c2 --expanded > gpurun_out/encl_smoke_$l.txt 2>&1 || { echo "$l hung or failed"; exit 1; }
  BOLT_LIB=$l timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "encode or c1 or host or code_buffer" > gpurun_out/encl_tests_$l.log 2>&1
  tail -2 gpurun_out/encl_tests_$l.log
done
for i in 1 2 3; do for c in c2 c3 c4; do for l in libbolt_encbase.so libbolt_encfbg.so libbolt_ence4.so libbolt.so; do
  echo "$c $l $(BOLT_LIB=$l timeout 60 python tools/prof_scan.py --what encode --reps 10 --config $c --expanded | tail -1)"
done
echo "$c nofallback $(BOLT_LIB=libbolt_x.so BOLT_ENC_XMODE=2 timeout 60 python tools/prof_scan.py --what encode --reps 10 --config $c --expanded | tail -1)"
echo "$c x_full $(BOLT_LIB=libbolt_x.so timeout 60 python tools/prof_scan.py --what encode --reps 10 --config $c --expanded | tail -1)"
done; done > gpurun_out/encl.txt 2>&1
cat gpurun_out/encl.txt
