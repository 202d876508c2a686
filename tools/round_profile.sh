#!/bin/bash
# One pass of the round's measurements (run under gpurun): GPU tests, benches of
# every workload, the ncu launch list of the default bench and full captures of
# the dominant kernels.  Outputs in gpurun_out/ (summaries copied to profiles/rN/).
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python bench.py --config c3 --steps 10 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python bench.py --config c4 --steps 10 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python bench.py --config c1 --steps 10 --warmup 3 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
python bench.py --config sweep --steps 10 --warmup 3 > gpurun_out/bench_sweep.json 2> gpurun_out/bench_sweep.err
python bench.py --config c2nq --steps 3 --warmup 3 > gpurun_out/bench_c2nq.json 2> gpurun_out/bench_c2nq.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_c2.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_launch.log 2>&1
python tools/prof_scan.py --variant tc --reps 2 --config c2 > gpurun_out/p1.txt 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:topk_tc -s 2 -c 1 -o gpurun_out/tc_c2 -f \
  python tools/prof_scan.py --variant tc --reps 2 --config c2 > gpurun_out/ncu_tc.log 2>&1
python tools/prof_scan.py --variant tc --reps 2 --config c4 --nq 1024 --what dequant > gpurun_out/p2.txt 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:topk_tc -s 2 -c 1 -o gpurun_out/tc_c4 -f \
  python tools/prof_scan.py --variant tc --reps 2 --config c4 --nq 1024 --what dequant > gpurun_out/ncu_c4.log 2>&1
python tools/prof_scan.py --variant prmt --reps 2 --n 20000000 --nq 1 > gpurun_out/p3.txt 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:topk_small -s 2 -c 1 -o gpurun_out/small_q1 -f \
  python tools/prof_scan.py --variant prmt --reps 2 --n 20000000 --nq 1 > gpurun_out/ncu_small.log 2>&1
python tools/prof_scan.py --variant sp --reps 2 --config c2 > gpurun_out/p5.txt 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:topk_sp -s 2 -c 1 -o gpurun_out/sp_c2 -f \
  python tools/prof_scan.py --variant sp --reps 2 --config c2 > gpurun_out/ncu_sp.log 2>&1
python bench.py --config c5 --steps 3 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
python tools/prof_scan.py --what encode --reps 2 --config c2 > gpurun_out/p6.txt 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:encode -s 1 -c 1 -o gpurun_out/enc_c2 -f \
  python tools/prof_scan.py --what encode --reps 1 --config c2 > gpurun_out/ncu_enc.log 2>&1
# summaries on the box (the .ncu-rep files would exceed gpurun's 64 MiB copy-back)
for r in gpurun_out/*.ncu-rep; do
  b=${r%.ncu-rep}
  python tools/ncu_summary.py $r > $b.summary.txt 2>&1
  python tools/ncu_regions.py $r 0.005 > $b.regions.txt 2>&1
  rm -f $r
done
