cd $GRAFT_REPO_ROOT
BOLT_LIB=libbolt_prof.so BOLT_COUNTERS=1 timeout 300 python tools/prof_scan.py --variant tc --reps 1 --config c2 > gpurun_out/counters_c2.txt 2>&1
BOLT_LIB=libbolt_prof.so BOLT_COUNTERS=1 BOLT_TC_XMODE=16 timeout 300 python tools/prof_scan.py --variant tc --reps 1 --config c2 --prefill > gpurun_out/counters_c2_prefill.txt 2>&1
for i in 1 2; do timeout 300 python tools/prof_scan.py --variant tc --reps 10 --config c2; done > gpurun_out/c2_times.txt 2>&1
