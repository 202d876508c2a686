for x in 68 64; do echo "== xmode=$x"; BOLT_LIB=libbolt_x.so BOLT_TC_XMODE=$x TRACE_OUT=gpurun_out/trace_$x.npy timeout 120 python tools/trace_scan.py --variant tc --config c2; done
BOLT_LIB=libbolt_prof.so BOLT_COUNTERS=1 timeout 120 python tools/prof_scan.py --variant tc --reps 3 --config c2
