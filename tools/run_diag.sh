bash tools/ab.sh libbolt_base.so libbolt.so
for x in 64 65; do echo "== xmode=$x"; BOLT_LIB=libbolt_x.so BOLT_TC_XMODE=$x TRACE_OUT=gpurun_out/trace_$x.npy timeout 120 python tools/trace_scan.py --variant tc --config c2; done
