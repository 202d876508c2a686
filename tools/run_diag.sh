for x in 0 64; do echo "== xmode=$x"; BOLT_LIB=libbolt_x.so BOLT_TC_XMODE=$x TRACE_OUT=gpurun_out/trace_c4_$x.npy timeout 120 python tools/trace_scan.py --variant tc --config c4 --nq 1024 --what dequant; done
echo "== xmode=1 (no epilogue processing)"; BOLT_LIB=libbolt_x.so BOLT_TC_XMODE=1 timeout 120 python tools/prof_scan.py --variant tc --config c4 --nq 1024 --what dequant
echo "== u16"; BOLT_LIB=libbolt_x.so timeout 120 python tools/prof_scan.py --variant tc --config c4 --nq 1024 --what full
