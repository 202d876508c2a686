for x in 0 16; do echo "xmode=$x"; BOLT_LIB=libbolt_x.so BOLT_TC_XMODE=$x timeout 120 python tools/prof_scan.py --variant tc --reps 5 --config c2 $([ $x = 16 ] && echo --prefill); done
for x in 0 16; do echo "xmode=$x c3"; BOLT_LIB=libbolt_x.so BOLT_TC_XMODE=$x timeout 120 python tools/prof_scan.py --variant tc --reps 5 --config c3 --nq 1000 $([ $x = 16 ] && echo --prefill); done
