for l in libbolt_base.so libbolt.so libbolt_base.so libbolt.so; do echo -n "$l "; BOLT_LIB=$l timeout 120 python tools/prof_scan.py --what encode --reps 10; done
