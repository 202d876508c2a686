# diagnostic stage switches of the tcgen05 scan (libbolt_x.so, BOLT_TC_XMODE bits:
# 1 = no epilogue processing, 2 = no one-hot expansion, 4 = filter only, 8 = no TMEM loads)
for x in 0 1 2 3 4 8 9 10 11 12; do echo "xmode=$x"; BOLT_LIB=libbolt_x.so BOLT_TC_XMODE=$x timeout 60 python tools/prof_scan.py --variant tc --reps 5 "$@"; done
