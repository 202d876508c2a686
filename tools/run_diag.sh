for q in 1 2 4 8 16 32; do timeout 120 python tools/prof_scan.py --variant prmt --n 20000000 --nq $q --k 10 --reps 5; done
for q in 1 8 32; do timeout 120 python tools/prof_scan.py --variant prmt --n 1000000 --nq $q --config c2 --reps 5; done
