for i in 1 2; do timeout 120 python tools/prof_scan.py --what encode --reps 10; done
