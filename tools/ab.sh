#!/bin/bash
# Same-box A/B of the scan: tools/ab.sh <lib1> <lib2> ... [-- prof_scan args]
# (libs are names under paper_1706_10283_b200/, e.g. libbolt_base.so libbolt.so)
libs=(); while [ $# -gt 0 ] && [ "$1" != "--" ]; do libs+=("$1"); shift; done; shift
for round in 1 2; do for l in "${libs[@]}"; do
  echo -n "$l: "; BOLT_LIB=$l timeout 120 python tools/prof_scan.py --variant tc --reps 5 --config c2 "$@" | tail -1
done; done
