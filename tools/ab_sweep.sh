#!/bin/bash
# A/B of library builds build_ab/<v>.so on one box: median search times (tools/opt_sweep.py), two
# alternating passes:  bash tools/ab_sweep.sh base new ...
for pass in 1 2; do for v in "$@"; do
  echo -n "$v: "; PFG_LIB=build_ab/$v.so timeout 300 python tools/opt_sweep.py ${SWEEP:-'{}'} 2>&1 | tail -1
done; done
