#!/bin/bash
# per-kernel launch times of one config-2 search for library builds build_ab/*.so (development)
for v in "$@"; do
  PFG_LIB=build_ab/$v.so ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab_$v.csv python tools/prof_search.py > /dev/null 2>&1
  echo "== $v"; python tools/launch_summary.py gpurun_out/ab_$v.csv | head -1
done
