#!/bin/bash
# ncu --set full (with source) of one kernel instance in a config-2 search: ncu_kernel.sh REGEX SKIP ENGINE
mkdir -p gpurun_out
ncu --profile-from-start off --set full --import-source on --clock-control none \
  --kernel-name regex:"$1" --launch-skip "$2" --launch-count 1 \
  -o gpurun_out/kern_full -f python tools/prof_search.py --engine "${3:-0}" > gpurun_out/ncu_kernel.log 2>&1
tail -n 2 gpurun_out/ncu_kernel.log
