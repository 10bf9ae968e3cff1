#!/bin/bash
# ncu --set full (with source) of the fused k_query in one config-2 search
mkdir -p gpurun_out
ncu --profile-from-start off --set full --import-source on --clock-control none \
  --kernel-name regex:'k_query' --launch-count 1 \
  -o gpurun_out/fused_full -f python tools/prof_search.py --engine 1 > gpurun_out/ncu_fused.log 2>&1
tail -n 3 gpurun_out/ncu_fused.log
