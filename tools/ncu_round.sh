#!/bin/bash
# ncu --set full of the round engine's kernels in one config-2 search
mkdir -p gpurun_out
ncu --profile-from-start off --set full --import-source on --clock-control none \
  --kernel-name regex:'k_qbounds|k_collect|k_sims|k_merge|k_fht_qcodes|k_hp_bits' --launch-count 9 \
  -o gpurun_out/round_full -f python tools/prof_search.py --engine 0 > gpurun_out/ncu_round.log 2>&1
ncu -i gpurun_out/round_full.ncu-rep --page raw --csv > gpurun_out/round_full_raw.csv 2>/dev/null
tail -n 3 gpurun_out/ncu_round.log
