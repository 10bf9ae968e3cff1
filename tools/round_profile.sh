#!/bin/bash
# the round's measurement set (GPU box), into gpurun_out/: launch list of the bench command, DRAM
# traffic of one search (query phase and every k_sims launch), ncu --set full summaries of the
# dominant kernels and the hashing kernels
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_bench.csv > gpurun_out/launches_bench.txt 2>&1
ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none --csv --log-file gpurun_out/traffic.csv python tools/prof_search.py --config 2 > /dev/null 2>&1
python tools/ncu_traffic.py gpurun_out/traffic.csv 2 > /dev/null
cp profiles/query_phase_traffic_config2.json gpurun_out/ 2>/dev/null
ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none --kernel-name regex:k_sims --csv --log-file gpurun_out/ksims_c2.csv \
    python tools/prof_search.py --config 2 > /dev/null 2>&1
python tools/ksims_traffic.py gpurun_out/ksims_c2.csv gpurun_out/ksims_traffic_config2.json > /dev/null
KERNELS="k_sims:1 k_dedupe:1 k_scan:1 k_merge:1 k_expand:1 k_hp_bits2:0 k_fht_qcodes_g:1" bash tools/gpu_ncu_src.sh \
    > gpurun_out/ncu_src_summary.txt 2>&1
ncu --profile-from-start off --set full --clock-control none --kernel-name regex:k_cp_funcs --launch-count 1 \
    -o gpurun_out/full_k_cp_funcs -f python tools/prof_search.py --config 7 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/full_k_cp_funcs.ncu-rep gpurun_out/full_k_cp_funcs.json > /dev/null 2>&1
rm -f gpurun_out/*.ncu-rep
tail -c 400 gpurun_out/launches_bench.txt; cat gpurun_out/ksims_traffic_config2.json | head -c 300
