# round-2 measurement set (GPU box): build launch list + ncu --set full of k_fht_keys; ncu --set full
# with source of the query-phase kernels (round 1 launches) -> gpurun_out/
mkdir -p gpurun_out
python tools/prof_build.py > gpurun_out/build_time.txt 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_build.csv python tools/prof_build.py > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_build.csv > gpurun_out/launches_build.txt 2>&1
ncu --profile-from-start off --set full --import-source on --clock-control none --kernel-name regex:k_fht_keys \
    --launch-count 1 -o gpurun_out/full_k_fht_keys -f python tools/prof_build.py > gpurun_out/ncu_k_fht_keys.log 2>&1
python tools/ncu_summary.py gpurun_out/full_k_fht_keys.ncu-rep gpurun_out/full_k_fht_keys.json > /dev/null 2>&1
ncu -i gpurun_out/full_k_fht_keys.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_k_fht_keys.csv 2>/dev/null
python tools/src_hot.py gpurun_out/src_k_fht_keys.csv 20 > gpurun_out/hot_k_fht_keys.txt 2>&1
KERNELS="${KERNELS:-k_dedupe:1 k_merge:1 k_expand:1 k_scan:1 k_sims:1}" bash tools/gpu_ncu_src.sh > gpurun_out/ncu_src_summary.txt 2>&1
rm -f gpurun_out/*.ncu-rep
cat gpurun_out/build_time.txt; tail -15 gpurun_out/launches_build.txt; python -c "
import json; d=json.load(open('gpurun_out/full_k_fht_keys.json')); print({k: d[k] for k in ('duration_s','dram_gbs','warps_active_per_sm','registers_per_thread','instructions','sm_throughput_pct','fma_pipe_active_pct')}); print(d['top_stalls_share'])"
cat gpurun_out/ncu_src_summary.txt
