# ncu --set full with source of selected kernels of one config-2 search (engine 0), summaries +
# hottest SASS lines into gpurun_out/:  KERNELS="k_dedupe:1 k_merge:1" bash tools/gpu_ncu_src.sh
mkdir -p gpurun_out
for ks in ${KERNELS:-k_dedupe:1 k_merge:1 k_scan:1 k_expand:1}; do
  k=${ks%%:*}; skip=${ks##*:}
  ncu --profile-from-start off --set full --import-source on --clock-control none \
    --kernel-name regex:"$k" --launch-skip $skip --launch-count 1 \
    -o gpurun_out/full_$k -f python tools/prof_search.py --engine 0 > gpurun_out/ncu_$k.log 2>&1
  python tools/ncu_summary.py gpurun_out/full_$k.ncu-rep gpurun_out/full_$k.json > /dev/null 2>&1
  ncu -i gpurun_out/full_$k.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_$k.csv 2>/dev/null
  python tools/src_hot.py gpurun_out/src_$k.csv 30 > gpurun_out/hot_$k.txt 2>&1
  echo "== $k"; python -c "
import json; d=json.load(open('gpurun_out/full_$k.json')); print({k: d[k] for k in ('duration_s','dram_gbs','warps_active_per_sm','registers_per_thread','instructions','sm_throughput_pct')}); print(d['top_stalls_share'])"
  head -25 gpurun_out/hot_$k.txt
done
rm -f gpurun_out/*.ncu-rep
