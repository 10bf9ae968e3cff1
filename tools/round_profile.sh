#!/bin/bash
# the round's measurement set (GPU box): tests, bench line, launch list of the bench command,
# ncu --set full of the dominant kernels, query-phase traffic
mkdir -p gpurun_out
[ -z "$SKIP_TESTS" ] && python -m pytest tests -m gpu -q 2>&1 | tail -2 > gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none --csv --log-file gpurun_out/traffic.csv python tools/prof_search.py --config 2 > /dev/null 2>&1
python tools/ncu_traffic.py gpurun_out/traffic.csv 2 > /dev/null
ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none --kernel-name regex:k_sims --csv --log-file gpurun_out/ksims_c2.csv \
    python tools/prof_search.py --config 2 > /dev/null 2>&1
python tools/ksims_traffic.py gpurun_out/ksims_c2.csv gpurun_out/ksims_traffic_config2.json > /dev/null
for k in k_sims k_dedupe k_scan k_merge; do
  ncu --profile-from-start off --set full --import-source on --clock-control none --kernel-name $k --launch-skip 1 \
      --launch-count 1 -o gpurun_out/full_$k -f python tools/prof_search.py > /dev/null 2>&1
  python tools/ncu_summary.py gpurun_out/full_$k.ncu-rep gpurun_out/full_$k.json > /dev/null 2>&1
done
# hashing kernels (FMA pipe): the query sketch GEMM and the eager FHT-CP codes of config 2, and
# the exact-CP argmax kernel of config 7
for k in k_hp_bits2 k_fht_qcodes_g; do
  ncu --profile-from-start off --set full --clock-control none --kernel-name regex:$k --launch-count 1 \
      -o gpurun_out/full_$k -f python tools/prof_search.py > /dev/null 2>&1
  python tools/ncu_summary.py gpurun_out/full_$k.ncu-rep gpurun_out/full_$k.json > /dev/null 2>&1
done
ncu --profile-from-start off --set full --clock-control none --kernel-name regex:k_cp_funcs --launch-count 1 \
    -o gpurun_out/full_k_cp_funcs -f python tools/prof_search.py --config 7 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/full_k_cp_funcs.ncu-rep gpurun_out/full_k_cp_funcs.json > /dev/null 2>&1
cp profiles/query_phase_traffic_config2.json gpurun_out/ 2>/dev/null
rm -f gpurun_out/*.ncu-rep   # summaries kept; the reports exceed what gpurun copies back
cat gpurun_out/pytest_gpu.log; tail -c 600 gpurun_out/bench.jsonl
