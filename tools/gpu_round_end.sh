# round-end measurement set (GPU box) -> gpurun_out/: the GPU suite, the default bench line, the other
# configs, the launch list of one config-2 search, ncu --set full of the main kernels
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; tail -n 1 gpurun_out/bench_default.log > gpurun_out/bench_default.jsonl
rm -f gpurun_out/bench_other_configs.jsonl
for a in "--config 2 --storage i16" "--config 2 --tau-rule 1" "--config 3 --steps 10" "--config 3 --steps 10 --tau-rule 1" "--config 4 --steps 10" "--config 4 --steps 10 --storage i16" "--config 5 --steps 10" "--config 6 --steps 5 --warmup 6 --tau-rule 1" "--config 7 --steps 10"; do
  timeout 900 python bench.py $a --no-cpu-baseline > gpurun_out/b.log 2>&1; tail -n 1 gpurun_out/b.log >> gpurun_out/bench_other_configs.jsonl
done
python - <<'PY'
import json
for l in open('gpurun_out/bench_default.jsonl').read().splitlines() + open('gpurun_out/bench_other_configs.jsonl').read().splitlines():
    try:
        d = json.loads(l)
        print(d['config']['workload'][:8], d['config'].get('storage'), d['config'].get('tau_rule', '')[:8], round(d['value']), round(d['ms_per_step'], 3), round(d['recall'], 4),
              round(d['roofline']['frac'], 3), round(d['roofline_step']['frac'], 3), round(d['e2e']['value']), d.get('build_s'))
    except Exception as e:
        print('bad line', e, l[:200])
PY
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_s.csv python tools/prof_search.py > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_s.csv > gpurun_out/launches_search_config2.txt; head -c 600 gpurun_out/launches_search_config2.txt
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_bench.csv > gpurun_out/launches_bench.txt
ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --kernel-name regex:k_sims --csv --log-file gpurun_out/ksims_c2.csv python tools/prof_search.py > /dev/null 2>&1
python tools/ksims_traffic.py gpurun_out/ksims_c2.csv gpurun_out/ksims_traffic_config2.json > /dev/null
KERNELS="k_sims:1 k_dedupe:1 k_merge:1 k_expand:1 k_scan:1 k_hp_bits_tc:0 k_fht_qcodes_g:1" bash tools/gpu_ncu_src.sh > gpurun_out/ncu_src_summary.txt 2>&1
ncu --profile-from-start off --set full --clock-control none --kernel-name regex:k_cp_tc --launch-count 1 -o gpurun_out/full_k_cp_tc -f python tools/prof_search.py --config 7 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/full_k_cp_tc.ncu-rep gpurun_out/full_k_cp_tc.json > /dev/null 2>&1
rm -f gpurun_out/*.ncu-rep
grep -A2 "^== " gpurun_out/ncu_src_summary.txt | head -40
