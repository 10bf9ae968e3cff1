#!/bin/bash
# one GPU round trip used during development: parity tests, both engines' bench lines, launch list
# usage (on the box): bash tools/gpu_check.sh [pytest-args]
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q "$@" 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
tail -n 3 gpurun_out/pytest_gpu.log
for e in 0 1; do
  python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --engine $e > gpurun_out/bench_e$e.log 2>&1
  tail -n 1 gpurun_out/bench_e$e.log | python -c "
import json,sys
l=json.loads(sys.stdin.read()); r=l['roofline']
print('engine $e: value %.0f ms_step %.3f kernel_ms %.3f prep_ms %.3f frac %.3f recall %.4f launches %d' % (l['value'], l['ms_per_step'], r['kernel_ms'], r['prep_ms'], r['frac'], l['recall'], l['gpu_launches'])); print(l['counters'])" || tail -n 20 gpurun_out/bench_e$e.log
done
PFG_PHASE_PROF=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof_e0.csv python tools/prof_search.py --engine 0 > gpurun_out/prof_e0.log 2>&1
python tools/launch_summary.py gpurun_out/prof_e0.csv
