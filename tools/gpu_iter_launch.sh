#!/bin/bash
# development round trip: a parity subset (PYTEST_K), median search times (SWEEP option sets), and
# the ncu launch list of one config-2 search summarised into gpurun_out/launches_now.txt
mkdir -p gpurun_out
if [ -n "$PYTEST_K" ]; then
  timeout 1500 python -m pytest ${PYTEST_FILES:-tests/test_gpu_parity.py} -m gpu -q -x -k "$PYTEST_K" 2>&1 | tail -4
fi
eval timeout 600 python tools/opt_sweep.py ${SWEEP:-"'{}'"} 2>&1 | tail -12
if [ -z "$NO_NCU" ]; then
  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_now.csv python tools/prof_search.py --engine 0 > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/launches_now.csv | tee gpurun_out/launches_now.txt
fi
