#!/bin/bash
# quick perf probe: kernel/prep ms of the config-2 bench (used during optimisation)
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e "$@" 2>&1 | tail -1 | python -c "
import json,sys
l=json.loads(sys.stdin.read())
r=l['roofline']; print('value %.0f kernel_ms %.3f prep_ms %.3f frac %.3f recall %.4f' % (l['value'], r['kernel_ms'], r['prep_ms'], r['frac'], l['recall'])); print(l['counters'])"
