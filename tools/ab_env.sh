#!/bin/bash
# A/B of environment switches on the default build (development): ab_env.sh "VAR=1" "VAR2=1" ...
for rep in 1 2; do for e in "none=1" "$@"; do
  env $e python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -n 1 | python -c "
import json,sys
l=json.loads(sys.stdin.read()); r=l['roofline']
print('$e: value %.0f ms_step %.3f kernel_ms %.3f prep_ms %.3f' % (l['value'], l['ms_per_step'], r['kernel_ms'], r['prep_ms']))"
done; done
