#!/bin/bash
# A/B of library builds in build_ab/*.so on one config: CONFIG=3 bash tools/ab_cfg.sh a b ...
CONFIG=${CONFIG:-2}
STEPS=${STEPS:-5}
for v in "$@"; do
  PFG_LIB=build_ab/$v.so timeout 900 python bench.py --config $CONFIG --steps $STEPS --warmup ${WARM:-3} --no-cpu-baseline --no-e2e --storage ${STORAGE:-f32} 2>&1 | tail -n 1 | python -c "
import json,sys
l=json.loads(sys.stdin.read()); r=l['roofline_query_phase']
print('cfg $CONFIG $v: value %.0f ms_step %.3f kernel_ms %.3f recall %.4f' % (l['value'], l['ms_per_step'], r['kernel_ms'], l['recall']))"
done
