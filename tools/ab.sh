#!/bin/bash
# A/B of library builds in build_ab/*.so on the fused engine (development)
ENGINE=${ENGINE:-1}
for rep in 1 2; do for v in "$@"; do
  PFG_LIB=build_ab/$v.so python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --engine $ENGINE 2>&1 | tail -n 1 | python -c "
import json,sys
l=json.loads(sys.stdin.read()); r=l['roofline_query_phase']; c=l['counters']
print('$v: value %.0f ms_step %.3f kernel_ms %.3f prep_ms %.3f recall %.4f evaluated %.1f' % (l['value'], l['ms_per_step'], r['kernel_ms'], r['prep_ms'], l['recall'], c['evaluated_per_q']))"
done; done
