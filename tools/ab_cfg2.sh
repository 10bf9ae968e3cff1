#!/bin/bash
# A/B of library builds in build_ab/*.so on config 2, engine 0 (development): ab_cfg2.sh v1 v2 ...
for rep in 1 2; do for v in "$@"; do
  PFG_LIB=build_ab/$v.so timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e $BENCH_ARGS 2>&1 | tail -n 1 | python -c "
import json,sys
l=json.loads(sys.stdin.read()); r=l['roofline_query_phase']; c=l['counters']
print('$v: value %.0f ms_step %.3f kernel_ms %.3f prep_ms %.3f recall %.4f evaluated %.1f frac %.3f step %.3f' % (l['value'], l['ms_per_step'], r['kernel_ms'], r['prep_ms'], l['recall'], c['evaluated_per_q'], l['roofline']['frac'], l['roofline_step']['frac'])); print(r['phases_ms_untimed'])"
done; done
