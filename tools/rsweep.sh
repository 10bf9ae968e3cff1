#!/bin/bash
# bench sweep over engines and chunk sizes (development)
for R in "$@"; do for e in 0 1; do
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --engine $e --rep-chunk $R 2>&1 | tail -n 1 | python -c "
import json,sys
l=json.loads(sys.stdin.read()); r=l['roofline']; c=l['counters']
print('R $R engine $e: value %.0f ms_step %.3f kernel_ms %.3f prep_ms %.3f frac %.3f recall %.4f evaluated %.1f emitted %.1f' % (l['value'], l['ms_per_step'], r['kernel_ms'], r['prep_ms'], r['frac'], l['recall'], c['evaluated_per_q'], c['emitted_per_q']))"
done; done
