# A/B of library builds on config 2 (bench value lines), alternating: LIBS="a.so b.so" bash tools/ab_quick.sh
for rep in 1 2; do
for L in ${LIBS}; do
  PFG_LIB=$L timeout 120 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e ${BARGS} | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline_query_phase']['phases_ms_untimed']
print('%-40s %.0f q/s %.4f ms recall %.4f | ' % ('$L', d['value'], d['ms_per_step'], d['recall']) + ' '.join('%s %.3f' % (k, v) for k, v in r.items()))"
done; done
