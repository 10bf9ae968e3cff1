# A/B of library builds on config 2: value, step time and k_sims rows/s per build (LIBS="a.so b.so")
for L in ${LIBS:-paper_1906_12211_b200/libpfg.so}; do
  PFG_LIB=$L timeout 120 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e ${BARGS} | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline_query_phase']['phases_ms_untimed']; rs=d['round_stats']
print('%-34s %.0f q/s %.4f ms rec %.4f rows %d sims %.3f ms -> %.2f Grows/s | ksims frac %.3f' % ('$L', d['value'], d['ms_per_step'], d['recall'], rs['sims_rows'], r['sims'], rs['sims_rows']/r['sims']/1e6, d['roofline']['frac']))"
done
