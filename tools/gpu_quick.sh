# quick GPU round trip: smoke, selected parity tests (PYTEST_K), bench lines (BENCHES, ';'-separated), timeline
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
if [ -n "$PYTEST_K" ]; then
timeout 1500 python -m pytest ${PYTEST_FILES:-tests/test_gpu_parity.py} -m gpu -q -x -k "$PYTEST_K" 2>&1 | tail -15 > gpurun_out/pytest_quick.log
tail -4 gpurun_out/pytest_quick.log
fi
IFS=';' read -ra SETS <<< "${BENCHES:---engine 0}"
for cfg in "${SETS[@]}"; do
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e $cfg > gpurun_out/bench.log 2>&1
tail -n 1 gpurun_out/bench.log | python -c "
import json,sys
l=json.loads(sys.stdin.read()); r=l['roofline_query_phase']
print('$cfg: value %.0f ms_step %.3f kernel_ms %.3f prep_ms %.3f recall %.4f build_s %.3f launches %d ksims_frac %.3f step_frac %.3f' % (l['value'], l['ms_per_step'], r['kernel_ms'], r['prep_ms'], l['recall'], l['build_s'], l['gpu_launches'], l['roofline']['frac'], l['roofline_step']['frac']))" || tail -n 20 gpurun_out/bench.log
done
if [ -n "$TIMELINE" ]; then
timeout 300 python tools/timeline.py $TIMELINE 2>&1 | grep "timeline\|==" > gpurun_out/timeline.txt
cat gpurun_out/timeline.txt
fi
