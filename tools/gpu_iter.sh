# development round trip on the GPU box: parity suite, bench lines and timelines
# BENCHES="--engine 0;--engine 0 --tau-rule 1" (semicolon-separated bench argument sets); TESTS=pytest target
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
if [ "${TESTS:-tests}" != "none" ]; then
timeout 1500 python -m pytest ${TESTS:-tests} -m gpu -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
tail -6 gpurun_out/pytest_gpu.log
fi
IFS=';' read -ra SETS <<< "${BENCHES:---engine 0}"
for cfg in "${SETS[@]}"; do
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e $cfg > gpurun_out/bench.log 2>&1
tail -n 1 gpurun_out/bench.log | python -c "
import json,sys
l=json.loads(sys.stdin.read()); r=l['roofline_query_phase']
print('$cfg: value %.0f ms_step %.3f kernel_ms %.3f prep_ms %.3f recall %.4f launches %d' % (l['value'], l['ms_per_step'], r['kernel_ms'], r['prep_ms'], l['recall'], l['gpu_launches'])); print(r['phases_ms_untimed']); print(l['round_stats'], l['roofline']['frac'], l['roofline_step']['frac'])" || tail -n 20 gpurun_out/bench.log
done
timeout 300 python tools/timeline.py --engine 0 2>&1 | grep "timeline\|==" > gpurun_out/timeline_e0.txt
cat gpurun_out/timeline_e0.txt
