# the whole GPU suite + smoke + the default bench line (GPU box) -> gpurun_out/
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; tail -n 1 gpurun_out/bench_default.log > gpurun_out/bench_default.jsonl
python -c "
import json; l=json.loads(open('gpurun_out/bench_default.jsonl').read()); print({k: l[k] for k in ('value','ms_per_step','recall','build_s')}, l['roofline']['frac'], l['roofline_step']['frac'], l['e2e'], l['cpu_baseline']['value'])"
