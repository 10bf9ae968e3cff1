timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "search_parity and not tensor or fuzz or degenerate or repeat or k_values" 2>&1 | grep -E "FAILED|passed|failed|Error|assert" | head -20
bash tools/ab_cfg2.sh hall loc2
BENCH_ARGS="--storage i16" bash tools/ab_cfg2.sh loc2
