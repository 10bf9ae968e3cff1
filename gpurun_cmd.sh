python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "search_parity and not tensor or fuzz or wide" 2>&1 | tail -2
bash tools/ab_cfg2.sh nopdl pdl
python tools/timeline.py 2>&1 | grep "timeline" | grep -v "qbounds"
