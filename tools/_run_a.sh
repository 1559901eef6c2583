echo "== parity"; timeout 1200 python -m pytest tests/test_gpu_tableau_parity.py -m gpu -q -x --timeout 600 2>&1 | tail -3
echo "== d=71 cond"; timeout 300 python tools/quick_time.py 71 71 4 2>&1 | grep -v phases | tail -3
echo "== d=71 no cond"; SK_GRAPH_COND=0 timeout 300 python tools/quick_time.py 71 71 4 2>&1 | grep -v phases | tail -3
echo "== e2e"; timeout 300 python tools/e2e_time.py 2>&1 | tail -4
