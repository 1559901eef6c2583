echo "== parity"; timeout 1200 python -m pytest tests/test_gpu_tableau_parity.py -m gpu -q -x --timeout 600 2>&1 | tail -3
echo "== d=71"; timeout 300 python tools/quick_time.py 71 71 4 2>&1 | grep -v phases | tail -3
echo "== d=25"; timeout 300 python tools/quick_time.py 25 25 3 2>&1 | grep -v phases | tail -2
