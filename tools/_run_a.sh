echo "== parity"; timeout 1200 python -m pytest tests/test_gpu_tableau_parity.py -m gpu -q -x --timeout 600 2>&1 | tail -3
echo "== e2e"; SK_DEBUG_E2E=1 timeout 300 python tools/e2e_time.py 2>&1 | tail -4
