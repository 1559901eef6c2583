#!/bin/bash
# One GPU visit: smoke, full GPU test-suite, quick timings.  Everything under `timeout`.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
echo "== smoke" ; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
echo "== pytest gpu"; timeout 1500 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -15
echo "== timing d=25"; timeout 300 python tools/quick_time.py 25 25 2 2>&1 | tail -3
echo "== timing d=71"; timeout 600 python tools/quick_time.py 71 71 2 2>&1 | tail -3
