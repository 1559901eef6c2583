#!/bin/bash
# Per-panel timeline of panel mode (debug build: -DSK_PANEL_TRACE costs the production kernel registers, so it is off by default).
# Prints, for the last cooperative launch of a d=71 run with one round + final data measurement (one block of 10 081 measurements =
# 158 panels): duration of phase 1 (F + V + D1, to the last CTA's arrival), barrier 1, phase 2 (D2 + A + next gather), barrier 2,
# and the number of active pairs; then rebuilds the production library.
mkdir -p gpurun_out
SK_BUILD_PANEL_TRACE=1 python -c "from paper_2507_03092_b200 import _build; _build.build(force=True)"
SK_DEBUG_PANELS=1 SK_DEBUG_PROF=1 python tools/quick_time_nofinal.py 71 1 1 > gpurun_out/panel_trace.txt 2>&1
grep "last panel-mode\|longest pair" gpurun_out/panel_trace.txt | tail -2
grep "  panel" gpurun_out/panel_trace.txt | tail -158 | awk 'NR%10==1'
python -c "from paper_2507_03092_b200 import _build; _build.build(force=True)"
