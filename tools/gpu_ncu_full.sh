#!/bin/bash
mkdir -p gpurun_out
SK_MEAS_GRID=${GRID:-1} SK_SEQ_THRESHOLD=${SEQ:-100000} timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_measure_block -c 1 -f -o gpurun_out/meas_seq python tools/quick_time.py 71 1 1 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
