#!/bin/bash
# one `ncu --set full` capture of the launch number $SKIP+1 of kernel $K (regex) in a d=71, 5-round run with the caches left warm
mkdir -p gpurun_out
SK_NO_GRAPH=1 timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:${K} -s ${SKIP:-3} -c 1 -f -o gpurun_out/${OUT:-kernel} python tools/quick_time.py 71 5 1 > gpurun_out/ncu_kernel.log 2>&1
tail -2 gpurun_out/ncu_kernel.log
ncu -i gpurun_out/${OUT:-kernel}.ncu-rep --page raw --csv > gpurun_out/${OUT:-kernel}_raw.csv 2>/dev/null
