#!/bin/bash
# per-launch device time and DRAM traffic with the caches left as the application leaves them (no flush between launches):
# what a steady-state round really pays.  d=71, 5 rounds.
mkdir -p gpurun_out
SK_NO_GRAPH=1 SK_FUSE_COLS=${SK_FUSE_COLS:-1} timeout 900 ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct -c 60 --csv --log-file gpurun_out/launches_warm.csv python tools/quick_time.py 71 5 1 > gpurun_out/ncu_warm.log 2>&1
tail -2 gpurun_out/ncu_warm.log
python - <<'PY'
import csv
lines = [l for l in open('gpurun_out/launches_warm.csv') if l.startswith('"')]
rows = list(csv.DictReader(lines))
by = {}
for r in rows:
    by.setdefault(r['ID'], {'k': r['Kernel Name'][:28]})[r['Metric Name']] = (r['Metric Value'], r['Metric Unit'])
for i, d in by.items():
    print(i, d['k'], ' '.join(f"{m.split('__')[1][:22]}={v[0]}{v[1]}" for m, v in d.items() if m != 'k'))
PY
