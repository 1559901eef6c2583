#!/bin/bash
# per-kernel device time of a GC grouping run (N=300k) -- shares of the first-fit pipeline
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 4000 --csv --log-file gpurun_out/launches_group.csv python tools/group_time.py 300000 0 1 > gpurun_out/ncu_group.log 2>&1
python - <<'PY'
import csv, collections
lines = [l for l in open('gpurun_out/launches_group.csv') if l.startswith('"')]
agg = collections.OrderedDict()
for row in csv.DictReader(lines):
    k = row['Kernel Name'].split('(')[0]; v = float(row['Metric Value'].replace(',', '')); u = row['Metric Unit']
    v = v / 1e3 if u == 'ns' else v * 1e3 if u == 'ms' else v * 1e6 if u == 's' else v
    agg.setdefault(k, []).append(v)
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:40s} launches={len(v):5d} total_us={sum(v):12.1f} share={100*sum(v)/tot:6.2f}% mean_us={sum(v)/len(v):10.1f} max_us={max(v):10.1f}")
PY
