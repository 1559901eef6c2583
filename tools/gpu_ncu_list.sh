#!/bin/bash
# per-launch device times (cold cache, serialised) for a short d=71 run
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_d71_r3.csv python tools/quick_time.py 71 3 1 > gpurun_out/ncu_list.log 2>&1
tail -3 gpurun_out/ncu_list.log
python - <<'PY'
import csv, collections
rows = []
with open('gpurun_out/launches_d71_r3.csv') as f:
    lines = [l for l in f if l.startswith('"')]
r = csv.DictReader(lines)
agg = collections.OrderedDict()
for row in r:
    k = row['Kernel Name'][:40]; v = float(row['Metric Value'].replace(',', ''))
    unit = row['Metric Unit']
    if unit == 'ns': v /= 1e3
    elif unit == 'ms': v *= 1e3
    elif unit == 's': v *= 1e6
    agg.setdefault(k, []).append(v)
for k, v in agg.items():
    print(f"{k:42s} n={len(v):4d} total={sum(v):10.1f} us  mean={sum(v)/len(v):9.1f}  max={max(v):9.1f}  first={v[0]:9.1f} last={v[-1]:9.1f}")
PY
