#!/bin/bash
# Round-2 evidence for profiles/: bench lines (both arms, c3/c4/c5), ncu launch list of the bench command, full captures of the top kernels.
mkdir -p gpurun_out
R=r02
timeout 900 python bench.py > gpurun_out/bench_${R}.json 2> gpurun_out/bench_${R}.err
tail -c 300 gpurun_out/bench_${R}.json
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_${R}.json 2> gpurun_out/bench_ref_${R}.err
timeout 900 python bench.py --config c4 > gpurun_out/bench_c4_gc_${R}.json 2> gpurun_out/bench_c4_${R}.err
timeout 900 python bench.py --config c4 --c4-mode qwc --no-cpu-baseline > gpurun_out/bench_c4_qwc_${R}.json 2>> gpurun_out/bench_c4_${R}.err
timeout 900 python bench.py --config c5 > gpurun_out/bench_c5_${R}.json 2> gpurun_out/bench_c5_${R}.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_bench_${R}.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_bench_${R}.log 2>&1
python - <<PY
import csv, collections
lines = [l for l in open('gpurun_out/launches_bench_${R}.csv') if l.startswith('"')]
agg = collections.OrderedDict()
for row in csv.DictReader(lines):
    k = row['Kernel Name'].split('(')[0]; v = float(row['Metric Value'].replace(',', '')); u = row['Metric Unit']
    v = v / 1e3 if u == 'ns' else v * 1e3 if u == 'ms' else v * 1e6 if u == 's' else v
    agg.setdefault(k, []).append(v)
tot = sum(sum(v) for v in agg.values())
with open('gpurun_out/launches_bench_${R}_summary.txt', 'w') as f:
    f.write("ncu --metrics gpu__time_duration.sum --clock-control none : python bench.py --steps 1 --warmup 1 (cold-cache, serialised; compare SHARES)\n")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        f.write(f"{k:40s} launches={len(v):5d} total_us={sum(v):12.1f} share={100*sum(v)/tot:6.2f}% mean_us={sum(v)/len(v):10.1f} max_us={max(v):10.1f}\n")
print(open('gpurun_out/launches_bench_${R}_summary.txt').read())
PY
bash tools/gpu_ncu_warm.sh > gpurun_out/launches_warm_${R}_summary.txt 2>&1
# full captures: k_layer (XCX/CX layer), the fused transposition + k_wave_cols, measurement block #0 (round 1: panel mode), k_wave_rows of round 2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_layer -s 10 -c 1 -f -o gpurun_out/k_layer_${R} python tools/quick_time.py 71 3 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_transpose -s 0 -c 1 -f -o gpurun_out/k_transpose_${R} python tools/quick_time.py 71 3 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_measure_block -s 0 -c 1 -f -o gpurun_out/k_measure_panel_${R} python tools/quick_time.py 71 3 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_wave_rows -s 1 -c 1 -f -o gpurun_out/k_wave_${R} python tools/quick_time.py 71 3 1 > /dev/null 2>&1
for k in k_layer k_transpose k_measure_panel k_wave; do
  ncu -i gpurun_out/${k}_${R}.ncu-rep --page raw --csv > gpurun_out/${k}_${R}_raw.csv 2>/dev/null
done
python tools/make_traffic_json.py ${R} gpurun_out > /dev/null
SK_DEBUG_PROF=1 timeout 300 python tools/quick_time.py 71 71 2 > gpurun_out/phases_${R}.log 2>&1
bash tools/panel_trace.sh > gpurun_out/panel_trace_${R}.txt 2>&1
ls -la gpurun_out/ | tail -30
