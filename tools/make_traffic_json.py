"""profiles/traffic_rNN.json from the `ncu --set full` raw pages (gpurun_out/<kernel>_rNN_raw.csv): per-launch DRAM traffic and the
few ncu figures DESIGN.md / bench.py quote.  Usage: python tools/make_traffic_json.py r02 [dir]"""
import csv, json, os, sys

R = sys.argv[1] if len(sys.argv) > 1 else "r02"
D = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out"
WHAT = {
    "k_layer": ("k_layer", "one XCX/CX sub-layer of a round (about 5 000 gates)"),
    "k_transpose": ("k_transpose_wave", "C->R transposition of the stabilizer half (register-block tiles) fused with k_wave_cols of a 5 040-measurement block"),
    "k_measure_panel": ("k_measure_block", "round 1 of d=71 (5 040 measurements, 2 520 random: 79 panels, replicated level-form path) incl. the in-kernel destabilizer C->R and final R->C"),
    "k_wave": ("k_wave_rows", "partner products of the 5 040 deterministic measurements of a round (one warp each)"),
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9, "second": 1.0}
out = {}
for stem, (name, what) in WHAT.items():
    path = os.path.join(D, f"{stem}_{R}_raw.csv")
    if not os.path.exists(path):
        continue
    rows = list(csv.reader(open(path)))
    if len(rows) < 3:
        continue
    hdr, units, vals = rows[0], rows[1], rows[2]
    m = {h: (u, v) for h, u, v in zip(hdr, units, vals)}
    def num(key, scale=True):
        u, v = m[key]
        x = float(v.replace(",", ""))
        return x * UNIT.get(u, 1) if scale else x
    rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
    out[name] = {"what": what, "duration_s_under_ncu": num("gpu__time_duration.sum"), "bytes": int(rd + wr), "dram_read": int(rd), "dram_write": int(wr),
                 "registers": int(num("launch__registers_per_thread", False)), "grid": int(num("launch__grid_size", False)), "block": int(num("launch__block_size", False)),
                 "sm_throughput_pct": num("sm__throughput.avg.pct_of_peak_sustained_elapsed", False), "warps_active_pct": num("sm__warps_active.avg.pct_of_peak_sustained_active", False),
                 "issue_active_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active", False), "inst_executed": int(num("smsp__inst_executed.sum", False))}
json.dump(out, open(os.path.join(D, f"traffic_{R}.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
