#!/usr/bin/env python
"""bench.py -- headline benchmark: surface-code memory experiment d=71, 71 rounds, Z-basis
(BASELINE.json configs[2]; fits one B200), one full CHP simulation per step.

    python bench.py --gpus N --steps K --warmup W            # our CUDA path
    python bench.py --impl reference --gpus N --steps K ...  # the reference algorithm on the host CPU

One JSON line on stdout (rank 0).  `value` = seconds per full simulation with the compiled program
and tableau already resident in HBM (CUDA events on the library's stream, max over ranks);
`e2e` = the same simulation through the C-ABI call `sk_sim` with HOST buffers (circuit in pinned
host memory -> compile -> upload -> simulate -> measurement record back to the host).
N > 1 runs BASELINE config 3 as it is stated -- ONE simulation whose tableau is row-sharded over the N ranks (
paper_2507_03092_b200/sharded.py; NCCL allreduce-min / broadcast / allgather per measurement window), strong scaling;
`--sharding replicas` instead lets every rank simulate the whole circuit (independent shots, seed ^ rank: the layout that is
fastest for a 102 MB working set, weak scaling).  `--local-shards L` puts L shards on each GPU (how the protocol is
exercised on a single B200).

`--config c4` / `--config c5` time the other two BASELINE workloads on one GPU (one line each, same keys):
    c4  first-fit commutation grouping of 10^6 random 128-qubit Pauli strings (`--c4-mode gc|qwc`)
    c5  Clifford+T transpile of a random 1000-qubit, 10^5-gate circuit with 10 % T gates
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEED = 20250703
D, ROUNDS = 71, 71
METRIC = "surface-code sim time (d=71, 71 rounds, Z-basis)"
WORKLOAD = f"rotated surface-code memory d={D}, {ROUNDS} rounds, final Z-basis data measurement (n=10081 qubits, 2132201 gates, 362881 measurements)"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons.  The sampler runs from before the warm-up (nvidia-smi needs a moment to
    start) at 20 ms; stop(t0, t1) keeps the samples whose timestamps fall inside the timed region [t0, t1] (wall clock),
    or, if the region was shorter than the sampling period, the samples closest to it."""

    def __init__(self, index: int, period_ms: int = 20):
        # (launch-heavy, second-long regions -- configs C4 / C5 -- are sampled at 250 ms: every nvidia-smi query takes the
        #  driver lock and the 20 ms cadence cost the grouping run up to 40 % of its time)
        self.index, self.rows, self.proc, self.period_ms = index, [], None, period_ms

    def start(self):
        q = "timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
            "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", str(self.period_ms)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _read(self):
        import datetime
        for line in self.proc.stdout:
            c = [x.strip() for x in line.split(",")]
            try:
                ts = datetime.datetime.strptime(c[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except Exception:
                ts = time.time()
            self.rows.append((ts, c[1:]))

    def stop(self, t0: float = 0.0, t1: float = float("inf")) -> dict:
        if self.proc:
            time.sleep(0.05)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                pass
        rows = [r for ts, r in self.rows if t0 <= ts <= t1]
        where = "inside the timed region"
        if not rows and self.rows:          # region shorter than the sampling period: nearest samples
            mid = 0.5 * (t0 + t1) if t1 != float("inf") else t0
            rows = [r for _, r in sorted(self.rows, key=lambda x: abs(x[0] - mid))[:3]]
            where = "nearest to the timed region"
        sm = sorted(int(r[0]) for r in rows if r and r[0].isdigit())
        mx = [int(r[1]) for r in rows if len(r) > 1 and r[1].isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for k, nme in enumerate(names):
                if len(r) > 2 + k and r[2 + k].lower().startswith("active"):
                    reasons.add(nme)
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm), "sampled": where}


def cpu_reference(full: bool = True, rounds_sample: int = 12):
    """The reference algorithm on the host cores: oracle port (kind 'port').  Imports nothing but oracle/ (the
    circuit comes from the oracle's own generator), so the reference arm never maps the CUDA library.

    full=True: ONE timed run of the complete workload (d=71, all 71 rounds + final data-qubit M), no warm-up --
    the number `--impl reference` reports.  full=False: a bounded sample for the cpu_baseline object of our arm
    (the circuit cut to `rounds_sample` rounds and to half of that; steady-state round cost x 71 + the rest once),
    labelled as an extrapolation.  Threads: Clifford runs are row-partitioned over all host threads;
    measure_z itself is single-threaded in the port, which is stated in `cores_note`."""
    from oracle import oracle_py as orc
    cores = os.cpu_count() or 1
    note = f"{cores} threads in Clifford runs (rows partitioned, SPEC:346); the measurement loop (pivot search + rowsums) is single-threaded"

    def run(rounds):
        n, gates, _ = orc.surface_code(D, rounds, True)
        t = orc.Tableau(n)
        t0 = time.perf_counter()
        out, det, rc = t.sim(gates, SEED, workers=cores)
        dt = time.perf_counter() - t0
        assert rc == 0
        return dt, (int(out.sum()), int(det.sum()))

    if full:
        dt, chk = run(ROUNDS)
        return {"value": dt, "unit": "s", "cores": cores, "kind": "port", "cores_note": note, "extrapolated": False,
                "sample": f"the full workload, measured once: d={D}, {ROUNDS} rounds + final data-qubit M ({dt:.2f} s wall, no warm-up)",
                "record_checksum": list(chk)}
    r_lo = max(2, rounds_sample // 2)
    t_hi, _ = run(rounds_sample)
    t_lo, _ = run(r_lo)
    per_round = max(0.0, (t_hi - t_lo) / (rounds_sample - r_lo))
    fixed = max(0.0, t_lo - r_lo * per_round)
    return {"value": fixed + ROUNDS * per_round, "unit": "s", "cores": cores, "kind": "port", "cores_note": note, "extrapolated": True,
            "measured_lower_bound_s": t_hi,
            "sample": f"EXTRAPOLATED from d={D} cut to {r_lo} and {rounds_sample} of {ROUNDS} rounds (+ final data-qubit M): {t_lo:.2f} s and {t_hi:.2f} s measured; "
                      f"{per_round:.3f} s per steady-state round x {ROUNDS} + {fixed:.2f} s once; `--impl reference` measures the full run"}


def bench_row_sharded(args, sk, skdist, torch, rank, local_rank, world, workload):
    """One d=71 simulation with the tableau row-sharded over the ranks (x local shards per GPU).  The circuit is a host
    buffer, so the timed region is end to end by construction (gates H2D per Clifford run, candidates / outcomes D2H)."""
    from paper_2507_03092_b200.sharded import ShardedTableau
    circ = sk.surface_code_circuit(D, ROUNDS, True)
    sampler = ClockSampler(local_rank); sampler.start()
    times, rec, stats, calls, xbytes, launches = [], None, None, None, 0, 0
    steps, warm = max(1, args.steps), max(args.warmup, 3)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local_rank}")     # > 126 MB L2
    t_region0 = time.time()
    for i in range(warm + steps):
        if i == warm:
            t_region0 = time.time()
        t = ShardedTableau.create_cuda(circ.n, local_shards=args.local_shards, device_index=local_rank)
        t.ctx.reset_counters()
        flush.zero_(); torch.cuda.synchronize()         # L2 flush, outside the event pair
        skdist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(t.stream)
        out, det = t.sim(circ, SEED)
        e1.record(t.stream); t.stream.synchronize()
        skdist.barrier()
        if i >= warm:
            times.append(e0.elapsed_time(e1))
            launches += t.ctx.counters()["kernel_launches"]
        rec, stats, calls, xbytes = (int(out.sum()), int(det.sum())), dict(t.stats), dict(t.ex.calls), t.ex.bytes
        t.close()
    clocks = sampler.stop(t_region0, time.time())
    ms = skdist.max_over_ranks(sum(times) / len(times))
    if rank == 0:
        G = world * args.local_shards
        line = {"metric": METRIC, "value": ms * 1e-3, "unit": "s", "n_gpus": world, "steps": steps, "warmup": warm, "ms_per_step": ms,
                "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
                "config": {"workload": workload, "seed": SEED, "parallelism": f"tableau row-sharded over {world} rank(s) x {args.local_shards} local shard(s) = {G} shards",
                           "l2": "flushed between steps (256 MiB write outside the event pair)",
                           "timing": "CUDA events on the library stream around the whole simulation, mean of steps, max over ranks"},
                "e2e": {"value": ms * 1e-3, "unit": "s", "h2d_bytes_per_step": int(len(circ.gates) * 12 * args.local_shards + 4 * 2 * circ.num_measurements),
                        "d2h_bytes_per_step": int(5 * circ.num_measurements), "call": "ShardedTableau.sim(circuit in host memory, seed)"},
                "gpu_launches": int(launches), "clocks": clocks, "record_checksum": list(rec),
                "sharding": {"global_shards": G, "n_rand": stats["n_rand"], "n_det": stats["n_det"], "pivot_search_windows": stats["searches"],
                             "collectives_per_step": calls, "exchange_bytes_per_step": xbytes}}
        print(json.dumps(line))
    skdist.finalize()
    return 0


def _load_workloads():
    """paper_2507_03092_b200/workloads.py without importing the package (the reference arm must not map the CUDA library)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("sk_workloads", os.path.join(ROOT, "paper_2507_03092_b200", "workloads.py"))
    m = importlib.util.module_from_spec(spec); spec.loader.exec_module(m)
    return m


def _golden_c4(N):
    p = os.path.join(ROOT, "tests", "golden", f"c4_groups_{N}.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return None


def _c4_cpu(mode, mname, N_full, N_sample=100_000):
    """CPU oracle on a bounded sample (N_sample terms), scaled to N_full by the predicate calls the oracle itself needed at
    N_full (tests/golden/c4_groups_*.json, measured once) or, without that file, by (N_full / N_sample)^2."""
    import numpy as np
    from oracle import oracle_py as orc
    wl = _load_workloads()
    x, z, _ = wl.c4_terms(N_sample)
    o = orc.Rows(128, x, z, np.zeros(N_sample, np.uint8))
    t0 = time.perf_counter(); g, ng, calls = o.group_first_fit(mode); dt = time.perf_counter() - t0
    gold = _golden_c4(N_full)
    if gold and mname in gold["modes"]:
        scale = gold["modes"][mname]["predicate_calls"] / max(1, calls); how = "ratio of the oracle's own predicate calls at the two sizes"
        full_s = gold["modes"][mname].get("oracle_seconds")
    else:
        scale = (N_full / N_sample) ** 2; how = "(N_full / N_sample)^2"; full_s = None
    return {"value": dt * scale, "unit": "s", "cores": 1, "kind": "port", "extrapolated": True,
            "sample": f"first-fit {mname} of the first-sorted N={N_sample} terms of the same generator: {dt:.2f} s, {calls} predicate calls, {ng} groups; scaled x{scale:.1f} ({how})"
                      + (f"; the oracle's one full N={N_full} run took {full_s} s (tools/make_c4_golden.py)" if full_s else "")}


def bench_c4(args):
    """BASELINE config 4: first-fit grouping of N random 128-qubit Pauli strings."""
    mode = 0 if args.c4_mode == "gc" else 1
    mname = "GC" if mode == 0 else "QWC"
    N = args.c4_n
    metric = f"Pauli commutation grouping time (N={N}, n=128, first fit {mname})"
    workload = f"{N} random Pauli strings on 128 qubits (SplitMix64 seed {SEED}, SURVEY 8d), sorted by |coeff| descending, first-fit {mname} grouping"
    if args.impl == "reference":
        cb = _c4_cpu(mode, mname, N)
        print(json.dumps({"impl": "reference", "metric": metric, "value": cb["value"], "unit": "s", "n_gpus": args.gpus, "steps": 1, "warmup": 0,
                          "ms_per_step": cb["value"] * 1e3, "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
                          "config": {"workload": workload, "seed": SEED, "parallelism": "one host thread"}, "cpu_baseline": cb,
                          "e2e": {"value": cb["value"], "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}, "gpu_launches": 0}))
        return 0
    import hashlib
    import numpy as np
    import torch
    import paper_2507_03092_b200 as sk
    from paper_2507_03092_b200 import workloads as wl
    sk.lib()
    ctx = sk.Context(0)
    stream = torch.cuda.ExternalStream(ctx.stream)
    x, z, _ = wl.c4_terms(N)
    xp = torch.from_numpy(x).pin_memory().numpy(); zp = torch.from_numpy(z).pin_memory().numpy(); sp = torch.zeros(N, dtype=torch.uint8).pin_memory().numpy()
    rows = sk.Rows(ctx, 128, xp, zp, sp)
    steps, warm = max(1, min(args.steps, 5)), max(3, min(args.warmup, 5))
    sampler = ClockSampler(0, 250); sampler.start()
    for _ in range(warm):
        g, ng = rows.group_first_fit(mode)
    ctx.sync(); ctx.reset_counters()
    t_region0 = time.time()
    ms = []
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream); g, ng = rows.group_first_fit(mode); e1.record(stream); ctx.sync()
        ms.append(e0.elapsed_time(e1))
    t_region1 = time.time()
    clocks = sampler.stop(t_region0, t_region1)
    cnt = ctx.counters()
    viol = rows.verify_grouping(mode, g)
    rows.close()
    # end to end: host arrays -> device rows -> groups -> group ids back on the host
    e2e = []
    for i in range(1 + max(1, min(args.e2e_steps, 3))):
        t0 = time.perf_counter()
        r2 = sk.Rows(ctx, 128, xp, zp, sp); g2, ng2 = r2.group_first_fit(mode); ctx.sync()
        dt = time.perf_counter() - t0
        r2.close()
        if i: e2e.append(dt)
    assert ng2 == ng and (g2 == g).all()
    ms_step = sum(ms) / len(ms)
    gold = _golden_c4(N)
    g32 = np.ascontiguousarray(g, np.uint32)
    parity = None
    if gold and mname in gold["modes"]:
        parity = bool(gold["modes"][mname]["groups"] == ng and hashlib.sha256(g32.tobytes()).hexdigest() == gold["modes"][mname]["sha256"])
    pred = cnt["pred_evals"] / steps
    peak = 148 * 16 * 1.965e9 / 4 / 1e9 if mode == 0 else 148 * 64 * 1.965e9 / 20 / 1e9
    line = {"metric": metric, "value": ms_step * 1e-3, "unit": "s", "n_gpus": 1, "steps": steps, "warmup": warm, "ms_per_step": ms_step, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": workload, "seed": SEED, "parallelism": "one GPU", "l2": "inputs (32 MB) + group store exceed nothing: L2 resident by design; not flushed",
                       "timing": "CUDA events on the library stream around sk_group_first_fit (rows resident, group ids copied back), mean of steps"},
            "e2e": {"value": sum(e2e) / len(e2e), "unit": "s", "h2d_bytes_per_step": int(N * 33), "d2h_bytes_per_step": int(N * 4),
                    "call": "sk_rows_create + sk_rows_upload (pinned host arrays) + sk_group_first_fit"},
            "gpu_launches": int(cnt["kernel_launches"]),
            "roofline": {"bound": "int", "kernel": "k_conflict_groups", "achieved": pred / (ms_step * 1e-3) / 1e9, "peak": peak, "unit": "Gpred/s",
                         "frac": pred / (ms_step * 1e-3) / 1e9 / peak, "traffic": None,
                         "predicates_per_step": pred, "pair_equivalents_per_step": N * (N - 1) / 2,
                         "peak_source": "nominal integer pipe: 148 SMs x 16 POPC/clk x 1.965 GHz / 4 POPC per 128-qubit predicate (GC); 148 x 64 INT32/clk / ~20 ops (QWC) -- no measured INT peak exists; "
                                        "the whole-run fraction is low because the single-CTA first-fit resolver (sequential in the term index) takes most of the time"},
            "clocks": clocks, "groups": int(ng), "verify_violations": int(viol), "bit_exact_vs_oracle_golden": parity}
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = _c4_cpu(mode, mname, N)
    print(json.dumps(line))
    ctx.close()
    return 0


def _c5_alg2_bytes(gates, n, kinds):
    """Algorithm 2 walks the circuit backwards; a Clifford gate sweeps R = 2n + |T_tab at that point| rows."""
    import numpy as np
    H, S, CX, T, TDG = kinds
    k = gates["kind"]
    is_t = (k == T) | (k == TDG)
    t_after = np.cumsum(is_t[::-1])[::-1] - is_t          # T rows already appended when gate i is reached
    cols = np.where(k == H, 4, np.where(k == S, 3, np.where(k == CX, 6, 0))).astype(np.float64)
    R = 2.0 * n + t_after
    return float((cols * R / 8.0).sum())


def bench_c5(args):
    """BASELINE config 5: Clifford+T transpile of a random 1000-qubit circuit, 10 % T gates."""
    n, G = 1000, 100_000
    metric = f"Clifford+T transpile time (n={n}, {G} gates, 10% T)"
    workload = f"random Clifford+T circuit on {n} qubits, {G} gates (SplitMix64 seed 20250704, SURVEY 8d: 5% t, 5% tdg, 30% h, 30% s, 30% cx), exact transpile to T layers + M_tab"
    wl = _load_workloads()
    import numpy as np
    dt12 = np.dtype([("kind", "u1"), ("pad", "u1", (3,)), ("q0", "<u4"), ("q1", "<u4")])
    kinds = (0, 1, 6, 10, 11)
    gates = wl.c5_gates(n, G, gate_dtype=dt12, kinds=kinds)
    if args.impl == "reference" or not args.no_cpu_baseline:
        from oracle import oracle_py as orc
        t0 = time.perf_counter(); op = orc.Pbc(n, gates, exact=True); cpu_s = time.perf_counter() - t0
        ostats = op.stats()
        cb = {"value": cpu_s, "unit": "s", "cores": 1, "kind": "port", "extrapolated": False,
              "sample": f"the full workload, measured once ({cpu_s:.2f} s): {ostats}"}
    if args.impl == "reference":
        print(json.dumps({"impl": "reference", "metric": metric, "value": cb["value"], "unit": "s", "n_gpus": args.gpus, "steps": 1, "warmup": 0,
                          "ms_per_step": cb["value"] * 1e3, "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
                          "config": {"workload": workload, "seed": 20250704, "parallelism": "one host thread"}, "cpu_baseline": cb,
                          "e2e": {"value": cb["value"], "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}, "gpu_launches": 0}))
        return 0
    import torch
    import paper_2507_03092_b200 as sk
    sk.lib()
    ctx = sk.Context(0)
    gp = torch.empty(G * 12, dtype=torch.uint8).pin_memory().numpy().view(sk.GATE_DTYPE); gp[:] = gates
    circ = sk.Circuit(n, gp)
    steps, warm = max(1, min(args.steps, 5)), max(3, min(args.warmup, 5))
    sampler = ClockSampler(0, 250); sampler.start()
    for _ in range(warm):
        sk.Pbc(ctx, circ).close()
    ctx.sync(); ctx.reset_counters()
    t_region0 = time.time()
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter(); pb = sk.Pbc(ctx, circ); ctx.sync(); ts.append(time.perf_counter() - t0)
        stats = pb.stats()
        if _ < steps - 1: pb.close()
    t_region1 = time.time()
    clocks = sampler.stop(t_region0, t_region1)
    cnt = ctx.counters()
    same = None
    if not args.no_cpu_baseline:
        same = stats == ostats
        for k in range(stats["layers"]):
            same = same and all((u == v).all() for u, v in zip(pb.layer(k), op.layer(k)))
        same = bool(same and all((u == v).all() for u, v in zip(pb.mtab(), op.mtab().get())))
    pb.close()
    sec = sum(ts) / len(ts)
    ab = _c5_alg2_bytes(gates, n, kinds)
    peak, peak_src = peaks()
    line = {"metric": metric, "value": sec, "unit": "s", "n_gpus": 1, "steps": steps, "warmup": warm, "ms_per_step": sec * 1e3, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": workload, "seed": 20250704, "parallelism": "one GPU", "l2": "working set ~3 MB: L2 resident by nature; not flushed",
                       "timing": "wall clock around sk_transpile_ex + sync (the call takes the gate list from pinned host memory: value and e2e are the same call), mean of steps"},
            "e2e": {"value": sec, "unit": "s", "h2d_bytes_per_step": int(G * 12), "d2h_bytes_per_step": 40, "call": "sk_transpile_ex(ctx, n, gates, ngates, flags=0) with a pinned host gate list"},
            "gpu_launches": int(cnt["kernel_launches"]),
            "roofline": {"bound": "hbm", "kernel": "k_layer (Algorithm 2 backward walk)", "achieved": ab / sec / 1e9, "peak": peak, "unit": "GB/s", "frac": ab / sec / 1e9 / peak,
                         "traffic": None, "peak_source": peak_src, "algorithmic_bytes": ab,
                         "note": "Algorithm 2 only (SURVEY 8d: a Clifford gate sweeps 2n + |T_tab| rows); the commutation scans and rowsum+i of Algorithms 3-4 are not counted, so this is a lower bound; "
                                 "the pass is a chain of ~10^5 small dependent launches on a 3 MB working set: launch bound, not bandwidth bound"},
            "clocks": clocks, "stats": stats, "bit_exact_vs_oracle": same}
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cb
    print(json.dumps(line))
    ctx.close()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", action="store_true", help="cpu_baseline: extrapolate from 6- and 12-round cuts instead of timing the full 71-round run (~25 s on 16 threads)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--sharding", default=None, choices=["replicas", "rows"], help="default: rows when --gpus > 1 (BASELINE config 3), replicas on one GPU")
    ap.add_argument("--config", default="c3", choices=["c3", "c4", "c5"])
    ap.add_argument("--c4-mode", default="gc", choices=["gc", "qwc"])
    ap.add_argument("--c4-n", type=int, default=1_000_000)
    ap.add_argument("--local-shards", type=int, default=1)
    args = ap.parse_args()
    if args.sharding is None:
        args.sharding = "rows" if (args.gpus > 1 or int(os.environ.get("WORLD_SIZE", "1")) > 1) else "replicas"
    if args.config != "c3":
        if int(os.environ.get("RANK", "0")) != 0:           # single-GPU configs: rank 0 alone works
            return 0
        return bench_c4(args) if args.config == "c4" else bench_c5(args)

    if args.impl == "reference":
        # Rank 0 alone works; nothing here imports the CUDA package (env_world is read from the environment directly).
        if int(os.environ.get("RANK", "0")) != 0:
            return 0
        cb = cpu_reference(full=True)                       # one measured full-length run (steps 1, warm-up 0)
        line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "s", "n_gpus": args.gpus, "steps": 1,
                "warmup": 0, "ms_per_step": cb["value"] * 1e3, "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
                "dtype": "u64", "data": "synthetic", "config": {"workload": WORKLOAD, "seed": SEED, "parallelism": "host threads"},
                "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "cores_note", "extrapolated")},
                "e2e": {"value": cb["value"], "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                "gpu_launches": 0, "record_checksum": cb["record_checksum"]}
        print(json.dumps(line))
        return 0

    from paper_2507_03092_b200 import dist as skdist
    rank, local_rank, world = skdist.env_world()
    workload = WORKLOAD

    import numpy as np
    import torch
    import paper_2507_03092_b200 as sk

    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device; the stabilizer hot path has no CPU fallback")
    torch.cuda.set_device(local_rank)
    skdist.init("nccl")
    barrier = skdist.barrier

    sk.lib()
    if args.sharding == "rows":
        return bench_row_sharded(args, sk, skdist, torch, rank, local_rank, world, workload)
    ctx = sk.Context(local_rank)
    stream = torch.cuda.ExternalStream(ctx.stream)
    circ = sk.surface_code_circuit(D, ROUNDS, True)
    seed = skdist.shot_seed(SEED, rank)
    prog = sk.Program(ctx, circ, mode=0)
    tab = sk.Tableau(ctx, circ.n)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")     # > 126 MB L2

    def one_step(timed: bool):
        with torch.cuda.stream(stream):
            flush.zero_()                                   # L2 flush, outside the event pair
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        tab.reset()                                         # identity tableau (part of the step: sim starts from |0..0>)
        prog.run(tab, seed)
        e1.record(stream)
        return e0, e1

    sampler = ClockSampler(local_rank); sampler.start()
    for _ in range(max(args.warmup, 3)):
        one_step(False)
    ctx.sync()
    ctx.reset_counters()
    barrier()
    t_region0 = time.time()
    evs = [one_step(True) for _ in range(args.steps)]
    ctx.sync()
    t_region1 = time.time()
    barrier()
    clocks = sampler.stop(t_region0, t_region1)
    step_ms = [a.elapsed_time(b) for a, b in evs]
    cnt = ctx.counters()
    out, det = prog.read_record()
    ms_per_step = skdist.max_over_ranks(sum(step_ms) / len(step_ms))

    # per-kernel-class device time (CUDA events around every launch) for the roofline lines
    tab.reset(); ctx.sync()
    cls = prog.run_profiled(tab, seed)

    # ---- end to end through the C ABI with host buffers -----------------------------------
    gates_pinned = torch.empty(len(circ.gates) * 12, dtype=torch.uint8).pin_memory()
    gates_np = gates_pinned.numpy().view(sk.GATE_DTYPE)
    gates_np[:] = circ.gates
    circ_pinned = sk.Circuit(circ.n, gates_np, circ.chunk_marks)
    e2e_times = []
    circ_pinned.num_measurements                            # counted once, outside the timed calls (binding bookkeeping, not the library)
    for i in range(3 + max(1, args.e2e_steps)):             # 3 warm-up calls: memory pool and pinned staging reach their steady state
        barrier()
        t0 = time.perf_counter()
        tt, o2, d2, _ = ctx.sim(circ_pinned, seed)          # compile + H2D + simulate + record D2H
        ctx.sync()
        dt = time.perf_counter() - t0
        tt.close()
        if i >= 3:
            e2e_times.append(dt)
    assert (o2 == out).all() and (d2 == det).all(), "e2e record differs from the resident-program record"
    e2e_s = skdist.max_over_ranks(sum(e2e_times) / len(e2e_times))

    if rank == 0:
        algorithmic_bytes = sk.algorithmic_bytes           # SURVEY 8d formula over the device's own counters
        per_step = {k: cnt[k] / args.steps for k in ("n_rand", "n_det", "k_rand", "k_det")}
        per_step["gate_hist"] = [v / args.steps for v in cnt["gate_hist"]]
        layers_per_step = cnt["layers"] / args.steps
        total_bytes = algorithmic_bytes(circ.n, per_step, fused_layers=layers_per_step)
        n = circ.n; W = (n + 63) // 64; col = 2 * n / 8.0
        meas_bytes = per_step["n_rand"] * (col + 48 * W) + per_step["k_rand"] * 32 * W + per_step["n_det"] * col + per_step["k_det"] * 16 * W
        gate_bytes = total_bytes - meas_bytes
        peak, peak_src = peaks()
        # the measurement class = the cooperative kernel + the wave kernels (the algorithmic bytes of SURVEY 8d do not say which of
        # them took a deterministic measurement); their serialised times are also reported one by one below
        kern = {"k_measure_block": (meas_bytes, cls["measure_ms"] + cls["wave_ms"]), "k_layer": (gate_bytes, cls["layer_ms"])}
        dom = max(kern, key=lambda k: kern[k][1])
        traffic_all = {}
        try:
            import glob
            tf = sorted(glob.glob(os.path.join(ROOT, "profiles", "traffic_r*.json")))
            if tf:
                with open(tf[-1]) as f:
                    traffic_all = json.load(f)
        except Exception:
            traffic_all = {}
        traffic = traffic_all.get(dom, {}).get("bytes")
        notes = {
            "k_measure_block": "k_measure_block (cooperative: panel mode with the replicated level-form factorisation for the blocks with "
                               "random measurements, an immediate exit for the deterministic ones) + the wave kernels k_wave_cols / k_wave_rows "
                               "(the deterministic measurements of long blocks, one warp each), times of the serialised profile added up -- "
                               "see measure_ms_per_step / wave_ms_per_step; bound by chains of dependent accesses and two grid barriers per 64 "
                               "measurements, not by bandwidth: the fraction of the HBM peak is reported, not claimed as a roof",
            "k_layer": "NOT at a bandwidth roof although the algorithmic figure exceeds the HBM peak: SURVEY 8d charges every column of every gate, the "
                       "kernel skips the dependent loads and all stores of all-zero source words (ncu, one XCX/CX sub-layer, cold: 28.5 MB of DRAM reads and 0 "
                       "written against 76 MB algorithmic; warm: 6-7 MB read, 4-5 MB written) and the 51 MB gate form is partly L2 resident; ncu shows 49 % warps active, 16 % SM "
                       "throughput, long-scoreboard stalls: the launch is as long as its chain of dependent loads (8 gates x 2 per thread).  H a ; CX a->d.. ; H a windows are rewritten to XCX gates by the program compiler (4 sub-layers per surface-code round instead of 6); the algorithmic bytes keep counting the circuit's own gates"}
        roof = {"bound": "hbm", "kernel": dom, "achieved": kern[dom][0] / (kern[dom][1] * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                "traffic": traffic, "peak_source": peak_src, "note": notes[dom],
                "whole_step": {"algorithmic_bytes": total_bytes, "achieved": total_bytes / (ms_per_step * 1e-3) / 1e9,
                               "frac": total_bytes / (ms_per_step * 1e-3) / 1e9 / peak},
                "kernels": {k: {"algorithmic_bytes": v[0], "ms_per_step": v[1], "achieved": v[0] / (v[1] * 1e-3) / 1e9,
                                "frac": v[0] / (v[1] * 1e-3) / 1e9 / peak, "note": notes[k],
                                "traffic_one_launch": traffic_all.get(k, {}).get("bytes"), "traffic_what": traffic_all.get(k, {}).get("what")}
                            for k, v in kern.items()},
                "transpose_ms_per_step": cls["transpose_ms"],
                "transpose_note": "k_transpose_regs (one 32x32-bit block per thread, transposed in registers) is issue bound (ncu: 56 % issue active at 50 % occupancy): pure layout cost, no algorithmic bytes",
                "measure_ms_per_step": cls["measure_ms"],
                "wave_ms_per_step": cls["wave_ms"],
                "wave_note": "k_wave_cols + k_wave_rows: the deterministic measurements of long blocks, one warp each.  In an ordinary run k_wave_cols shares a launch with the transposition (k_transpose_wave) and k_wave_rows runs on a side stream under the next gate layers, so most of this class is off the critical path",
                "class_ms_sum": cls["layer_ms"] + cls["transpose_ms"] + cls["measure_ms"] + cls["wave_ms"],
                "class_ms_source": "CUDA events around every launch with every kernel on one stream, in order (sk_program_run_profiled: no graph, no programmatic overlap, no side stream); `value` is the graph replay of the pipelined program and is shorter than their sum"}
        roof["frac"] = roof["achieved"] / peak
        line = {"metric": METRIC, "value": ms_per_step * 1e-3, "unit": "s", "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3),
                "ms_per_step": ms_per_step, "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
                "data": "synthetic",
                "config": {"workload": workload, "seed": SEED, "parallelism": "replicas x%d (one full simulation per rank per step)" % world,
                           "l2": "flushed between steps (256 MiB write outside the event pair); working set 102 MB",
                           "timing": "CUDA events on the library stream around each step, mean of steps, max over ranks"},
                "e2e": {"value": e2e_s, "unit": "s", "h2d_bytes_per_step": int(len(circ.gates) * 12 + len(circ.chunk_marks) * 4),
                        "d2h_bytes_per_step": int(2 * circ.num_measurements), "call": "sk_sim(ctx, n, gates, marks, mode=0, seed) with pinned host buffers"},
                "gpu_launches": int(cnt["kernel_launches"]), "roofline": roof, "clocks": clocks,
                "counters_per_step": {k: per_step[k] for k in ("n_rand", "n_det", "k_rand", "k_det")} | {"waves": cnt["waves"] / args.steps, "layers": layers_per_step},
                "record_checksum": [int(out.sum()), int(det.sum())]}
        if not args.no_cpu_baseline:
            cb = cpu_reference(full=not args.cpu_sample)
            line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "cores_note", "extrapolated") if k in cb}
            if "measured_lower_bound_s" in cb:
                line["cpu_baseline"]["measured_lower_bound_s"] = cb["measured_lower_bound_s"]
        print(json.dumps(line))
    skdist.finalize()
    return 0


if __name__ == "__main__":
    sys.exit(main())
