"""All five BASELINE.json configs on one GPU, each beside the CPU oracle (test infrastructure) on the
same inputs; parity is asserted wherever the oracle is run at the same size.  Scratch tool: the
headline line is bench.py.  Usage: python tools/bench_configs.py [--quick] [--c4-n N]"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2507_03092_b200 as sk
from oracle import oracle_py as orc

ap = argparse.ArgumentParser(); ap.add_argument("--quick", action="store_true"); ap.add_argument("--c4-n", type=int, default=1_000_000)
ap.add_argument("--c4-cpu-n", type=int, default=100_000); args = ap.parse_args()
ctx = sk.Context(0); SEED = 20250703; cores = os.cpu_count()
out = []

def timed(f):
    ctx.sync(); t0 = time.perf_counter(); r = f(); ctx.sync(); return r, time.perf_counter() - t0

# ---- C1-C3 surface code ------------------------------------------------------------------------
for name, d, cpu_rounds in (("C1 surface d=3", 3, 3), ("C2 surface d=25", 25, 25), ("C3 surface d=71", 71, 2 if args.quick else 6)):
    circ = sk.surface_code_circuit(d, d, True)
    ctx.sim(circ, SEED)[0].close()                               # warm-up
    (t, o, dt, _), gpu_s = timed(lambda: ctx.sim(circ, SEED))
    cc = sk.surface_code_circuit(d, cpu_rounds, True) if cpu_rounds != d else circ
    ot = orc.Tableau(cc.n); t0 = time.perf_counter(); oo, od, _ = ot.sim(cc.gates, SEED, workers=cores); cpu_s = time.perf_counter() - t0
    parity = None
    if cpu_rounds == d:
        x, z, r = t.download(); ox, oz, orr = ot.get()
        parity = bool((o == oo).all() and (dt == od).all() and (x == ox).all() and (z == oz).all() and (r == orr).all())
    out.append({"config": name, "gpu_e2e_s": gpu_s, "cpu_s": cpu_s * d / cpu_rounds, "cpu_sample": f"{cpu_rounds} of {d} rounds, {cores} threads", "bit_exact": parity})
    t.close(); print(json.dumps(out[-1]), flush=True)

# ---- C4 grouping: N random 128-qubit Paulis (SURVEY 8d generator) ----------------------------------
def c4_terms(N):
    raw = np.zeros(5 * N + 64, np.uint64); orc.lib().orc_seq_fill(SEED, orc._p(raw), len(raw))
    v = raw[:5 * N].reshape(N, 5)
    x = np.ascontiguousarray(v[:, 0:2]); z = np.ascontiguousarray(v[:, 2:4])
    coeff = 2.0 * ((v[:, 4] >> np.uint64(11)).astype(np.float64) * 2.0 ** -53) - 1.0
    order = np.argsort(-np.abs(coeff), kind="stable")            # |coeff| desc; ties (none in practice) keep input order
    return np.ascontiguousarray(x[order]), np.ascontiguousarray(z[order])
for mode, mname in ((0, "GC"), (1, "QWC")):
    N = 20000 if args.quick else args.c4_n
    x, z = c4_terms(N)
    rows = sk.Rows(ctx, 128, x, z)
    (g, ng), gpu_s = timed(lambda: rows.group_first_fit(mode))
    (nv), ver_s = timed(lambda: rows.verify_grouping(mode, g))
    Nc = min(N, 5000 if args.quick else args.c4_cpu_n)
    xo, zo = c4_terms(Nc)
    o = orc.Rows(128, xo, zo, np.zeros(Nc, np.uint8)); t0 = time.perf_counter(); og, ong, calls = o.group_first_fit(mode); cpu_s = time.perf_counter() - t0
    small = sk.Rows(ctx, 128, xo, zo); sg, sng = small.group_first_fit(mode)
    out.append({"config": f"C4 grouping {mname} N={N} n=128", "gpu_s": gpu_s, "groups": ng, "verify_violations": nv, "verify_s": ver_s,
                "pairs_per_s": N * (N - 1) / 2 / gpu_s, "cpu_s_at": {"N": Nc, "s": cpu_s, "pred_calls": calls},
                "bit_exact_at_cpu_N": bool(sng == ong and (sg == og).all())})
    rows.close(); small.close(); print(json.dumps(out[-1]), flush=True)

# ---- C5 Clifford+T transpile: n=1000, G gates, 10 % T (SURVEY 8d generator) -------------------------
def c5_circuit(n, G):
    raw = np.zeros(4 * G + 64, np.uint64); orc.lib().orc_seq_fill(20250704, orc._p(raw), len(raw))
    gates = np.zeros(G, sk.GATE_DTYPE); k = 0
    def nxt():
        nonlocal k; v = int(raw[k]); k += 1; return v
    for i in range(G):
        u = (nxt() >> 11) * 2.0 ** -53
        if u < 0.05: gates[i] = (sk.T, 0, nxt() % n, 0)
        elif u < 0.10: gates[i] = (sk.TDG, 0, nxt() % n, 0)
        elif u < 0.40: gates[i] = (sk.H, 0, nxt() % n, 0)
        elif u < 0.70: gates[i] = (sk.S, 0, nxt() % n, 0)
        else:
            c = nxt() % n; t = nxt() % n
            while t == c: t = nxt() % n
            gates[i] = (sk.CX, 0, c, t)
    return sk.Circuit(n, gates)
G = 10000 if args.quick else 100000
circ = c5_circuit(1000, G)
sk.Pbc(ctx, circ).close()
p, gpu_s = timed(lambda: sk.Pbc(ctx, circ))
t0 = time.perf_counter(); op = orc.Pbc(1000, circ.gates, exact=True); cpu_s = time.perf_counter() - t0
same = p.stats() == op.stats()
for k in range(p.stats()["layers"]):
    a, b = p.layer(k), op.layer(k); same = same and all((u == v).all() for u, v in zip(a, b))
same = same and all((u == v).all() for u, v in zip(p.mtab(), op.mtab().get()))
out.append({"config": f"C5 transpile n=1000 G={G}", "gpu_s": gpu_s, "cpu_s": cpu_s, "stats": p.stats(), "bit_exact": bool(same)})
print(json.dumps(out[-1]), flush=True)
json.dump(out, open("gpurun_out/configs.json", "w"), indent=1)
