"""Dense tableaux (deep random Clifford circuit, then every qubit measured): the regime of the paper's random workload where
each random measurement multiplies ~n rows.  GPU sk_sim (host buffers) beside the CPU oracle; parity asserted."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2507_03092_b200 as sk
from oracle import oracle_py as orc
H, S, CX, M = 0, 1, 6, 9
ctx = sk.Context(0); cores = os.cpu_count(); out = []
for n in (512, 1024, 2048, 4096):
    rng = np.random.default_rng(n)
    g = np.zeros(12 * n, sk.GATE_DTYPE)
    kinds = rng.choice([H, S, CX, CX], size=10 * n)
    a = rng.integers(0, n, 10 * n); b = rng.integers(0, n - 1, 10 * n); b += b >= a
    g["kind"][:10 * n] = kinds; g["q0"][:10 * n] = a; g["q1"][:10 * n] = np.where(kinds == CX, b, 0)
    g["kind"][10 * n:11 * n] = M; g["q0"][10 * n:11 * n] = rng.permutation(n)
    g = g[:11 * n]
    circ = sk.Circuit(n, g)
    ctx.sim(circ, 5)[0].close()
    ctx.reset_counters(); ctx.sync(); t0 = time.perf_counter(); t, o, d, _ = ctx.sim(circ, 5); ctx.sync(); gpu_s = time.perf_counter() - t0
    cnt = ctx.counters()
    ot = orc.Tableau(n); t0 = time.perf_counter(); oo, od, rc = ot.sim(circ.gates, 5, workers=cores); cpu_s = time.perf_counter() - t0
    x, z, r = t.download(); ox, oz, orr = ot.get()
    ok = bool(rc == 0 and (o == oo).all() and (d == od).all() and (x == ox).all() and (z == oz).all() and (r == orr).all())
    out.append({"n": n, "gates": int(10 * n), "measurements": n, "n_rand": cnt["n_rand"], "k_rand": cnt["k_rand"], "k_det": cnt["k_det"],
                "gpu_e2e_s": gpu_s, "cpu_s": cpu_s, "cpu_threads": cores, "bit_exact": ok})
    print(json.dumps(out[-1]), flush=True); t.close()
json.dump(out, open("gpurun_out/dense.json", "w"), indent=1)
