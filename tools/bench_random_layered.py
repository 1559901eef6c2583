"""SURVEY 8f item 1 / SPEC acceptance #6: random layered circuits n in {256..4096}, GPU (sk_sim, host buffers) beside the
CPU oracle (all host threads), parity asserted.  Mixes random and deterministic measurements on DENSE tableaux, so the
measurement kernel's column-form panel factorisation is what runs for the larger n."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2507_03092_b200 as sk
from oracle import oracle_py as orc
ctx = sk.Context(0); cores = os.cpu_count(); out = []
for n in (256, 512, 1024, 2048, 4096):
    circ = sk.random_layered_circuit(n, 20250703)
    ctx.sim(circ, 5)[0].close()
    ctx.reset_counters(); ctx.sync(); t0 = time.perf_counter(); t, o, d, _ = ctx.sim(circ, 5); ctx.sync(); gpu_s = time.perf_counter() - t0
    cnt = ctx.counters()
    ot = orc.Tableau(n); t0 = time.perf_counter(); oo, od, rc = ot.sim(circ.gates, 5, workers=cores); cpu_s = time.perf_counter() - t0
    x, z, r = t.download(); ox, oz, orr = ot.get()
    ok = bool(rc == 0 and (o == oo).all() and (d == od).all() and (x == ox).all() and (z == oz).all() and (r == orr).all())
    out.append({"n": n, "gates": int(len(circ.gates)), "measurements": int(circ.num_measurements), "n_rand": cnt["n_rand"], "n_det": cnt["n_det"],
                "k_rand": cnt["k_rand"], "k_det": cnt["k_det"], "gpu_e2e_s": gpu_s, "cpu_s": cpu_s, "cpu_threads": cores, "bit_exact": ok})
    print(json.dumps(out[-1]), flush=True); t.close()
json.dump(out, open("gpurun_out/random_layered.json", "w"), indent=1)
