"""Small mixed workload for compute-sanitizer (memcheck / racecheck): surface code d=5 + random circuits with
measurements, both panel factorisations.  Usage: compute-sanitizer --tool memcheck python tools/sanitize_case.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2507_03092_b200 as sk
from oracle import oracle_py as orc
H, S, CX, M = 0, 1, 6, 9
def rand_gates(rng, n, count, pm):
    g = []
    for _ in range(count):
        if rng.random() < pm: g.append((M, int(rng.integers(0, n)), 0))
        else:
            k = int(rng.choice([H, S, CX, CX])); a = int(rng.integers(0, n)); b = int(rng.integers(0, n - 1)); b += b >= a
            g.append((k, a, b))
    return g
ok = True
for columns in (0, 1):
    os.environ["SK_PANEL_COLUMNS"] = str(columns)
    ctx = sk.Context(0)
    rng = np.random.default_rng(5)
    circs = [(sk.surface_code_circuit(5, 2, True), 3), (sk.Circuit(70, rand_gates(rng, 70, 400, 0.2)), 9)]
    for circ, seed in circs:
        t, out, det, _ = ctx.sim(circ, seed)
        o = orc.Tableau(circ.n); oo, od, rc = o.sim(circ.gates, seed)
        x, z, r = t.download(); ox, oz, orr = o.get()
        ok = ok and rc == 0 and (out == oo).all() and (det == od).all() and (x == ox).all() and (z == oz).all() and (r == orr).all()
        t.close()
    ctx.close()
print("sanitize_case parity:", ok)
