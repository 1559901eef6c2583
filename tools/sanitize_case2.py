"""Second workload for compute-sanitizer memcheck: the kernels that only run at size -- the register-block transposition and the
split wave kernels (surface code d=47: 4 417 qubits, blocks of 2 208 measurements), the program path with its side stream, and the
pipelined grouping (resolver with precomputed conflicts, k_conflict_prev) on 5 000 random 128-qubit terms.
Usage: compute-sanitizer --tool memcheck python tools/sanitize_case2.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2507_03092_b200 as sk
from oracle import oracle_py as orc
ctx = sk.Context(0)
circ = sk.surface_code_circuit(47, 2, True)
t, out, det, _ = ctx.sim(circ, 7)
o = orc.Tableau(circ.n); oo, od, rc = o.sim(circ.gates, 7, workers=8)
ok = rc == 0 and (out == oo).all() and (det == od).all()
prog = sk.Program(ctx, circ); t2 = sk.Tableau(ctx, circ.n); prog.run(t2, 7); ctx.sync()
x, z, r = t2.download(); ox, oz, orr = o.get()
ok = ok and (x == ox).all() and (z == oz).all() and (r == orr).all()
t.close(); t2.close()
rng = np.random.default_rng(1)
N = 5000
xs = rng.integers(0, 2**64, (N, 2), dtype=np.uint64); zs = rng.integers(0, 2**64, (N, 2), dtype=np.uint64)
rows = sk.Rows(ctx, 128, xs, zs, np.zeros(N, np.uint8)); orows = orc.Rows(128, xs, zs, np.zeros(N, np.uint8))
for mode in (0, 1):
    g, ng = rows.group_first_fit(mode); og, ong, _ = orows.group_first_fit(mode)
    ok = ok and ng == ong and (g == og).all()
rows.close(); ctx.close()
print("sanitize_case2 parity:", bool(ok))
