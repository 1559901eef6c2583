"""Randomised parity stress: many random circuits (varied n, gate mixes, measurement densities, panel widths, row caps,
folded / standalone gather) against the CPU oracle.  Usage: python tools/stress_parity.py [seconds]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2507_03092_b200 as sk
from oracle import oracle_py as orc
H, S, SDG, X, Y, Z, CX, CZ, SWAP, M = range(10)
budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rng = np.random.default_rng(int(time.time()) & 0xffff)
t_end = time.time() + budget
runs = fails = sruns = 0
while time.time() < t_end:
    os.environ["SK_PANEL"] = str(int(rng.choice([1, 3, 8, 17, 64, 64, 64])))
    os.environ["SK_ROW_CAP"] = str(int(rng.choice([0, 0, 0, 10, 40, 150])))
    os.environ["SK_NO_FOLD"] = str(int(rng.random() < 0.25))
    os.environ["SK_PANEL_COLUMNS"] = str(int(rng.random() < 0.15))
    os.environ["SK_NO_GRAPH"] = str(int(rng.random() < 0.5))
    ctx = sk.Context(0)
    for _ in range(6):
        n = int(rng.choice([1, 2, 3, 7, 31, 64, 65, 100, 129, 200, 333, 640]))
        count = int(rng.integers(5, 12 * n + 50))
        pm = float(rng.choice([0.02, 0.1, 0.3, 0.6]))
        gates = []
        while len(gates) < count:
            if rng.random() < pm:
                for _ in range(int(rng.integers(1, 2 * n + 2))): gates.append((M, int(rng.integers(0, n)), 0))
            else:
                k = int(rng.choice([H, S, SDG, X, Y, Z, CX, CX, CX, CZ, SWAP])); a = int(rng.integers(0, n)); b = 0
                if k in (CX, CZ, SWAP):
                    if n == 1: k = H
                    else: b = int(rng.integers(0, n - 1)); b += b >= a
                gates.append((k, a, b))
        circ = sk.Circuit(n, gates); seed = int(rng.integers(0, 2**62))
        mode = int(rng.random() < 0.3)
        t, out, det, _ = ctx.sim(circ, seed, mode=mode)
        o = orc.Tableau(n); oo, od, rc = o.sim(circ.gates, seed, workers=4)
        x, z, r = t.download(); ox, oz, orr = o.get()
        ok = rc == 0 and (out == oo).all() and (det == od).all() and (x == ox).all() and (z == oz).all() and (r == orr).all()
        runs += 1
        if not ok:
            fails += 1
            print("MISMATCH n", n, "gates", len(gates), "env", {k: os.environ[k] for k in ("SK_PANEL", "SK_ROW_CAP", "SK_NO_FOLD", "SK_PANEL_COLUMNS", "SK_NO_GRAPH")}, flush=True)
        t.close()
        if rng.random() < 0.15 and len(gates) < 1500:        # the same circuit on a row-sharded tableau (1..8 shards on this GPU)
            from paper_2507_03092_b200.sharded import ShardedTableau
            L = int(rng.choice([1, 2, 3, 5, 8]))
            st = ShardedTableau.create_cuda(n, local_shards=L, device_index=0)
            so, sd = st.sim(circ, seed)
            sx, sz, sr = st.gather_tableau()
            st.close()
            sruns += 1
            if not ((so == oo).all() and (sd == od).all() and (sx == ox).all() and (sz == oz).all() and (sr == orr).all()):
                fails += 1
                print("SHARDED MISMATCH n", n, "gates", len(gates), "shards", L, flush=True)
    ctx.close()
print(f"stress: {runs} circuits ({sruns} also row-sharded), {fails} mismatches")
sys.exit(1 if fails else 0)
