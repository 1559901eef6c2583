"""Parity of the paths that only run at size, on circuits that are NOT surface codes: long measurement blocks (>= 2 048: the wave
kernels, fused with the register-block transposition when the word count is even) that are all-random, all-deterministic and mixed,
with Clifford layers in between.  n = 4 480 (even word count) and 4 416 (odd: shuffle transposition, separate k_wave_cols).
Usage: python tools/stress_wave.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2507_03092_b200 as sk
from oracle import oracle_py as orc
H, S, SDG, X, Y, Z, CX, CZ, SWAP, M = range(10)
ok = True
DEPTH = int(sys.argv[1]) if len(sys.argv) > 1 else 1          # extra entangling layers in front: denser rows, longer partner lists
for n in (4480, 4416):
    for seed in (1, 2):
        rng = np.random.default_rng(100 * n + seed)
        g = []
        def layer(kinds, frac):
            qs = rng.permutation(n)
            k = 0
            while k + 1 < int(frac * n):
                kind = int(rng.choice(kinds))
                if kind in (CX, CZ, SWAP): g.append((kind, int(qs[k]), int(qs[k + 1]))); k += 2
                else: g.append((kind, int(qs[k]), 0)); k += 1
        for _ in range(DEPTH): layer((H, S, X), 0.5); layer((CX, CZ), 0.8); layer((H, SDG, Y), 0.3); layer((CX, SWAP), 0.6)
        g += [(M, q, 0) for q in range(n)]                              # mixed random / deterministic
        g += [(M, int(q), 0) for q in rng.permutation(n)[:3000]]        # all deterministic now: the wave kernels own the block
        layer((H, H, S), 0.4); layer((CX, CZ), 0.9)
        g += [(M, int(q), 0) for q in rng.permutation(n)[:2500]]
        layer((CX,), 0.7)
        g += [(M, q, 0) for q in range(n - 1, -1, -1)]
        circ = sk.Circuit(n, g)
        ctx = sk.Context(0)
        t0 = time.time()
        t, out, det, _ = ctx.sim(circ, 77 + seed)
        prog = sk.Program(ctx, circ); t2 = sk.Tableau(ctx, n); prog.run(t2, 77 + seed); ctx.sync()
        o2, d2 = prog.read_record()
        t1 = time.time()
        o = orc.Tableau(n); oo, od, rc = o.sim(circ.gates, 77 + seed, workers=8)
        x, z, r = t.download(); x2, z2, r2 = t2.download(); ox, oz, orr = o.get()
        good = rc == 0 and (out == oo).all() and (det == od).all() and (o2 == oo).all() and (d2 == od).all() and \
               (x == ox).all() and (z == oz).all() and (r == orr).all() and (x2 == ox).all() and (z2 == oz).all() and (r2 == orr).all()
        print(f"n={n} seed={seed}: {len(g)} ops, {int((od == 0).sum())} random / {int((od == 1).sum())} deterministic measurements, gpu {t1 - t0:.2f} s, oracle {time.time() - t1:.1f} s ->", "ok" if good else "MISMATCH")
        ok = ok and good
        t.close(); t2.close(); ctx.close()
print("stress_wave parity:", ok)
