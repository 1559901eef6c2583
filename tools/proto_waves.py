"""CPU prototype of the out-of-order wave scheduler, validated against sequential CHP (oracle)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle_py as orc
import paper_2507_03092_b200 as sk
M = 9

def xcol(x, q):
    return ((x[:, q >> 6] >> np.uint64(q & 63)) & np.uint64(1)).astype(bool)

def run_block(t, n, qs, seed, ord0, GW=10**9, rule="r0"):
    """execute measurement list qs on oracle tableau t with the wave rule; returns outcomes, dets, waves"""
    m = len(qs); done = np.zeros(m, bool); out = np.zeros(m, np.uint8); det = np.zeros(m, np.uint8); waves = 0
    while not done.all():
        waves += 1
        x, z, r = t.get()
        pos = int(np.argmin(done))
        win = [j for j in range(pos, min(m, pos + GW)) if not done[j]]
        foot = {}; typ = {}
        for j in win:
            c = xcol(x, qs[j])
            slots = set(int(i) % n for i in np.nonzero(c)[0])
            rand = c[:n].any()
            if rand: slots.add(int(np.argmax(c[:n])))
            foot[j] = slots; typ[j] = rand
        rands = [j for j in win if typ[j]]
        r0 = rands[0] if rands else 10**18
        claim = {}
        for j in win:
            if j >= r0:
                for s in foot[j]: claim[s] = min(claim.get(s, 10**18), j)
        ex = []
        for j in win:
            if j < r0: ex.append(j)
            elif all(claim[s] >= j for s in foot[j]): ex.append(j)
        assert ex and ex[0] == win[0]
        # dets first (they read the wave-start state), then randoms -- any order within each class
        for j in [k for k in ex if not typ[k]] + [k for k in ex if typ[k]][::-1]:
            o, d, rc = t.sim([(M, qs[j], 0)], seed, ordinal0=ord0 + j)
            assert rc == 0 and d[0] == (0 if typ[j] else 1), (j, typ[j], d)
            out[j], det[j] = o[0], d[0]; done[j] = True
    return out, det, waves

def check(circ, seed, GW=10**9):
    g = circ.gates; n = circ.n
    ref = orc.Tableau(n); ro, rd, _ = ref.sim(g, seed)
    t = orc.Tableau(n); i = 0; ordn = 0; outs = []; dets = []; wv = []
    kinds = g["kind"]
    while i < len(g):
        j = i
        if kinds[i] == M:
            while j < len(g) and kinds[j] == M: j += 1
            qs = [int(q) for q in g["q0"][i:j]]
            o, d, w = run_block(t, n, qs, seed, ordn, GW)
            outs.append(o); dets.append(d); wv.append((len(qs), w)); ordn += len(qs)
        else:
            while j < len(g) and kinds[j] != M: j += 1
            t.sim(g[i:j], seed)
        i = j
    o = np.concatenate(outs); d = np.concatenate(dets)
    ok = (o == ro).all() and (d == rd).all() and all((a == b).all() for a, b in zip(t.get(), ref.get()))
    return ok, wv

if __name__ == "__main__":
    for d in (3, 5, 7, 9, 11):
        ok, wv = check(sk.surface_code_circuit(d, 3, True), 20250703)
        print("surface d", d, "ok", ok, "blocks (size,waves):", wv)
    rng = np.random.default_rng(0)
    bad = 0
    for trial in range(300):
        n = int(rng.integers(2, 14)); gates = []
        for _ in range(int(rng.integers(5, 80))):
            if rng.random() < 0.35:
                for _ in range(int(rng.integers(1, 12))): gates.append((M, int(rng.integers(0, n)), 0))
            else:
                k = int(rng.choice([0, 1, 6, 6, 6, 7, 8])); a = int(rng.integers(0, n)); b = int(rng.integers(0, n - 1)); b += b >= a
                gates.append((k, a, b))
        ok, wv = check(sk.Circuit(n, gates), int(rng.integers(0, 2**60)), GW=int(rng.choice([3, 5, 100])))
        bad += not ok
    print("random circuits: failures", bad, "of 300")
    for n in (16, 64):
        ok, wv = check(sk.random_layered_circuit(n, 5), 9)
        print("random_layered", n, ok, wv)
