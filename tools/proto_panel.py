"""CPU prototype of the PANEL (blocked elimination) measurement algorithm, validated against the
sequential CHP oracle.  A panel = B consecutive Z measurements.

  phase 1  symbolic: simulate the B measurements on the x bits of the panel's own columns only
           (R x B bit panel): pivots, frozen target masks m_l, pivot histories, deterministic
           partner sets -- no full-row work.
  phase 2  time-l pivot values  P_l' = (prod_{k in hist_l} P_k') * orig[p_l]      (B rows)
  phase 3  deterministic outcomes = sign( prod orig[i] * prod_{l in N_j} P_l' * prod (+-Z_{q_l}) )
  phase 4  every touched row replays its own multiplication list independently (row parallel).

Rows are python ints (bit q = qubit q); row index: stabilizer i -> i, destabilizer i -> n+i.
"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle_py as orc
import paper_2507_03092_b200 as sk
M = 9
MASK64 = (1 << 64) - 1


def splitmix64(x):
    x = (x + 0x9e3779b97f4a7c15) & MASK64
    x = ((x ^ (x >> 30)) * 0xbf58476d1ce4e5b9) & MASK64
    x = ((x ^ (x >> 27)) * 0x94d049bb133111eb) & MASK64
    return x ^ (x >> 31)


def counter_bit(seed, ordinal):
    return splitmix64(seed ^ splitmix64(ordinal ^ 0xd1b54a32d192ed03)) & 1


def g_sum(ax, az, bx, bz):
    """i-exponent of a*b (a = left factor)."""
    anti = (ax & bz) ^ (bx & az)
    plus = anti & ((ax & ~az & bx) | (ax & az & ~bx) | (~ax & az & ~bz))
    return bin(plus).count("1") - bin(anti & ~plus).count("1")


def lmul(a, b):
    """a * b for signed Hermitian commuting Paulis (x, z, r): rowsum(b, a)."""
    e = (2 * a[2] + 2 * b[2] + g_sum(a[0], a[1], b[0], b[1])) & 3
    assert e in (0, 2), "odd phase"
    return (a[0] ^ b[0], a[1] ^ b[1], e >> 1)


def to_int(words):
    v = 0
    for k, w in enumerate(words): v |= int(w) << (64 * k)
    return v


def panel(rows, n, qs, seed, ord0):
    """rows: list of 2n (x, z, r) tuples, updated in place.  Returns outcomes, dets."""
    B = len(qs)
    smask = (1 << n) - 1
    # phase 0: gather the panel (column form: bit h of cols[j] = x_{h, q_j})
    cols = [sum(((rows[h][0] >> q) & 1) << h for h in range(2 * n)) for q in qs]
    # phase 1
    frozen = [0] * B; piv = [-1] * B; hist = [0] * B; outc = [0] * B
    dN = [0] * B; dZ = [0] * B; dD = [0] * B
    pivmask = 0
    for j in range(B):
        col = cols[j]
        stab = col & smask
        if stab:
            p = (stab & -stab).bit_length() - 1
            piv[j] = p
            hist[j] = sum(((frozen[l] >> p) & 1) << l for l in range(j) if piv[l] >= 0)
            pw = sum(((cols[c] >> p) & 1) << c for c in range(j + 1, B))
            m = col & ~(1 << p) & ~(1 << (n + p))
            frozen[j] = m
            for c in range(j + 1, B):
                if (pw >> c) & 1: cols[c] ^= m
                cols[c] &= ~(1 << p)
                cols[c] = (cols[c] & ~(1 << (n + p))) | (((pw >> c) & 1) << (n + p))
            outc[j] = counter_bit(seed, ord0 + j)
            pivmask |= 1 << p
        else:
            D = col >> n
            nonpiv = D & ~pivmask
            dD[j] = nonpiv
            dN[j] = sum((bin(frozen[l] & nonpiv).count("1") & 1) << l for l in range(j) if piv[l] >= 0)
            dZ[j] = sum(((D >> piv[l]) & 1) << l for l in range(j) if piv[l] >= 0)
    # phase 2: time-l pivot values
    P = [None] * B
    for k in range(B):
        if piv[k] < 0: continue
        acc = rows[piv[k]]
        for l in range(k):
            if (hist[k] >> l) & 1: acc = lmul(P[l], acc)
        P[k] = acc
    # phase 3: deterministic outcomes (reads panel-start rows)
    for j in range(B):
        if piv[j] >= 0: continue
        acc = (0, 0, 0)
        for i in range(n):
            if (dD[j] >> i) & 1: acc = lmul(rows[i], acc)
        for l in range(j):
            if (dN[j] >> l) & 1: acc = lmul(P[l], acc)
        for l in range(j):
            if (dZ[j] >> l) & 1: acc = lmul((0, 1 << qs[l], outc[l]), acc)
        assert acc[0] == 0 and acc[1] == 1 << qs[j], "deterministic product is not +-Z_q"
        outc[j] = acc[2]
    # phase 4: row-parallel replay
    new = {}
    touched = 0
    for l in range(B): touched |= frozen[l]
    ow = {}     # destabilizer row -> step that overwrote it
    for k in range(B):
        if piv[k] >= 0: ow[n + piv[k]] = k
    for h in range(2 * n):
        if h < n and (pivmask >> h) & 1:
            k = piv.index(h)
            new[h] = (0, 1 << qs[k], outc[k]); continue
        if h in ow:
            k = ow[h]; acc = P[k]; start = k + 1
        elif (touched >> h) & 1:
            acc = rows[h]; start = 0
        else:
            continue
        for l in range(start, B):
            if piv[l] >= 0 and (frozen[l] >> h) & 1: acc = lmul(P[l], acc)
        new[h] = acc
    for h, v in new.items(): rows[h] = v
    return outc, [int(p < 0) for p in piv]


def check(circ, seed, B):
    g = circ.gates; n = circ.n
    ref = orc.Tableau(n); ro, rd, rc = ref.sim(g, seed)
    assert rc == 0
    t = orc.Tableau(n); i = 0; ordn = 0; outs = []; dets = []
    kinds = g["kind"]
    while i < len(g):
        j = i
        if kinds[i] == M:
            while j < len(g) and kinds[j] == M: j += 1
            qs = [int(q) for q in g["q0"][i:j]]
            x, z, r = t.get()
            rows = [(to_int(x[h]), to_int(z[h]), int(r[h])) for h in range(2 * n)]
            for b0 in range(0, len(qs), B):
                o, d = panel(rows, n, qs[b0:b0 + B], seed, ordn + b0)
                outs += o; dets += d
            W = x.shape[1]
            for h in range(2 * n):
                for w in range(W):
                    x[h, w] = (rows[h][0] >> (64 * w)) & MASK64; z[h, w] = (rows[h][1] >> (64 * w)) & MASK64
                r[h] = rows[h][2]
            t.set(x, z, r)
            ordn += len(qs)
        else:
            while j < len(g) and kinds[j] != M: j += 1
            t.sim(g[i:j], seed)
        i = j
    o = np.array(outs, np.uint8); d = np.array(dets, np.uint8)
    return (o == ro).all() and (d == rd).all() and all((a == b).all() for a, b in zip(t.get(), ref.get()))


if __name__ == "__main__":
    for d in (3, 5, 7):
        for B in (1, 4, 64):
            print("surface d", d, "B", B, "ok", check(sk.surface_code_circuit(d, 3, True), 20250703, B))
    rng = np.random.default_rng(0)
    bad = 0
    for trial in range(400):
        n = int(rng.integers(1, 14)); gates = []
        for _ in range(int(rng.integers(5, 80))):
            if rng.random() < 0.35 or n == 1:
                for _ in range(int(rng.integers(1, 12))): gates.append((M, int(rng.integers(0, n)), 0))
            else:
                k = int(rng.choice([0, 1, 6, 6, 6, 7, 8])); a = int(rng.integers(0, n)); b = int(rng.integers(0, n - 1)); b += b >= a
                gates.append((k, a, b))
        ok = check(sk.Circuit(n, gates), int(rng.integers(0, 2**60)), B=int(rng.choice([1, 2, 3, 5, 8, 64])))
        bad += not ok
    print("random circuits: failures", bad, "of 400")
    for n in (16, 64):
        print("random_layered", n, check(sk.random_layered_circuit(n, 5), 9, 16))
