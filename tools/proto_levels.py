"""CPU prototype of the LEVEL-FORM panel factorisation (kernels_panel.cuh: lv_factorise; kernels_measure.cuh:
panel_factorise_levels), validated against the step-by-step symbolic elimination `seq` below.

State: pairs (stabilizer i, destabilizer n+i) with their bits in the panel's columns (sb, db).  A round executes every step
whose outcome no earlier unfinished step can influence (see DESIGN.md section 5 for the rule); `levelset3` returns the same
pivots, pivot histories, step masks, `born` markers and deterministic partner sets as `seq`.
Usage: python tools/proto_levels.py        (30 000 random bit matrices)"""
import random

INF = -1
K = 4          # rows with more set bits than this contribute for their lowest column only (kLevelK)


def above(l): return ~((2 << l) - 1)
def seq(pairs, B):
    # pairs: dict i -> [sbits, dbits]; returns piv, hist, Ms, Md (dict), born, dpart, dZ
    sb = {i: v[0] for i, v in pairs.items()}; db = {i: v[1] for i, v in pairs.items()}
    Ms = {i: 0 for i in pairs}; Md = {i: 0 for i in pairs}; born = {i: 0 for i in pairs}
    piv = [INF] * B; hist = [0] * B; dpart = [set() for _ in range(B)]; dZ = [0] * B; rowM = {}
    for l in range(B):
        st = [i for i in sb if (sb[i] >> l) & 1]
        if not st:
            for i in db:
                if (db[i] >> l) & 1:
                    if born[i]: dZ[l] |= 1 << (born[i] - 1)
                    else: dpart[l].add(i)
            continue
        p = min(st); bp = sb[p]; piv[l] = p; hist[l] = Ms[p]; rowM[p] = Ms[p]
        for i in sb:
            if i != p and (sb[i] >> l) & 1: sb[i] ^= bp & above(l) | (1 << l); Ms[i] |= 1 << l
        for i in db:
            if i != p and (db[i] >> l) & 1: db[i] ^= bp & above(l) | (1 << l); Md[i] |= 1 << l
        sb[p] = 0; db[p] = bp & above(l); Md[p] = 0; born[p] = l + 1
    return piv, hist, Ms, Md, born, dpart, dZ


def below(l): return (1 << l) - 1
def levelset3(pairs, B, stats=None):
    sb = {i: v[0] for i, v in pairs.items()}; db = {i: v[1] for i, v in pairs.items()}
    Ms = {i: 0 for i in pairs}; Md = {i: 0 for i in pairs}; born = {i: 0 for i in pairs}
    piv = [INF] * B; hist = [0] * B; dpart = [set() for _ in range(B)]; dZ = [0] * B
    U = (1 << B) - 1; rounds = 0
    while U:
        rounds += 1
        cand = {}; A = [0] * B; forced = 0
        for i in sb:
            s = sb[i] & U
            if not s: continue
            d = db[i] & U
            nb = bin(s).count('1')
            if nb > K:
                low = (s & -s).bit_length() - 1
                forced |= 1 << low
                cand[low] = min(cand.get(low, 1 << 60), i)
                A[low] |= (s | d) & above(low)
            else:
                t = s
                while t:
                    j = (t & -t).bit_length() - 1; t &= t - 1
                    cand[j] = min(cand.get(j, 1 << 60), i)
                    A[j] |= (s | d) & above(j)
        T = [0] * B; J = [0] * B; Js = [0] * B; conf = 0; H = 0
        for j in range(B):
            if not (U >> j) & 1: continue
            if j not in cand: H |= 1 << j; continue      # deterministic step: modifies nothing
            c = cand[j]
            s = sb[c] & U; d = db[c] & U
            T[j] = (s | d) & above(j); J[j] = (s | d) & below(j); Js[j] = s & below(j)
            t = Js[j]
            while t:
                j2 = (t & -t).bit_length() - 1; t &= t - 1
                if cand[j2] == c: conf |= 1 << j
            if T[j] == 0 and not (forced >> j) & 1: H |= 1 << j
        acc = 0
        for l in range(B):
            if (U >> l) & 1 and not (H >> l) & 1: acc |= A[l]
        while True:
            ready = 0
            for l in range(B):
                if (U >> l) & 1 and not (acc >> l) & 1 and not (conf >> l) & 1 and (J[l] & ~H) == 0: ready |= 1 << l
            newH = H & ready
            if newH == H: break
            for l in range(B):
                if ((H & ~newH) >> l) & 1: acc |= A[l]
            H = newH
        assert ready, (bin(U), bin(acc))
        pv = {l: cand[l] for l in range(B) if (ready >> l) & 1 and l in cand}
        nsb = dict(sb); ndb = dict(db)
        for i in sb:
            s = sb[i] & ready
            ispiv = False
            l = None
            t = s
            while t:
                l = (t & -t).bit_length() - 1; t &= t - 1
                if pv[l] == i: ispiv = True; break
            if ispiv:
                assert sb[i] & ready & above(l) == 0
                Ms[i] |= sb[i] & ready & below(l)
                piv[l] = i; hist[l] = Ms[i]
                nsb[i] = 0; ndb[i] = sb[i] & above(l); Md[i] = 0; bornold = born[i]; born[i] = l + 1
                h = db[i] & ready & below(l)
                while h:
                    l2 = (h & -h).bit_length() - 1; h &= h - 1
                    if l2 not in pv:
                        if bornold: dZ[l2] |= 1 << (bornold - 1)
                        else: dpart[l2].add(i)
            else:
                v = sb[i]; t = s
                while t:
                    l = (t & -t).bit_length() - 1; t &= t - 1
                    v ^= (sb[pv[l]] & above(l)) | (1 << l); Ms[i] |= 1 << l
                nsb[i] = v
                h = db[i] & ready; v = db[i]
                while h:
                    l = (h & -h).bit_length() - 1; h &= h - 1
                    if l in pv:
                        v ^= (sb[pv[l]] & above(l)) | (1 << l); Md[i] |= 1 << l
                    else:
                        if born[i]: dZ[l] |= 1 << (born[i] - 1)
                        else: dpart[l].add(i)
                ndb[i] = v
        sb, db = nsb, ndb
        U &= ~ready
    return (piv, hist, Ms, Md, born, dpart, dZ), rounds

if __name__ == '__main__':
    random.seed(2)
    tot = 0; N = 30000
    for trial in range(N):
        B = random.choice([1, 2, 5, 8, 16, 64])
        npairs = random.randint(1, 40)
        dens = random.choice([0.01, 0.02, 0.05, 0.15, 0.5])
        pairs = {}
        for i in random.sample(range(100), npairs):
            s = sum((random.random() < dens * random.choice([0, 1, 1])) << c for c in range(B))
            d = sum((random.random() < dens) << c for c in range(B))
            if s | d: pairs[i] = [s, d]
        a = seq(pairs, B); b, r = levelset3(pairs, B); tot += r
        if a != b:
            print("MISMATCH", trial, B, pairs); print(a); print(b); break
    else:
        print("all equal; mean rounds", tot / N)
