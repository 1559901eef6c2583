"""SPEC.md known-answer examples on the oracle (the reference ships these algorithms as
specification only, so these examples are what pins the oracle's drivers)."""
import numpy as np
import pytest

H, S, SDG, X, Y, Z, CX, CZ, SWAP, M, T, TDG = range(12)


def rows_after(orc, texts, gates):
    r = orc.Rows.from_text(texts); r.apply(gates); return r.texts()


def test_sign_identities(orc):                      # SPEC:141-143,151-153,161-163, acceptance #4
    assert rows_after(orc, ["Z", "Y", "X"], [(H, 0)]) == ["+X", "-Y", "+Z"]
    assert rows_after(orc, ["X", "Y", "Z"], [(S, 0)]) == ["+Y", "-X", "+Z"]
    assert rows_after(orc, ["X", "Y"], [(SDG, 0)]) == ["-Y", "+X"]
    assert rows_after(orc, ["XI", "IZ", "YY"], [(CX, 0, 1)]) == ["+XX", "+ZZ", "-XZ"]
    assert rows_after(orc, ["Z"], [(X, 0)]) == ["-Z"]
    assert rows_after(orc, ["XI", "IZ"], [(SWAP, 0, 1)]) == ["+IX", "+ZI"]
    assert rows_after(orc, ["Y", "Z"], [(H, 0), (H, 0)]) == ["+Y", "+Z"]


def test_new_identity(orc):
    assert orc.Tableau(1).texts() == ["+Z", "+X"]
    assert orc.Tableau(3).texts()[:3] == ["+ZII", "+IZI", "+IIZ"]
    assert not orc.lib().orc_tab_new(0)


def test_rowsum_examples(orc):
    def rs(h, i):
        t = orc.Tableau(2)
        x, z, r = t.get()
        for row, text in ((0, h), (1, i)):
            _, px, pz, ps = orc.pauli_from_text(text); x[row], z[row], r[row] = px, pz, ps
        t.set(x, z, r); assert t.rowsum(0, 1) == 0
        return t.texts()[0]
    assert rs("+ZZ", "+ZZ") == "+II"
    assert rs("+YY", "+XX") == "-ZZ"
    assert rs("-XI", "+IZ") == "-XZ"


def test_measure_examples(orc):
    t = orc.Tableau(1); o, d, rc = t.sim([(M, 0)], seed=1)
    assert (o[0], d[0], rc) == (0, 1, 0)
    for seed in range(6):
        t = orc.Tableau(1); o, d, _ = t.sim([(H, 0), (M, 0)], seed)
        assert d[0] == 0 and o[0] == orc.lib().orc_counter_bit(seed, 0)
        assert t.texts()[0] == ("-Z" if o[0] else "+Z")
        t = orc.Tableau(2); o, d, _ = t.sim([(H, 0), (CX, 0, 1), (M, 0), (M, 1)], seed)   # Bell
        assert list(d) == [0, 1] and o[0] == o[1]
        o2, d2, _ = t.sim([(M, 0)], seed, ordinal0=2)                                       # idempotence SPEC:202
        assert d2[0] == 1 and o2[0] == o[0]
    assert orc.Tableau(1).sim([(T, 0)], 0)[2] == 2


def test_gate_inverse_restores(orc):
    rng = np.random.default_rng(3)
    n = 9
    t = orc.Tableau(n)
    gates = []
    for _ in range(150):
        k = int(rng.choice([H, S, SDG, X, Y, Z, CX, CZ, SWAP])); a = int(rng.integers(0, n)); b = int(rng.integers(0, n - 1)); b += b >= a
        gates.append((k, a, b))
    t.sim(gates, 0)
    inv = {H: [H], S: [SDG], SDG: [S], X: [X], Y: [Y], Z: [Z], CX: [CX], CZ: [CZ], SWAP: [SWAP]}
    t.sim([(ik, a, b) for (k, a, b) in reversed(gates) for ik in inv[k]], 0)
    assert t.texts() == orc.Tableau(n).texts()


def test_schedule_determinism(orc, sk):             # SPEC:341, acceptance #3: workers in {1,2,4,8}
    c = sk.random_layered_circuit(64, 5)
    ref = None
    for w in (1, 2, 4, 8):
        t = orc.Tableau(c.n); o, d, rc = t.sim(c.gates, 11, workers=w)
        cur = (t.texts(), list(o), list(d))
        ref = ref or cur
        assert cur == ref and rc == 0


def test_surface_code_behaviour(orc, sk):           # SPEC:396, acceptance #5
    for d in (3, 5):
        rounds = 3
        c = sk.surface_code_circuit(d, rounds)
        assert c.n == 2 * d * d - 1 and c.num_measurements == rounds * (d * d - 1)
        t = orc.Tableau(c.n); o, det, rc = t.sim(c.gates, 20250703)
        assert rc == 0
        na = d * d - 1
        # which ancillas are X checks: they get an H
        xanc = set(int(g["q0"]) for g in c.gates if g["kind"] == H)
        mq = [int(g["q0"]) for g in c.gates if g["kind"] == M]
        for r in range(rounds):
            for k in range(na):
                q, i = mq[r * na + k], r * na + k
                if q in xanc:
                    assert det[i] == (0 if r == 0 else 1)
                    # no reset gate: the ancilla keeps its last outcome, so the check value
                    # "relative to the prior outcome" o[r]^o[r-1] repeats the round-1 value
                    if r: assert (o[i] ^ o[i - na]) == o[k]
                else:
                    assert det[i] == 1 and o[i] == 0


def test_grouping_examples(orc):
    r = orc.Rows.from_text(["ZZ", "XX", "ZI"])      # already sorted by |coeff|: 1.0, 0.9, 0.5
    g, ng, _ = r.group_first_fit(0); assert list(g) == [0, 0, 1] and ng == 2          # GC
    g, ng, _ = r.group_first_fit(1); assert list(g) == [0, 1, 0] and ng == 2          # QWC
    assert orc.Rows.from_text(["ZI", "XX"]).verify_grouping(0, [0, 0]) == 1
    rng = np.random.default_rng(5)
    for _ in range(10):
        n, m = 10, 120
        W = 1
        x = rng.integers(0, 1 << n, (m, W), dtype=np.uint64); z = rng.integers(0, 1 << n, (m, W), dtype=np.uint64)
        r = orc.Rows(n, x, z, np.zeros(m, np.uint8))
        ggc, ngc, _ = r.group_first_fit(0); gq, nq, _ = r.group_first_fit(1)
        assert r.verify_grouping(0, ggc) == 0 and r.verify_grouping(1, gq) == 0 and ngc <= nq


def test_transpiler_examples(orc):                  # SPEC:521-523, 531-533, 541-543, 551-553, acceptance #9
    p = orc.Pbc(1, [(T, 0), (H, 0)])                # time order [t 0, h 0]
    assert p.stats()["initial_t"] == 1 and orc.pauli_to_text(1, *[a[0] for a in p.layer(0)]) == "+Z"
    assert p.mtab().texts()[0] == "+X"
    p = orc.Pbc(1, [(H, 0), (T, 0)])
    assert orc.pauli_to_text(1, *[a[0] for a in p.layer(0)]) == "+X" and p.mtab().texts()[0] == "+X"
    p = orc.Pbc(2, [(H, 0), (CX, 0, 1), (M, 0), (M, 1)])                             # Bell prep
    assert p.stats()["layers"] == 0 and p.status == 0
    p = orc.Pbc(1, [(T, 0), (T, 0)])                                                  # T.T = S absorbed
    s = p.stats(); assert (s["initial_t"], s["final_rotations_rowcount"], s["layers"]) == (2, 0, 0)
    assert p.mtab().texts() == ["+Z", "-Y"]          # stabilizer unchanged; destabilizer X -> (i Z X) = -Y (pauli.cpp:239-254)
    p = orc.Pbc(1, [(T, 0)] * 8)                                                      # T^8 = I
    assert p.stats()["layers"] == 0 and p.mtab().texts() == ["+Z", "+X"]
    p = orc.Pbc(1, [(T, 0), (TDG, 0)])
    assert p.stats()["layers"] == 0 and p.mtab().texts() == ["+Z", "+X"]
    p = orc.Pbc(1, [(H, 0), (T, 0), (H, 0), (M, 0)])
    assert p.stats()["layers"] == 1 and orc.pauli_to_text(1, *[a[0] for a in p.layer(0)]) == "+X"
    assert orc.Pbc(2, [(M, 0), (H, 0)]).status == 2                                   # mid-circuit M
    # t_separate examples SPEC:531-533 through the staged entry point
    import ctypes as C
    L = orc.lib()
    def sep(gates, n):
        g = orc.gates_array(gates); st = C.c_int(); m = orc.Tableau(n)
        tt = L.orc_build_ttab(n, orc._p(g), len(g), m.h, C.byref(st))
        k = L.orc_rows_count(tt); ids = np.zeros(max(k, 1), np.uint32)
        nl = L.orc_t_separate_ids(tt, orc._p(ids)); L.orc_rows_free(tt)
        return list(ids[:k]), nl
    assert sep([(T, 0), (T, 0)], 1) == ([0, 0], 1)
    assert sep([(T, 0), (H, 0), (T, 0)], 1)[1] == 2
    ids, nl = sep([(T, 0), (T, 1), (H, 0), (T, 0), (H, 0)], 2)   # rows (append order): X0?  check layer count only
    assert nl == 2


def test_transpiler_properties(orc, sk):
    rng = np.random.default_rng(11)
    reduced = 0
    for trial in range(60):
        n = int(rng.integers(2, 7)); G = int(rng.integers(10, 60))
        gates = []
        for _ in range(G):
            u = rng.random()
            a = int(rng.integers(0, n)); b = int(rng.integers(0, n - 1)); b += b >= a
            if u < 0.15: gates.append((T, a))
            elif u < 0.30: gates.append((TDG, a))
            elif u < 0.55: gates.append((H, a))
            elif u < 0.75: gates.append((S, a))
            else: gates.append((CX, a, b))
        p = orc.Pbc(n, gates); assert p.status == 0
        s = p.stats()
        assert s["final_rotations_rowcount"] <= s["initial_t"]
        reduced += s["final_rotations_rowcount"] < s["initial_t"]
        for k in range(s["layers"]):                 # layer commutativity SPEC:577
            x, z, r = p.layer(k); L = orc.lib()
            for a in range(len(r)):
                for b in range(a + 1, len(r)):
                    assert L.orc_commutes(orc._p(x[a]), orc._p(z[a]), orc._p(x[b]), orc._p(z[b]), x.shape[1])
                    assert not ((x[a] == x[b]).all() and (z[a] == z[b]).all())   # converged: no duplicates left
    assert reduced >= 12
