"""-m gpu: grouping and Clifford+T kernels (through the C ABI) against the CPU oracle, bit-exact."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
H, S, SDG, X, Y, Z, CX, CZ, SWAP, M, T, TDG = range(12)


def rand_rows(rng, n, m, density=0.5):
    W = (n + 63) // 64
    x = np.zeros((m, W), np.uint64); z = np.zeros((m, W), np.uint64)
    bx = rng.random((m, n)) < density; bz = rng.random((m, n)) < density
    for w in range(W):
        for b in range(min(64, n - 64 * w)):
            x[:, w] |= (bx[:, 64 * w + b].astype(np.uint64) << np.uint64(b))
            z[:, w] |= (bz[:, 64 * w + b].astype(np.uint64) << np.uint64(b))
    return x, z, rng.integers(0, 2, m).astype(np.uint8)


@pytest.mark.parametrize("n,m", [(1, 3), (2, 5), (17, 40), (64, 100), (130, 257), (1000, 600)])
def test_row_primitives(sk, ctx, orc, n, m):
    rng = np.random.default_rng(n * 7 + m)
    x, z, s = rand_rows(rng, n, m, 0.3)
    d = sk.Rows(ctx, n, x, z, s); o = orc.Rows(n, x, z, s)
    assert d.weight_sum() == o.weight_sum()                                   # pauli.cpp:100-106
    for _ in range(3):                                                        # pauli.cpp:215-237
        px, pz, _ = rand_rows(rng, n, 1, 0.4)
        assert (d.commutation_vector(px[0], pz[0]) == o.commutation_vector(px[0], pz[0])).all()
    # plant duplicates, then compare the first pair in scan order
    assert d.find_first_duplicate() == o.first_duplicate()
    if m >= 5:
        x[m - 1] = x[1]; z[m - 1] = z[1]; x[m - 2] = x[0]; z[m - 2] = z[0]; x[3] = x[1]; z[3] = z[1]
        d.upload(x, z, s); o = orc.Rows(n, x, z, s)
        assert d.find_first_duplicate() == o.first_duplicate()
        if n >= 64: assert o.first_duplicate() == (0, m - 2)
    # conj_* on every row (pauli.cpp:146-187)
    gates = []
    for _ in range(60):
        k = int(rng.choice([H, S, SDG, X, Y, Z, CX, CZ, SWAP])); a = int(rng.integers(0, n)); b = 0
        if k in (CX, CZ, SWAP):
            if n == 1: k = H
            else: b = int(rng.integers(0, n - 1)); b += b >= a
        gates.append((k, a, b))
    d.conj_layer(gates); o.apply(gates)
    dx, dz, ds = d.download(); ox, oz, os_ = o.get()
    assert (dx == ox).all() and (dz == oz).all() and (ds == os_).all()
    # rowsum_plus_i on all anticommuting rows (pauli.cpp:239-254)
    px, pz, ps = rand_rows(rng, n, 1, 0.4)
    anti = o.commutation_vector(px[0], pz[0])
    cnt = 0
    for i in range(m):
        if (int(anti[i >> 6]) >> (i & 63)) & 1:
            assert o.rowsum_plus_i(i, px[0], pz[0], ps[0]) == 0; cnt += 1
    assert d.rowsum_plus_i_where_anticommuting(px[0], pz[0], int(ps[0])) == cnt
    dx, dz, ds = d.download(); ox, oz, os_ = o.get()
    assert (dx == ox).all() and (dz == oz).all() and (ds == os_).all()


def test_grouping_examples(sk, ctx, orc):
    n, x, z, s = 2, [], [], []
    for t in ("ZZ", "XX", "ZI"):
        _, px, pz, _ = orc.pauli_from_text(t); x.append(px); z.append(pz)
    d = sk.Rows(ctx, 2, np.stack(x), np.stack(z))
    g, ng = d.group_first_fit(0); assert list(g) == [0, 0, 1] and ng == 2
    g, ng = d.group_first_fit(1); assert list(g) == [0, 1, 0] and ng == 2
    assert d.verify_grouping(0, [0, 0, 1]) == 0 and d.verify_grouping(0, [0, 1, 1]) == 1   # {XX, ZI} anticommute
    one = sk.Rows(ctx, 2, np.stack(x[:1]), np.stack(z[:1])); g, ng = one.group_first_fit(0); assert list(g) == [0] and ng == 1


@pytest.mark.parametrize("n,m,density", [(16, 500, 0.5), (10, 3000, 0.3), (128, 2500, 0.5), (128, 5000, 0.05), (300, 1500, 0.02),
                                         (64, 9000, 0.5), (100, 7000, 0.01), (5, 4100, 0.5)])
def test_grouping_matches_oracle(sk, ctx, orc, n, m, density):
    rng = np.random.default_rng(m + n)
    x, z, s = rand_rows(rng, n, m, density)
    d = sk.Rows(ctx, n, x, z); o = orc.Rows(n, x, z, np.zeros(m, np.uint8))
    counts = {}
    for mode in (0, 1):
        g, ng = d.group_first_fit(mode)
        og, ong, _ = o.group_first_fit(mode)
        assert ng == ong and (g == og).all()
        assert d.verify_grouping(mode, g) == 0 == o.verify_grouping(mode, og)
        counts[mode] = ng
    if density >= 0.05:                        # first fit is a heuristic: on very sparse strings GC may need one group more than QWC
        assert counts[0] <= counts[1]
    bad = np.zeros(m, np.uint32)                                              # everything in one group
    assert d.verify_grouping(0, bad) == o.verify_grouping(0, bad) > 0


def rand_ct(rng, n, G, pt=0.1):
    gates = []
    for _ in range(G):
        u = rng.random(); a = int(rng.integers(0, n)); b = 0
        if n > 1: b = int(rng.integers(0, n - 1)); b += b >= a
        if u < pt / 2: gates.append((T, a, 0))
        elif u < pt: gates.append((TDG, a, 0))
        elif u < pt + 0.3: gates.append((H, a, 0))
        elif u < pt + 0.6 or n == 1: gates.append((S, a, 0))
        else: gates.append((CX, a, b))
    return gates


def assert_same_pbc(d, o):
    ds, os_ = d.stats(), o.stats()
    assert ds == os_, (ds, os_)
    for k in range(ds["layers"]):
        dx, dz, dsg = d.layer(k); ox, oz, osg = o.layer(k)
        assert dx.shape == ox.shape and (dx == ox).all() and (dz == oz).all() and (dsg == osg).all(), f"layer {k}"
    mx, mz, ms = d.mtab(); ox, oz, osg = o.mtab().get()
    assert (mx == ox).all() and (mz == oz).all() and (ms == osg).all()


def test_transpile_examples(sk, ctx, orc):
    for n, gates in ((1, [(T, 0, 0), (H, 0, 0)]), (1, [(H, 0, 0), (T, 0, 0)]), (2, [(H, 0, 0), (CX, 0, 1), (M, 0, 0), (M, 1, 0)]),
                     (1, [(T, 0, 0)] * 2), (1, [(T, 0, 0)] * 8), (1, [(T, 0, 0), (TDG, 0, 0)]), (1, [(H, 0, 0), (T, 0, 0), (H, 0, 0), (M, 0, 0)]),
                     (3, [(H, 1, 0), (CX, 1, 2)])):
        assert_same_pbc(sk.Pbc(ctx, sk.Circuit(n, gates)), orc.Pbc(n, gates, exact=True))          # default = unitary-exact form
        assert_same_pbc(sk.Pbc(ctx, sk.Circuit(n, gates), exact=False), orc.Pbc(n, gates))         # SK_TRANSPILE_PUBLISHED
    with pytest.raises(sk.UnsupportedError):
        sk.Pbc(ctx, sk.Circuit(2, [(M, 0, 0), (H, 0, 0)]))


def test_transpile_random_small(sk, ctx, orc):                                # SPEC:576-580 (acceptance #8 sizes)
    rng = np.random.default_rng(8)
    for trial in range(120):
        n = int(rng.integers(1, 7)); gates = rand_ct(rng, n, int(rng.integers(5, 60)), pt=float(rng.uniform(0.1, 0.5)))
        assert_same_pbc(sk.Pbc(ctx, sk.Circuit(n, gates)), orc.Pbc(n, gates, exact=True))
        assert_same_pbc(sk.Pbc(ctx, sk.Circuit(n, gates), exact=False), orc.Pbc(n, gates))


@pytest.mark.parametrize("n,G,pt", [(20, 2000, 0.2), (100, 4000, 0.1), (1000, 6000, 0.1), (70, 6000, 0.4)])
def test_transpile_random_large(sk, ctx, orc, n, G, pt):                      # BASELINE config 5 shape
    rng = np.random.default_rng(n + G)
    gates = rand_ct(rng, n, G, pt)
    assert_same_pbc(sk.Pbc(ctx, sk.Circuit(n, gates)), orc.Pbc(n, gates, exact=True))
    assert_same_pbc(sk.Pbc(ctx, sk.Circuit(n, gates), exact=False), orc.Pbc(n, gates))


def test_transpile_default_matches_oracle_and_the_statevector(sk, ctx, orc):
    """The DEFAULT transpile path (sk_transpile, flags 0; circuits with S / S-dagger gates included): bit parity with the
    oracle's exact variant, and -- independently of any tableau convention -- the dense-statevector equivalence check of
    SPEC:563-573 on the DEVICE output (TV < 1e-9)."""
    from oracle import dense as dn
    rng = np.random.default_rng(77)
    for trial in range(80):
        n = int(rng.integers(1, 6)); gates = rand_ct(rng, n, int(rng.integers(5, 60)), pt=float(rng.uniform(0.1, 0.5)))
        d = sk.Pbc(ctx, sk.Circuit(n, gates))
        assert_same_pbc(d, orc.Pbc(n, gates, exact=True))
        st = d.stats()
        layers = [[(int(x[i, 0]), int(z[i, 0]), int(r[i])) for i in range(len(r))] for x, z, r in (d.layer(k) for k in range(st["layers"]))]
        mx, mz, mr = d.mtab()
        rows = [(int(mx[i, 0]), int(mz[i, 0]), int(mr[i])) for i in range(n)]
        assert dn.verify_transpile(n, [g for g in gates if g[0] != M], layers, rows) < 1e-9
    for n, G, pt in ((20, 2000, 0.2), (100, 4000, 0.1), (70, 3000, 0.4)):
        gates = rand_ct(np.random.default_rng(n + G + 1), n, G, pt)
        assert_same_pbc(sk.Pbc(ctx, sk.Circuit(n, gates)), orc.Pbc(n, gates, exact=True))


# ---- BASELINE configs C4 / C5 at their stated size (SURVEY 8d generators: paper_2507_03092_b200/workloads.py) -----------------
def test_c4_grouping_1e5_matches_oracle(sk, ctx, orc):
    """Config C4 at N = 10^5 (the largest size the CPU oracle finishes in seconds): identical group ids, GC and QWC."""
    from paper_2507_03092_b200 import workloads as wl
    N = 100_000
    x, z, _ = wl.c4_terms(N)
    d = sk.Rows(ctx, 128, x, z); o = orc.Rows(128, x, z, np.zeros(N, np.uint8))
    for mode in (0, 1):
        g, ng = d.group_first_fit(mode)
        og, ong, _ = o.group_first_fit(mode)
        assert ng == ong and (g == og).all(), f"mode {mode}"
        assert d.verify_grouping(mode, g) == 0
    d.close()


def test_c4_grouping_1e6_matches_golden(sk, ctx):
    """Config C4 at its full size N = 10^6: the device's group ids against the checksum the CPU oracle produced once
    (tools/make_c4_golden.py -> tests/golden/c4_groups_1000000.json; ~10-20 minutes of CPU per mode)."""
    import hashlib, json, os
    from paper_2507_03092_b200 import workloads as wl
    path = os.path.join(os.path.dirname(__file__), "golden", "c4_groups_1000000.json")
    if not os.path.exists(path): pytest.skip("golden file not generated")
    gold = json.load(open(path))
    N = gold["N"]
    x, z, _ = wl.c4_terms(N, gold["seed"])
    d = sk.Rows(ctx, 128, x, z)
    for mode, name in ((0, "GC"), (1, "QWC")):
        g, ng = d.group_first_fit(mode)
        g = np.ascontiguousarray(g, np.uint32)
        assert ng == gold["modes"][name]["groups"], name
        assert g[:16].tolist() == gold["modes"][name]["first16"] and g[-4:].tolist() == gold["modes"][name]["last4"], name
        assert hashlib.sha256(g.tobytes()).hexdigest() == gold["modes"][name]["sha256"], name
    d.close()


def test_c5_transpile_1e5_matches_oracle(sk, ctx, orc):
    """Config C5 at its full size: n = 1000, G = 10^5 gates, 10 % T: identical T layers, M_tab and statistics (exact form,
    the default) and the published form of Algorithms 2-3."""
    from paper_2507_03092_b200 import workloads as wl
    gates = wl.c5_gates(1000, 100_000, gate_dtype=sk.GATE_DTYPE, kinds=(sk.H, sk.S, sk.CX, sk.T, sk.TDG))
    circ = sk.Circuit(1000, gates)
    assert abs(int(((gates["kind"] == sk.T) | (gates["kind"] == sk.TDG)).sum()) - 10_000) < 400
    for exact in (True, False):
        d = sk.Pbc(ctx, circ, exact=exact); o = orc.Pbc(1000, circ.gates, exact=exact)
        assert_same_pbc(d, o)
        d.close()


def test_rows_append_and_commute_tile(sk, ctx, orc):
    """sk_rows_append (T_tab grows row by row) and sk_commute_matrix_tile (pauli.cpp:117-140 over a tile of the pair
    matrix) against the oracle's scalar predicates; appending beyond the capacity is SK_EDIM."""
    rng = np.random.default_rng(8)
    for n, m in ((5, 40), (130, 300), (128, 700)):
        x, z, s = rand_rows(rng, n, m, 0.3)
        d = sk.Rows(ctx, n, x[:m // 3], z[:m // 3], s[:m // 3], capacity=m)
        d.append(x[m // 3:m - 7], z[m // 3:m - 7], s[m // 3:m - 7]); d.append(x[m - 7:], z[m - 7:], s[m - 7:])
        assert d.count == m
        dx, dz, ds = d.download()
        assert (dx == x).all() and (dz == z).all() and (ds == s).all()
        with pytest.raises(sk.DimensionError): d.append(x[:1], z[:1], s[:1])
        W = x.shape[1]
        for mode in (0, 1):
            i0, ni, j0, nj = 3, min(37, m - 3), m // 4, m - m // 4
            t = d.commute_tile(mode, i0, ni, j0, nj)
            f = orc.lib().orc_commutes if mode == 0 else orc.lib().orc_qw_commutes
            for a in (0, 5, ni - 1):
                for b in (0, 1, 63, 64, 65, nj - 1):
                    if b >= nj: continue
                    ok = f(orc._p(x[i0 + a]), orc._p(z[i0 + a]), orc._p(x[j0 + b]), orc._p(z[j0 + b]), W)
                    assert bool(t[a, b]) == (not ok), (n, mode, a, b)
            # the whole tile through numpy: anticommutation parity / any overlap
            v = (x[i0:i0 + ni, None, :] & z[None, j0:j0 + nj, :]) ^ (x[None, j0:j0 + nj, :] & z[i0:i0 + ni, None, :])
            if mode == 0:
                par = np.zeros((ni, nj), np.uint64)
                for w in range(W):
                    u = v[:, :, w].copy()
                    for sh in (32, 16, 8, 4, 2, 1): u ^= u >> np.uint64(sh)
                    par ^= u & np.uint64(1)
                assert (t == (par == 1)).all()
            else:
                assert (t == (v != 0).any(axis=2)).all()
        d.close()


def test_tableau_audit_counts_violations(sk, ctx):
    """sk_tableau_audit (EngineConfig.audit): 0 for tableaux the engine produced, the exact number of broken
    row pairs after rows are tampered with."""
    for circ in (sk.surface_code_circuit(7, 3, True), sk.random_layered_circuit(200, 4)):
        t, _, _, _ = ctx.sim(circ, 5)
        assert t.audit() == 0
        x, z, r = t.download()
        n = circ.n
        x[0], z[0] = x[n].copy(), z[n].copy()            # stabilizer 0 := destabilizer 0: row 0 now commutes with its partner (1 pair broken),
        t.upload(x, z, r)                                 # and anticommutes with whatever destabilizer 0 anticommuted with
        bad = t.audit()
        # expected count from the symplectic form on the host
        def sym(a, b): return int(np.bitwise_xor.reduce([bin(int(v)).count("1") & 1 for v in ((x[a] & z[b]) ^ (x[b] & z[a]))]))
        exp = 0
        for b in range(1, 2 * n): exp += sym(0, b) != (1 if b == n else 0)
        assert bad == exp and bad >= 1
        t.close()
    c = ctx.counters()
    assert c["algorithmic_bytes"] > 0 and len(c["class_ms"]) == 4 and c["pred_evals"] >= 0
