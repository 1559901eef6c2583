"""-m gpu: bit-exact parity of the CUDA tableau path (through the C ABI) against the CPU oracle."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

H, S, SDG, X, Y, Z, CX, CZ, SWAP, M, T, TDG = range(12)
SEED = 20250703


def rand_gates(rng, n, count, kinds=(H, S, SDG, X, Y, Z, CX, CZ, SWAP), pm=0.0):
    out = []
    for _ in range(count):
        if pm and rng.random() < pm:
            out.append((M, int(rng.integers(0, n)), 0)); continue
        k = int(rng.choice(kinds))
        a = int(rng.integers(0, n)); b = 0
        if k in (CX, CZ, SWAP):
            if n == 1: k = H
            else: b = int(rng.integers(0, n - 1)); b += b >= a
        out.append((k, a, b))
    return out


def assert_same_tableau(t_dev, t_orc):
    x, z, r = t_dev.download()
    ox, oz, orr = t_orc.get()
    assert (x == ox).all(), "x bits differ"
    assert (z == oz).all(), "z bits differ"
    assert (r == orr).all(), "signs differ"


@pytest.mark.parametrize("n", [1, 2, 5, 17, 63, 64, 65, 130, 257, 1249])
def test_gate_sequences_match_oracle(sk, ctx, orc, n):
    rng = np.random.default_rng(n)
    gates = rand_gates(rng, n, 40 + 6 * n if n < 200 else 3000)
    t = sk.Tableau(ctx, n); t.apply_gates(gates)
    o = orc.Tableau(n); assert o.sim(gates, 0)[2] == 0
    assert_same_tableau(t, o)
    # gate . inverse restores the identity bit-for-bit
    inv = {H: H, S: SDG, SDG: S, X: X, Y: Y, Z: Z, CX: CX, CZ: CZ, SWAP: SWAP}
    t.apply_gates([(inv[k], a, b) for k, a, b in reversed(gates)])
    assert_same_tableau(t, orc.Tableau(n))


def test_each_gate_kind_as_single_layer(sk, ctx, orc):
    n = 70
    rng = np.random.default_rng(1)
    prep = rand_gates(rng, n, 500)
    for k in (H, S, SDG, X, Y, Z, CX, CZ, SWAP):
        perm = rng.permutation(n)
        layer = [(k, int(perm[2 * i]), int(perm[2 * i + 1])) for i in range(n // 2)] if k in (CX, CZ, SWAP) \
            else [(k, int(q), 0) for q in perm[: n - 3]]
        t = sk.Tableau(ctx, n); t.apply_gates(prep); t.apply_layer(layer)
        o = orc.Tableau(n); o.sim(prep + layer, 0)
        assert_same_tableau(t, o)


def test_upload_download_roundtrip_and_rows_under_gates(sk, ctx, orc):
    rng = np.random.default_rng(2)
    for n in (3, 64, 100, 321):
        W = sk.words_for(n)
        mask = np.full(W, np.uint64(2**64 - 1)); rem = n % 64
        if rem: mask[-1] = np.uint64((1 << rem) - 1)
        x = rng.integers(0, 2**64, (2 * n, W), dtype=np.uint64) & mask
        z = rng.integers(0, 2**64, (2 * n, W), dtype=np.uint64) & mask
        r = rng.integers(0, 2, 2 * n).astype(np.uint8)
        t = sk.Tableau(ctx, n); t.upload(x, z, r)
        x2, z2, r2 = t.download()
        assert (x2 == x).all() and (z2 == z).all() and (r2 == r).all()
        gates = rand_gates(rng, n, 200)          # conj_* rules hold for ARBITRARY rows, not only valid tableaux
        t.apply_gates(gates)
        rows = orc.Rows(n, x, z, r); rows.apply(gates)
        ox, oz, orr = rows.get()
        x3, z3, r3 = t.download()
        assert (x3 == ox).all() and (z3 == oz).all() and (r3 == orr).all()


def test_error_behaviour(sk, ctx):
    t = sk.Tableau(ctx, 4)
    with pytest.raises(sk.DimensionError): t.apply_layer([(H, 4, 0)])
    with pytest.raises(sk.UnsupportedError): t.apply_layer([(T, 0, 0)])
    with pytest.raises(sk.StabkitError): t.apply_layer([(H, 0, 0), (CX, 0, 1)])  # collision in a layer
    with pytest.raises(sk.StabkitError): t.apply_gates([(CX, 1, 1)])
    with pytest.raises(sk.DimensionError): t.measure_z(9, 0, 0)
    with pytest.raises(sk.DimensionError): sk.Tableau(ctx, 0)
    with pytest.raises(sk.UnsupportedError):
        ctx.sim(sk.Circuit(2, [(H, 0, 0), (T, 1, 0)]), 0)
    with pytest.raises(sk.DimensionError): t.rowsum(0, 0)


def test_measurement_examples(sk, ctx, orc):
    t = sk.Tableau(ctx, 1)
    assert t.measure_z(0, 1, 0) == (0, 1)
    for seed in range(8):
        t = sk.Tableau(ctx, 1); t.apply_gates([(H, 0, 0)])
        o, d = t.measure_z(0, seed, 0)
        assert d == 0 and o == orc.lib().orc_counter_bit(seed, 0)
        assert t.measure_z(0, seed, 1) == (o, 1)
        t = sk.Tableau(ctx, 2); t.apply_gates([(H, 0, 0), (CX, 0, 1)])
        o0, d0 = t.measure_z(0, seed, 0); o1, d1 = t.measure_z(1, seed, 1)
        assert (d0, d1) == (0, 1) and o0 == o1


def test_rowsum_api(sk, ctx, orc):
    n = 6
    rng = np.random.default_rng(4)
    gates = rand_gates(rng, n, 80)
    t = sk.Tableau(ctx, n); t.apply_gates(gates)
    o = orc.Tableau(n); o.sim(gates, 0)
    for h, i in ((0, 1), (2, 5), (4, 0)):           # stabilizer rows commute: even phase
        t.rowsum(h, i); assert o.rowsum(h, i) == 0
    assert_same_tableau(t, o)
    t.apply_gates([(H, 0, 0)])                      # C form must have been kept consistent
    o.sim([(H, 0, 0)], 0)
    assert_same_tableau(t, o)
    with pytest.raises(sk.InvariantError):          # stabilizer x its own destabilizer: odd phase
        t.rowsum(0, n)


@pytest.mark.parametrize("n,count,pm", [(1, 30, 0.3), (2, 60, 0.3), (5, 200, 0.2), (10, 200, 0.1), (33, 600, 0.15),
                                        (64, 800, 0.1), (65, 900, 0.2), (130, 1500, 0.1), (300, 3000, 0.05)])
def test_random_circuits_with_measurements(sk, ctx, orc, n, count, pm):
    for trial in range(4):
        rng = np.random.default_rng(1000 * n + trial)
        gates = rand_gates(rng, n, count, pm=pm)
        seed = int(rng.integers(0, 2**63))
        circ = sk.Circuit(n, gates)
        t, out, det, warn = ctx.sim(circ, seed)
        o = orc.Tableau(n); oo, od, rc = o.sim(gates, seed)
        assert rc == 0
        assert (out == oo).all() and (det == od).all()
        assert_same_tableau(t, o)
        c = o.counters()
        t.close()


def test_measure_batch_equals_sequential(sk, ctx, orc):
    n = 40
    rng = np.random.default_rng(8)
    gates = rand_gates(rng, n, 400, kinds=(H, S, CX))
    qs = [int(q) for q in rng.integers(0, n, 60)]
    a = sk.Tableau(ctx, n); a.apply_gates(gates)
    b = sk.Tableau(ctx, n); b.apply_gates(gates)
    oa, da = a.measure_batch(qs, 5, ordinal0=3)
    ob = [b.measure_z(q, 5, 3 + i) for i, q in enumerate(qs)]
    assert [(int(x), int(y)) for x, y in zip(oa, da)] == ob
    xa, za, ra = a.download(); xb, zb, rb = b.download()
    assert (xa == xb).all() and (za == zb).all() and (ra == rb).all()
    o = orc.Tableau(n); o.sim(gates, 0)
    oo, od, _ = o.sim([(M, q, 0) for q in qs], 5, ordinal0=3)
    assert (oa == oo).all() and (da == od).all()
    assert_same_tableau(a, o)


def test_counters_match_oracle(sk, ctx, orc):
    c = sk.random_layered_circuit(128, 77)
    ctx.reset_counters()
    t, out, det, _ = ctx.sim(c, 9)
    o = orc.Tableau(c.n); oo, od, _ = o.sim(c.gates, 9)
    assert (out == oo).all() and (det == od).all()
    dc, oc = ctx.counters(), o.counters()
    for k in ("n_rand", "n_det", "k_rand", "k_det"):
        assert dc[k] == oc[k], k
    assert dc["gate_hist"] == oc["gate_hist"]


@pytest.mark.parametrize("d,rounds", [(3, 3), (5, 5), (7, 3), (25, 25)])
def test_surface_code_parity(sk, ctx, orc, d, rounds):      # BASELINE configs 1 and 2
    c = sk.surface_code_circuit(d, rounds, final_data_measure=True)
    t, out, det, _ = ctx.sim(c, SEED)
    o = orc.Tableau(c.n); oo, od, rc = o.sim(c.gates, SEED, workers=8)
    assert rc == 0 and (out == oo).all() and (det == od).all()
    assert_same_tableau(t, o)
    t2, out2, det2, warn = ctx.sim(c, SEED, mode=1)          # sim2d == sim
    assert warn == 0 and (out2 == out).all() and (det2 == det).all()
    x, z, r = t.download(); x2, z2, r2 = t2.download()
    assert (x == x2).all() and (z == z2).all() and (r == r2).all()


def test_sim2d_fallback_warning(sk, ctx, orc):
    c = sk.parse_native("qubits 3\nh 0\nh 1\nh 2\nchunk\nh 0\ncx 0 1\nchunk\nm 0\nm 1\nm 2\n")
    t, out, det, warn = ctx.sim(c, 3, mode=1)
    assert warn == 1
    o = orc.Tableau(3); oo, od, _ = o.sim(c.gates, 3)
    assert (out == oo).all() and (det == od).all()
    assert_same_tableau(t, o)


def test_random_layered_parity_and_sim2d(sk, ctx, orc):      # SPEC:328; SURVEY 8f item 1
    for n in (8, 64, 256, 1024):
        c = sk.random_layered_circuit(n, 123 + n)
        t, out, det, _ = ctx.sim(c, 42)
        t2, out2, det2, warn = ctx.sim(c, 42, mode=1)
        o = orc.Tableau(n); oo, od, _ = o.sim(c.gates, 42, workers=8)
        assert warn == 0
        assert (out == oo).all() and (det == od).all() and (out2 == oo).all() and (det2 == od).all()
        assert_same_tableau(t, o); assert_same_tableau(t2, o)


def test_surface_code_d71_oracle_rounds_and_full_properties(sk, ctx, orc):   # BASELINE config 3
    d = 71
    # (a) oracle parity at full width on the first 2 rounds (the oracle needs minutes for all 71)
    c2 = sk.surface_code_circuit(d, 2)
    t, out, det, _ = ctx.sim(c2, SEED)
    o = orc.Tableau(c2.n); oo, od, _ = o.sim(c2.gates, SEED, workers=8)
    assert (out == oo).all() and (det == od).all()
    assert_same_tableau(t, o)
    # (b) full size: size-independent properties (acceptance #5)
    c = sk.surface_code_circuit(d, d, final_data_measure=True)
    ctx.reset_counters()
    t, out, det, _ = ctx.sim(c, SEED)
    na = d * d - 1
    xanc = np.zeros(c.n, bool); xanc[c.gates["q0"][c.gates["kind"] == H]] = True
    mq = c.gates["q0"][c.gates["kind"] == M]
    isx = xanc[mq[:na]]
    o_r = out[: na * d].reshape(d, na); d_r = det[: na * d].reshape(d, na)
    assert (d_r[0, isx] == 0).all() and (d_r[1:, isx] == 1).all() and (d_r[:, ~isx] == 1).all()
    assert (o_r[:, ~isx] == 0).all()
    rel = o_r[1:, isx] ^ o_r[:-1, isx]
    assert (rel == o_r[0, isx][None, :]).all()
    assert (o_r[0, isx] == np.array([orc.lib().orc_counter_bit(SEED, int(i)) for i in np.nonzero(isx)[0]], np.uint8)).all()
    # final data-qubit Z measurements: every Z plaquette has even parity (all Z checks gave 0)
    data = out[na * d:]
    assert len(data) == d * d
    for g0 in range(0, 0):
        pass
    zpar = {}
    for g in c2.gates[c2.gates["kind"] == CX]:
        a, b = int(g["q0"]), int(g["q1"])
        if b >= d * d and a < d * d and not xanc[b]:
            zpar.setdefault(b, set()).add(a)
    assert len(zpar) == (d * d - 1) // 2
    for anc, qs in zpar.items():
        assert sum(int(data[q]) for q in qs) % 2 == 0
    cnt = ctx.counters()
    assert cnt["n_rand"] + cnt["n_det"] == len(out)
    # idempotence at scale: measuring every qubit again is deterministic and repeats
    again, adet = t.measure_batch(np.arange(d * d, dtype=np.uint32), SEED, ordinal0=len(out))
    assert (adet == 1).all() and (again == data).all()


def test_surface_code_d71_full_length_bit_parity(sk, ctx, orc):           # BASELINE config 3 at its stated size
    """The headline workload, all 71 rounds + the final data-qubit M: the whole measurement record (362 881 outcome and
    deterministic bytes), every x/z word and every sign of the final tableau equal the oracle's (SPEC:730 bit-exact
    schedule determinism).  The circuit comes from the ORACLE's own generator, which must equal the product's
    gate for gate.  One oracle run of the full circuit costs ~25 s on the box's 16 host threads."""
    d = 71
    n, gates, marks = orc.surface_code(d, d, True)
    c = sk.surface_code_circuit(d, d, final_data_measure=True)
    assert n == c.n and (gates == c.gates).all() and (marks == c.chunk_marks).all()
    o = orc.Tableau(n)
    oo, od, rc = o.sim(gates, SEED, workers=os.cpu_count() or 8)
    assert rc == 0 and len(oo) == 362881
    for mode in (0, 1):                                                    # sim and sim2d
        t, out, det, warn = ctx.sim(c, SEED, mode=mode)
        assert warn == 0
        assert (out == oo).all(), "outcome bytes differ at d=71 x 71"
        assert (det == od).all(), "deterministic flags differ at d=71 x 71"
        assert_same_tableau(t, o)
        t.close()
    # the resident-program path bench.py times (sk_program_run on a reset tableau) gives the same record and tableau
    prog = sk.Program(ctx, c, mode=0); tab = sk.Tableau(ctx, n)
    for _ in range(2):                                                     # second run = CUDA-graph replay
        tab.reset(); prog.run(tab, SEED)
        o2, d2 = prog.read_record()
        assert (o2 == oo).all() and (d2 == od).all()
        assert_same_tableau(tab, o)
    prog.close(); tab.close()


@pytest.mark.parametrize("n", [4480, 4416])
def test_long_measurement_blocks_off_the_surface_code(sk, ctx, orc, n):
    """The kernels that only run at size -- k_wave_cols / k_wave_rows for blocks of >= 2 048 measurements, k_transpose_wave and the
    register-block transposition when the word count is even (n = 4 480), the shuffle transposition + a separate k_wave_cols when it
    is odd (4 416) -- on circuits that are not surface codes: blocks that are mixed, all deterministic (the wave kernels own them)
    and random again, Clifford layers in between; through sk_sim and through the replayed program."""
    rng = np.random.default_rng(n)
    g = []
    def layer(kinds, frac):
        qs = rng.permutation(n); k = 0
        while k + 1 < int(frac * n):
            kind = int(rng.choice(kinds))
            if kind in (CX, CZ, SWAP): g.append((kind, int(qs[k]), int(qs[k + 1]))); k += 2
            else: g.append((kind, int(qs[k]), 0)); k += 1
    for _ in range(2): layer((H, S, X), 0.5); layer((CX, CZ), 0.8); layer((H, SDG, Y), 0.3); layer((CX, SWAP), 0.6)
    g += [(M, q, 0) for q in range(n)]
    g += [(M, int(q), 0) for q in rng.permutation(n)[:3000]]
    layer((H, H, S), 0.4); layer((CX, CZ), 0.9)
    g += [(M, int(q), 0) for q in rng.permutation(n)[:2500]]
    layer((CX,), 0.7)
    g += [(M, q, 0) for q in range(n - 1, -1, -1)]
    circ = sk.Circuit(n, g)
    t, out, det, _ = ctx.sim(circ, SEED)
    o = orc.Tableau(n); oo, od, rc = o.sim(circ.gates, SEED, workers=8)
    assert rc == 0 and (out == oo).all() and (det == od).all()
    assert (od == 0).sum() > 1000 and (od == 1).sum() > 5000
    assert_same_tableau(t, o)
    prog = sk.Program(ctx, circ); t2 = sk.Tableau(ctx, n)
    for _ in range(2):                                   # second run: graph replay
        t2.reset(); prog.run(t2, SEED); ctx.sync()
        o2, d2 = prog.read_record()
        assert (o2 == oo).all() and (d2 == od).all()
        assert_same_tableau(t2, o)
    t.close(); t2.close()


@pytest.mark.parametrize("fuse", ["1", "0"])
def test_h_window_rewriting(sk, orc, fuse):
    """The program compiler drops  H a ; CX a->d ... ; H a  windows in favour of the internal XCX gate (sk_api.cu
    fuse_h_windows; SK_FUSE_H=0 keeps the program as written).  Programs made of such windows -- closed, interrupted by other
    gates on the window qubit, by the qubit becoming a target, nested on both qubits of a CX, cut by a measurement -- leave the
    tableau and the record of the oracle."""
    os.environ["SK_FUSE_H"] = fuse
    try:
        ctx = sk.Context(0)
    finally:
        del os.environ["SK_FUSE_H"]
    rng = np.random.default_rng(41)
    fixed = [
        (3, [(H, 0, 0), (CX, 0, 1), (CX, 0, 2), (H, 0, 0)]),
        (3, [(X, 0, 0), (H, 0, 0), (H, 1, 0), (CX, 0, 1), (H, 0, 0), (H, 1, 0)]),              # windows on both qubits of one CX
        (3, [(S, 0, 0), (H, 0, 0), (CX, 0, 1), (S, 0, 0), (CX, 0, 2), (H, 0, 0)]),             # interrupted by S
        (3, [(H, 1, 0), (H, 0, 0), (CX, 0, 1), (CX, 2, 0), (H, 0, 0), (CX, 0, 2), (H, 0, 0)]),   # became a target, reopened
        (2, [(H, 0, 0), (H, 0, 0), (S, 1, 0), (H, 1, 0), (CX, 1, 0), (M, 1, 0), (H, 1, 0), (M, 0, 0), (M, 1, 0)]),
        (4, [(H, 0, 0), (S, 1, 0), (H, 1, 0), (CX, 0, 2), (Y, 2, 0), (CZ, 2, 3), (CX, 0, 3), (H, 0, 0), (CX, 1, 3), (H, 1, 0), (M, 0, 0), (M, 3, 0), (M, 1, 0)]),
    ]
    cases = [(n, g) for n, g in fixed]
    for n in (2, 3, 6, 20, 70):
        for pm in (0.0, 0.05):
            cases.append((n, [(S, q, 0) for q in range(0, n, 2)] + rand_gates(rng, n, 60 * n, kinds=(H, H, H, CX, CX, CX, CX, S, X, CZ), pm=pm)))
    for n, gates in cases:
        circ = sk.Circuit(n, gates)
        t, out, det, _ = ctx.sim(circ, SEED)
        o = orc.Tableau(n)
        oo, od, rc = o.sim(gates, SEED)
        assert rc == 0 and (out == oo).all() and (det == od).all(), (n, gates[:12])
        assert_same_tableau(t, o)
        prog = sk.Program(ctx, circ); t2 = sk.Tableau(ctx, n)
        prog.run(t2, SEED); ctx.sync()
        assert_same_tableau(t2, o)
        t.close(); t2.close()


@pytest.mark.parametrize("seq", [0, 1])
@pytest.mark.parametrize("columns,width,rowcap,fold", [(1, 64, 0, 1), (1, 5, 0, 1), (1, 1, 0, 1), (0, 7, 0, 1), (0, 1, 0, 1),
                                                       (0, 64, 12, 1), (0, 9, 30, 1), (0, 64, 0, 0), (0, 16, 25, 0)])
def test_panel_factorisation_variants(sk, orc, columns, width, rowcap, fold, seq):
    """Panel mode (kernels_measure.cuh) has three factorisations -- the level form (all mutually independent steps of a
    panel per round; the default), the step-by-step row form in registers (SK_PANEL_SEQ=1) and the
    column form in shared memory (TMA staged) used when too many rows are active -- any panel
    width 1..64, and the gather of the next panel either folded into the apply phase or on its own (a panel
    that outgrows the row form after a folded gather asks for a full one: SK_ROW_CAP makes that happen on
    small inputs).  Every variant must reproduce sequential CHP bit for bit."""
    if seq and columns: pytest.skip("SK_PANEL_SEQ only selects between the two row-form factorisations")
    old = {k: os.environ.get(k) for k in ("SK_PANEL_COLUMNS", "SK_PANEL", "SK_ROW_CAP", "SK_NO_FOLD", "SK_PANEL_SEQ")}
    os.environ["SK_PANEL_COLUMNS"] = str(columns); os.environ["SK_PANEL"] = str(width); os.environ["SK_PANEL_SEQ"] = str(seq)
    os.environ["SK_ROW_CAP"] = str(rowcap); os.environ["SK_NO_FOLD"] = str(1 - fold)      # small caps force the regather path
    try:
        c2 = sk.Context(0)
        circs = [(sk.surface_code_circuit(7, 3, True), SEED), (sk.random_layered_circuit(256, 5), 11)]
        rng = np.random.default_rng(99)
        for n, count, pm in ((9, 300, 0.3), (70, 900, 0.15), (130, 800, 0.3)):
            circs.append((sk.Circuit(n, rand_gates(rng, n, count, pm=pm)), int(rng.integers(0, 2**63))))
        for circ, seed in circs:
            c2.reset_counters()
            t, out, det, _ = c2.sim(circ, seed)
            o = orc.Tableau(circ.n); oo, od, rc = o.sim(circ.gates, seed, workers=8)
            assert rc == 0 and (out == oo).all() and (det == od).all()
            assert_same_tableau(t, o)
            dc, oc = c2.counters(), o.counters()
            for k in ("n_rand", "n_det", "k_rand", "k_det"):
                assert dc[k] == oc[k], k
            t.close()
        c2.close()
    finally:
        for k, v in old.items():
            if v is None: os.environ.pop(k, None)
            else: os.environ[k] = v


def test_dense_tableau_falls_back_to_column_form(sk, orc):
    """A deep random Clifford circuit on 2304 qubits: nearly every row has an x in any 64 measured columns, i.e. more
    than the 1984 active rows the register-resident factorisation holds, so the kernel itself switches to the
    column-form (shared-memory, TMA-staged) factorisation -- checked through the panel counters."""
    n = 2304
    rng = np.random.default_rng(31)
    gates = rand_gates(rng, n, 10 * n, kinds=(H, S, CX, CX))
    gates += [(M, int(q), 0) for q in rng.integers(0, n, 150)]
    circ = sk.Circuit(n, gates)
    c2 = sk.Context(0)
    t, out, det, _ = c2.sim(circ, 17)
    o = orc.Tableau(n); oo, od, rc = o.sim(circ.gates, 17, workers=8)
    assert rc == 0 and (out == oo).all() and (det == od).all()
    assert_same_tableau(t, o)
    dc, oc = c2.counters(), o.counters()
    for k in ("n_rand", "n_det", "k_rand", "k_det"):
        assert dc[k] == oc[k], k
    assert dc["k_rand"] > 1984 * 10          # dense indeed: thousands of rows multiplied per random measurement
    t.close(); c2.close()


def test_run_shots_histogram_and_per_shot_records(sk, ctx, orc):
    """SPEC:330-338 run_shots: seeds seed ^ shot; |+> is 50/50 within 3 sigma, |0> all zero, GHZ-3 only 000 / 111;
    every shot's record equals the oracle run with that seed."""
    shots = 2000
    circ = sk.Circuit(5, [(H, 0, 0), (M, 0, 0), (M, 1, 0), (H, 2, 0), (CX, 2, 3), (CX, 3, 4), (M, 2, 0), (M, 3, 0), (M, 4, 0)])
    prog = sk.Program(ctx, circ); t = sk.Tableau(ctx, circ.n)
    ones, rec = prog.run_shots(t, shots, SEED, records=True)
    assert abs(ones[0] / shots - 0.5) < 0.034 and ones[1] == 0
    assert (rec[:, 2] == rec[:, 3]).all() and (rec[:, 3] == rec[:, 4]).all() and 0 < ones[2] < shots
    assert (ones == rec.sum(axis=0)).all()
    for s in (0, 1, 7, 1999):
        o = orc.Tableau(circ.n)
        oo, _, rc = o.sim(circ.gates, SEED ^ s)
        assert rc == 0 and (rec[s] == oo).all()
    sc = sk.surface_code_circuit(5, 5, True)
    prog2 = sk.Program(ctx, sc); t2 = sk.Tableau(ctx, sc.n)
    ones2, rec2 = prog2.run_shots(t2, 16, 3, records=True)
    for s in range(16):
        o = orc.Tableau(sc.n)
        oo, _, rc = o.sim(sc.gates, 3 ^ s)
        assert rc == 0 and (rec2[s] == oo).all()
    assert (ones2 == rec2.sum(axis=0)).all()
    prog.close(); prog2.close(); t.close(); t2.close()
