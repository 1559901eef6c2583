"""CPU-only checks of the product's host logic and of the C-ABI surface (no compute calls)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol(sk):
    hdr = open(os.path.join(ROOT, "include", "stabkit_b200.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    declared = sorted(set(re.findall(r"\b(sk_[a-z0-9_]+)\s*\(", hdr)))
    assert len(declared) >= 45
    L = C.CDLL(sk.LIB_PATH)
    missing = [s for s in declared if not hasattr(L, s)]
    assert not missing, missing
    assert sorted(sk.EXPORTS) == declared


def test_no_cpu_fallback_without_device(sk):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    with pytest.raises(sk.CudaError):
        sk.Context(0)


def test_product_does_not_touch_the_oracle():
    bad = []
    for base, _, files in os.walk(os.path.join(ROOT, "paper_2507_03092_b200")):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".hpp", ".h")):
                txt = open(os.path.join(base, f), errors="ignore").read()
                if re.search(r"oracle_py|liboracle|stab_oracle|from oracle|import oracle|oracle/", txt):
                    bad.append(f)
    for f in os.listdir(os.path.join(ROOT, "include", "stabkit")) if os.path.isdir(os.path.join(ROOT, "include", "stabkit")) else []:
        txt = open(os.path.join(ROOT, "include", "stabkit", f)).read()
        if re.search(r"liboracle|stab_oracle|oracle/", txt):
            bad.append(f)
    assert not bad, bad


def test_surface_code_generator(sk):                # SPEC:375-383, 397; SURVEY 8 config sizes
    c = sk.surface_code_circuit(3, 1)
    assert (c.n, c.num_measurements) == (17, 8)
    assert sk.surface_code_circuit(3, 2).num_measurements == 16
    with pytest.raises(sk.StabkitError):
        sk.surface_code_circuit(2, 1)
    with pytest.raises(sk.StabkitError):
        sk.surface_code_circuit(3, 0)
    for d, nH, nCX, nM in ((25, 15600, 60000, 15600 + 625), (71, 357840, 1411480, 357840 + 5041)):
        c = sk.surface_code_circuit(d, d, True)
        k = c.gates["kind"]
        assert c.n == 2 * d * d - 1
        assert ((k == sk.H).sum(), (k == sk.CX).sum(), (k == sk.M).sum()) == (nH, nCX, nM)
    for d, r, f in ((3, 1, False), (5, 2, False), (7, 3, True)):
        c = sk.surface_code_circuit(d, r, f)
        assert sk.validate_chunks(c) == []                              # every emitted chunk passes
        v = sk.validate_chunks(c, strict=True)                          # strict: the M blocks are reported, and nothing else
        assert len(v) == c.num_measurements and all(kind == "measurement" for _, _, kind in v)
    # every ancilla has 2 or 4 neighbours; X and Z checks each (d^2-1)/2
    deg = {}
    for g in sk.surface_code_circuit(5, 1).gates:
        if g["kind"] == sk.CX:
            a = int(max(g["q0"], g["q1"])); deg[a] = deg.get(a, 0) + 1
    assert len(deg) == 24 and set(deg.values()) == {2, 4}


def test_surface_code_generator_equals_the_oracles_independent_one(sk, orc):
    """The product generator (csrc/circuit_host.cpp) and the oracle's own (oracle/stab_oracle.cpp: orc_surface_code), written
    separately from SPEC:375-403 + DESIGN section 8, agree gate for gate and mark for mark."""
    for d, r, f in ((3, 1, False), (3, 3, True), (5, 2, True), (7, 7, False), (9, 1, True), (25, 2, True), (71, 2, True)):
        c = sk.surface_code_circuit(d, r, f)
        n, g, m = orc.surface_code(d, r, f)
        assert n == c.n and len(g) == len(c.gates) and (g == c.gates).all() and (m == c.chunk_marks).all(), (d, r, f)
    with pytest.raises(ValueError):
        orc.surface_code(4, 1)


def test_random_layered_generator(sk):
    c = sk.random_layered_circuit(8, 1)
    k = c.gates["kind"]
    assert len(c.gates) == 3 * (4 + 4 + 1) and (k == sk.M).sum() == 3 and (k == sk.CX).sum() == 12
    a, b = sk.random_layered_circuit(4, 9), sk.random_layered_circuit(4, 9)
    assert (a.gates == b.gates).all()
    with pytest.raises(sk.StabkitError):
        sk.random_layered_circuit(7, 1)
    c = sk.random_layered_circuit(64, 3)
    assert sk.validate_chunks(c) == []
    assert all(kind == "measurement" for _, _, kind in sk.validate_chunks(c, strict=True))
    m = [int(g["q0"]) for g in c.gates[:32 + 32 + 7] if g["kind"] == sk.M]
    assert len(m) == 7 and len(set(m)) == 7 and all(q >= 32 for q in m)


def test_parse_native(sk):
    c = sk.parse_native("qubits 2\nh 0\ncx 0 1\nm 0\nm 1")
    assert c.n == 2 and [int(k) for k in c.gates["kind"]] == [sk.H, sk.CX, sk.M, sk.M]
    with pytest.raises(sk.ParseError) as e:
        sk.parse_native("qubits 1\ncx 0 0")
    assert e.value.line == 2
    c = sk.parse_native("qubits 2\nh 0\nchunk\nh 1")
    assert len(c.gates) == 2 and list(c.chunk_marks) == [1]
    for bad, line in (("h 0\n", 1), ("qubits 2\nfoo 1\n", 2), ("qubits 2\n# c\n\nh 5\n", 4), ("qubits 2\nh\n", 2), ("qubits 2\ncx 0\n", 2)):
        with pytest.raises(sk.ParseError) as e:
            sk.parse_native(bad)
        assert e.value.line == line
    c = sk.random_layered_circuit(16, 4)
    c2 = sk.parse_native(c.emit_native())
    assert c2.n == c.n and (c2.gates == c.gates).all() and (c2.chunk_marks == c.chunk_marks).all()


def test_validate_chunks(sk):
    assert sk.validate_chunks(sk.parse_native("qubits 2\nh 0\nh 1")) == []
    assert sk.validate_chunks(sk.parse_native("qubits 2\nh 0\ncx 0 1")) == [(0, 1, "collision")]
    assert sk.validate_chunks(sk.parse_native("qubits 1\nm 0"), strict=True) == [(0, 0, "measurement")]   # SPEC:270, literal
    assert sk.validate_chunks(sk.parse_native("qubits 1\nm 0")) == []                  # a measurement barrier region
    assert sk.validate_chunks(sk.parse_native("qubits 2\nh 0\nm 1")) == [(0, 1, "measurement")]          # M next to a gate
    assert sk.validate_chunks(sk.parse_native("qubits 2\nh 0\nchunk\nm 1\nm 1\nchunk\nh 1")) == []


def test_parse_qasm2_subset(sk):
    bell = sk.parse_native("qubits 2\nh 0\ncx 0 1\nm 0\nm 1")
    q = sk.parse_qasm2_subset('OPENQASM 2.0;\ninclude "qelib1.inc";\nqreg q[2];\ncreg c[2];\n// Bell pair\nh q[0];\ncx q[0],q[1];\nmeasure q[0] -> c[0];\nmeasure q[1] -> c[1];\n')
    assert q.n == 2 and (q.gates == bell.gates).all() and len(q.chunk_marks) == 0
    with pytest.raises(sk.UnsupportedError) as e:
        sk.parse_qasm2_subset("OPENQASM 2.0;\nqreg q[1];\nrz(0.1) q[0];\n")
    assert e.value.line == 3 and "rz" in str(e.value)
    c = sk.parse_qasm2_subset("OPENQASM 2.0;\nqreg q[4];\nt q[2];\n")
    assert c.n == 4 and len(c.gates) == 1 and int(c.gates[0]["kind"]) == sk.T and int(c.gates[0]["q0"]) == 2
    # barrier -> chunk mark; register-wide statements; every supported mnemonic
    c = sk.parse_qasm2_subset("OPENQASM 2.0; qreg r[3]; creg m[3]; h r; barrier r; s r[0]; sdg r[1]; x r[2]; y r[0]; z r[1];\n"
                              "cz r[0],r[1]; swap r[1],r[2]; tdg r[0]; barrier r[0],r[1]; measure r -> m;")
    assert [int(k) for k in c.gates["kind"]] == [sk.H] * 3 + [sk.S, sk.SDG, sk.X, sk.Y, sk.Z, sk.CZ, sk.SWAP, sk.TDG] + [sk.M] * 3
    assert list(c.chunk_marks) == [3, 11]
    for bad, exc in (("OPENQASM 2.0; qreg a[2]; qreg b[2];", sk.UnsupportedError), ("OPENQASM 2.0; qreg q[2]; creg c[2]; if (c==1) x q[0];", sk.UnsupportedError),
                     ("OPENQASM 2.0; qreg q[2]; gate foo a { h a; }", sk.UnsupportedError), ("OPENQASM 2.0; qreg q[2]; ccx q[0],q[1],q[0];", sk.UnsupportedError),
                     ("OPENQASM 2.0; qreg q[2]; h q[2];", sk.ParseError), ("OPENQASM 2.0; qreg q[2]; cx q[0],q[0];", sk.ParseError),
                     ("OPENQASM 2.0; qreg q[2]; h q[0]", sk.ParseError), ("OPENQASM 2.0; h q[0];", sk.ParseError),
                     ("OPENQASM 3.0; qreg q[2];", sk.UnsupportedError), ("OPENQASM 2.0; qreg q[2]; measure q[0] -> c[0];", sk.ParseError)):
        with pytest.raises(exc):
            sk.parse_qasm2_subset(bad)
    # the parsed circuit round-trips through the native format
    assert (sk.parse_native(c.emit_native()).gates == c.gates).all()


def test_algorithmic_bytes_formula_matches_the_oracles_copy(sk, orc):
    """bench.py's roofline numerator lives in the product package; the oracle keeps its own copy."""
    cnt = {"gate_hist": [7, 3, 2, 5, 1, 4, 11, 6, 2, 9, 0, 0], "n_rand": 13, "n_det": 29, "k_rand": 101, "k_det": 57}
    for n in (17, 1249, 10081):
        assert sk.algorithmic_bytes(n, cnt, fused_layers=5) == orc.algorithmic_bytes(n, cnt, fused_layers=5)
        assert sk.algorithmic_bytes(n, cnt) == orc.algorithmic_bytes(n, cnt)


def test_workload_generators_follow_the_reference_stream():
    """paper_2507_03092_b200/workloads.py restates SplitMix64 (proj/include/stabkit/rng.hpp:42-65) in vector form: pinned
    against the oracle's sequential generator (itself pinned by the compiled reference, tests/test_oracle_golden.py) and
    SURVEY 8c's known answers; C4 terms are sorted by |coeff| descending, C5 has ~10 % T gates."""
    import importlib.util, os
    import numpy as np
    from oracle import oracle_py as orc
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("wl", os.path.join(root, "paper_2507_03092_b200", "workloads.py"))
    wl = importlib.util.module_from_spec(spec); spec.loader.exec_module(wl)
    raw = np.zeros(4096, np.uint64); orc.lib().orc_seq_fill(20250703, orc._p(raw), len(raw))
    assert (wl.splitmix_stream(20250703, 4096) == raw).all()
    assert [hex(int(v)) for v in wl.splitmix_stream(42, 4)] == ["0xbdd732262feb6e95", "0x28efe333b266f103", "0x47526757130f9f52", "0x581ce1ff0e4ae394"]
    x, z, c = wl.c4_terms(2000)
    assert x.shape == (2000, 2) and (np.abs(c[:-1]) >= np.abs(c[1:])).all() and (np.abs(c) < 1).all()
    dt = np.dtype([("kind", "u1"), ("pad", "u1", 3), ("q0", "<u4"), ("q1", "<u4")])
    g = wl.c5_gates(50, 4000, gate_dtype=dt, kinds=(0, 1, 6, 10, 11))
    nt = int(((g["kind"] == 10) | (g["kind"] == 11)).sum())
    assert 300 < nt < 500 and (g["q0"] < 50).all() and ((g["kind"] != 6) | (g["q0"] != g["q1"])).all()
