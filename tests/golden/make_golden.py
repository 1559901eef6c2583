"""Regenerate tests/golden/pauli_ref_vectors.json from the COMPILED REFERENCE
(oracle/_ref/libstabkit_ref.so == /root/reference/proj/src/pauli.cpp + oracle/ref_shim.cpp).

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
The JSON is committed; the tests then pin oracle/liboracle.so (and through it the CUDA
kernels) to the reference's own outputs even where /root/reference is absent.
"""
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle_py as o  # noqa: E402

o.build(ref=True)
R = o.ref()
assert R is not None, "oracle/_ref/libstabkit_ref.so missing (make -C oracle ref)"
p = o._p
rng = np.random.default_rng(20250703)


def rand_rows(n, m, density=0.5):
    W = o.words_for(n)
    bits = rng.random((m, 2, n)) < density
    x = np.zeros((m, W), np.uint64); z = np.zeros((m, W), np.uint64)
    for i in range(m):
        for q in np.nonzero(bits[i, 0])[0]: x[i, q >> 6] |= np.uint64(1 << int(q & 63))
        for q in np.nonzero(bits[i, 1])[0]: z[i, q >> 6] |= np.uint64(1 << int(q & 63))
    return x, z


def hexl(a):
    return [format(int(v), "016x") for v in np.asarray(a).reshape(-1)]


out = {"comment": "outputs of the compiled reference pauli.cpp; see make_golden.py", "cases": []}

# rng ------------------------------------------------------------------------------------
out["splitmix64"] = {str(v): format(R.ref_splitmix64(v), "016x") for v in (0, 1, 2, 0xdeadbeef, 2**64 - 1)}
out["counter_bits"] = {str(s): "".join(str(R.ref_counter_bit(s, k)) for k in range(64)) for s in (0, 7, 0xdeadbeef, 20250703)}
seq = np.zeros(8, np.uint64)
out["seq"] = {}
for s in (0, 42, 20250703):
    R.ref_seq_fill(s, p(seq), 8); out["seq"][str(s)] = hexl(seq)
out["seq_unit_42_skip0"] = R.ref_seq_unit(42, 0)

# row arithmetic --------------------------------------------------------------------------
for n in (1, 2, 5, 63, 64, 65, 130, 200):
    W = o.words_for(n)
    for density in (0.5, 0.1):
        m = 6
        x, z = rand_rows(n, m, density)
        signs = rng.integers(0, 2, m).astype(np.uint8)
        case = {"n": n, "x": hexl(x), "z": hexl(z), "signs": [int(s) for s in signs], "m": m}
        # pairwise g_sum / commutes / qw_commutes of row i with row (i+1)%m
        case["g_sum"] = []; case["commutes"] = []; case["qw"] = []; case["weight"] = []
        for i in range(m):
            j = (i + 1) % m
            case["g_sum"].append(int(R.ref_g_sum(p(x[i]), p(z[i]), p(x[j]), p(z[j]), W)))
            case["commutes"].append(int(R.ref_commutes(n, p(x[i]), p(z[i]), p(x[j]), p(z[j]))))
            case["qw"].append(int(R.ref_qw_commutes(n, p(x[i]), p(z[i]), p(x[j]), p(z[j]))))
            case["weight"].append(int(R.ref_weight(n, p(x[i]), p(z[i]))))
        # commutation_vector of row 0 against all rows
        cv = np.zeros(1, np.uint64)
        R.ref_commutation_vector(n, p(x[0]), p(z[0]), p(x), p(z), m, p(cv))
        case["commutation_vector_row0"] = format(int(cv[0]), "x")
        # a fixed gate sequence applied to every row through conj_*
        gates = []
        for _ in range(12):
            k = int(rng.choice([0, 1, 2, 6] if n > 1 else [0, 1, 2]))
            a = int(rng.integers(0, n)); b = 0
            if k == 6:
                b = int(rng.integers(0, n - 1)); b += b >= a
            gates.append([k, a, b])
        case["gates"] = gates
        xo, zo, so = x.copy(), z.copy(), signs.astype(np.int32).copy()
        for i in range(m):
            s = C.c_int(int(so[i]))
            for k, a, b in gates:
                R.ref_conj(n, p(xo[i]), p(zo[i]), C.byref(s), k, a, b)
            so[i] = s.value
        case["after_x"] = hexl(xo); case["after_z"] = hexl(zo); case["after_signs"] = [int(v) for v in so]
        # rowsum_plus_i(target=row i, pushed=row (i+1)%m)
        case["rpi"] = []
        for i in range(m):
            j = (i + 1) % m
            tx, tz = x[i].copy(), z[i].copy(); ts = C.c_int(int(signs[i]))
            rc = R.ref_rowsum_plus_i(n, p(tx), p(tz), C.byref(ts), p(x[j]), p(z[j]), int(signs[j]))
            case["rpi"].append({"rc": rc, "x": hexl(tx), "z": hexl(tz), "sign": ts.value})
        out["cases"].append(case)

# parse/str
buf = C.create_string_buffer(128)
out["parse"] = {}
for t in ("XZ", "-Y", "IQ", "+", "+IXYZ", "ZZZZ"):
    rc = R.ref_parse_str(t.encode(), buf, 128)
    out["parse"][t] = {"rc": rc if rc < 0 else 0, "text": buf.value.decode()}

path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "pauli_ref_vectors.json")
with open(path, "w") as f:
    json.dump(out, f, indent=0, separators=(",", ":"))
print("wrote", path, os.path.getsize(path), "bytes")
