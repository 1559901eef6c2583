"""Pin the oracle's row arithmetic to the REFERENCE: committed golden vectors (generated from
the compiled /root/reference/proj/src/pauli.cpp by tests/golden/make_golden.py) and, when
oracle/_ref/libstabkit_ref.so is present, the live compiled reference on fresh random inputs."""
import ctypes as C
import json
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden", "pauli_ref_vectors.json")


def unhex(h, shape):
    return np.array([int(v, 16) for v in h], dtype=np.uint64).reshape(shape)


@pytest.fixture(scope="module")
def gold():
    with open(GOLD) as f:
        return json.load(f)


def test_rng_golden(orc, gold):
    L = orc.lib()
    for k, v in gold["splitmix64"].items():          # rng.hpp:23-28
        assert format(L.orc_splitmix64(int(k)), "016x") == v
    for s, bits in gold["counter_bits"].items():     # rng.hpp:33-39
        assert "".join(str(L.orc_counter_bit(int(s), k)) for k in range(64)) == bits
    buf = np.zeros(8, np.uint64)
    for s, vals in gold["seq"].items():              # rng.hpp:43-65
        L.orc_seq_fill(int(s), orc._p(buf), 8)
        assert [format(int(v), "016x") for v in buf] == vals
    # SURVEY 8c probes
    assert gold["splitmix64"]["0"] == "e220a8397b1dcdaf" and gold["counter_bits"]["0"][:32] == "01111010000000100000010000111101"


def test_row_arithmetic_golden(orc, gold):
    L, p = orc.lib(), orc._p
    for case in gold["cases"]:
        n, m = case["n"], case["m"]; W = orc.words_for(n)
        x, z = unhex(case["x"], (m, W)), unhex(case["z"], (m, W))
        signs = np.array(case["signs"], np.uint8)
        for i in range(m):
            j = (i + 1) % m
            assert L.orc_g_sum(p(x[i]), p(z[i]), p(x[j]), p(z[j]), W) == case["g_sum"][i]          # pauli.cpp:189-205
            assert L.orc_commutes(p(x[i]), p(z[i]), p(x[j]), p(z[j]), W) == case["commutes"][i]    # pauli.cpp:117-127
            assert L.orc_qw_commutes(p(x[i]), p(z[i]), p(x[j]), p(z[j]), W) == case["qw"][i]       # pauli.cpp:129-140
        rows = orc.Rows(n, x, z, signs)
        assert sum(case["weight"]) == rows.weight_sum()                                             # pauli.cpp:100-106
        assert format(int(rows.commutation_vector(x[0], z[0])[0]), "x") == case["commutation_vector_row0"]  # :215-237
        rows.apply([tuple(g) for g in case["gates"]])                                               # pauli.cpp:146-187
        xo, zo, so = rows.get()
        assert (xo == unhex(case["after_x"], (m, W))).all() and (zo == unhex(case["after_z"], (m, W))).all()
        assert [int(v) for v in so] == case["after_signs"]
        for i in range(m):                                                                          # pauli.cpp:239-254
            j = (i + 1) % m
            t = orc.Rows(n, x[i:i + 1], z[i:i + 1], signs[i:i + 1])
            rc = t.rowsum_plus_i(0, x[j], z[j], signs[j])
            g = case["rpi"][i]
            assert rc == g["rc"]
            if rc == 0:
                tx, tz, ts = t.get()
                assert (tx[0] == unhex(g["x"], (W,))).all() and (tz[0] == unhex(g["z"], (W,))).all() and int(ts[0]) == g["sign"]


def test_parse_text_golden(orc, gold):
    # our text helpers follow pauli.cpp:23-57 / :88-98 conventions (leftmost = qubit 0, explicit sign)
    for t, g in gold["parse"].items():
        if g["rc"] == 0:
            n, x, z, s = orc.pauli_from_text(t)
            assert orc.pauli_to_text(n, x, z, s) == g["text"]


def test_oracle_vs_live_reference(orc):
    R = orc.ref()
    if R is None:
        pytest.skip("oracle/_ref/libstabkit_ref.so not built (needs /root/reference)")
    L, p = orc.lib(), orc._p
    rng = np.random.default_rng(7)
    for n in (3, 64, 97, 300):
        W = orc.words_for(n)
        mask = np.full(W, np.uint64(2**64 - 1)); rem = n % 64
        if rem: mask[-1] = np.uint64((1 << rem) - 1)
        for _ in range(40):
            a = rng.integers(0, 2**64, (4, W), dtype=np.uint64) & mask
            ax, az, bx, bz = a
            assert L.orc_g_sum(p(ax), p(az), p(bx), p(bz), W) == R.ref_g_sum(p(ax), p(az), p(bx), p(bz), W)
            assert L.orc_commutes(p(ax), p(az), p(bx), p(bz), W) == R.ref_commutes(n, p(ax), p(az), p(bx), p(bz))
            assert L.orc_qw_commutes(p(ax), p(az), p(bx), p(bz), W) == R.ref_qw_commutes(n, p(ax), p(az), p(bx), p(bz))
            sa, sb = int(rng.integers(0, 2)), int(rng.integers(0, 2))
            t = orc.Rows(n, ax[None], az[None], np.array([sa], np.uint8))
            rc = t.rowsum_plus_i(0, bx, bz, sb)
            tx, tz, ts = ax.copy(), az.copy(), C.c_int(sa)
            rc2 = R.ref_rowsum_plus_i(n, p(tx), p(tz), C.byref(ts), p(bx), p(bz), sb)
            assert rc == rc2
            if rc == 0:
                ox, oz, os_ = t.get()
                assert (ox[0] == tx).all() and (oz[0] == tz).all() and int(os_[0]) == ts.value
            # one random gate through conj_*
            k = int(rng.choice([0, 1, 2, 6])); qa = int(rng.integers(0, n)); qb = int(rng.integers(0, n - 1)); qb += qb >= qa
            t = orc.Rows(n, ax[None], az[None], np.array([sa], np.uint8)); t.apply([(k, qa, qb)])
            tx, tz, ts = ax.copy(), az.copy(), C.c_int(sa)
            R.ref_conj(n, p(tx), p(tz), C.byref(ts), k, qa, qb)
            ox, oz, os_ = t.get()
            assert (ox[0] == tx).all() and (oz[0] == tz).all() and int(os_[0]) == ts.value
    for s in (0, 1, 99):
        for k in range(50):
            assert L.orc_counter_bit(s, k) == R.ref_counter_bit(s, k)
