"""ctypes wrapper over oracle/liboracle.so (our CPU restatement) and, when present,
oracle/_ref/libstabkit_ref.so (the reference's own pauli.cpp).

TEST INFRASTRUCTURE ONLY: importable from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  Never imported by paper_2507_03092_b200/.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
REFLIB = os.path.join(HERE, "_ref", "libstabkit_ref.so")
GATE_DTYPE = np.dtype([("kind", "u1"), ("pad", "u1", (3,)), ("q0", "<u4"), ("q1", "<u4")])


def build(ref: bool = True) -> None:
    """make liboracle.so, and _ref/ when the reference tree is mounted (this container only)."""
    src = os.path.join(HERE, "stab_oracle.cpp")
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(src):
        subprocess.run(["make", "-C", HERE, "all"], check=True, capture_output=True)
    if ref and os.path.exists("/root/reference/proj/src/pauli.cpp"):
        shim = os.path.join(HERE, "ref_shim.cpp")
        if not os.path.exists(REFLIB) or os.path.getmtime(REFLIB) < os.path.getmtime(shim):
            subprocess.run(["make", "-C", HERE, "ref"], check=True, capture_output=True)


_lib = None
_ref = None


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def lib():
    global _lib
    if _lib is None:
        build(ref=False)
        L = C.CDLL(LIB)
        vp, u64, sz = C.c_void_p, C.c_uint64, C.c_size_t
        L.orc_splitmix64.restype = u64; L.orc_splitmix64.argtypes = [u64]
        L.orc_counter_bit.restype = C.c_int; L.orc_counter_bit.argtypes = [u64, u64]
        L.orc_seq_fill.argtypes = [u64, vp, sz]
        L.orc_g_sum.restype = C.c_int64; L.orc_g_sum.argtypes = [vp, vp, vp, vp, sz]
        L.orc_commutes.restype = C.c_int; L.orc_commutes.argtypes = [vp, vp, vp, vp, sz]
        L.orc_qw_commutes.restype = C.c_int; L.orc_qw_commutes.argtypes = [vp, vp, vp, vp, sz]
        L.orc_rows_new.restype = vp; L.orc_rows_new.argtypes = [sz, sz]
        L.orc_rows_free.argtypes = [vp]
        L.orc_rows_count.restype = sz; L.orc_rows_count.argtypes = [vp]
        L.orc_rows_set.argtypes = [vp, vp, vp, vp]; L.orc_rows_get.argtypes = [vp, vp, vp, vp]
        L.orc_rows_apply.argtypes = [vp, vp, sz]
        L.orc_commutation_vector.argtypes = [vp, vp, vp, vp]
        L.orc_rowsum_plus_i.restype = C.c_int; L.orc_rowsum_plus_i.argtypes = [vp, sz, vp, vp, C.c_int]
        L.orc_weight_sum.restype = u64; L.orc_weight_sum.argtypes = [vp]
        L.orc_first_duplicate.restype = C.c_int; L.orc_first_duplicate.argtypes = [vp, C.POINTER(u64), C.POINTER(u64)]
        L.orc_group_first_fit.restype = u64; L.orc_group_first_fit.argtypes = [vp, C.c_int, vp, C.POINTER(u64)]
        L.orc_verify_grouping.restype = u64; L.orc_verify_grouping.argtypes = [vp, C.c_int, vp]
        L.orc_tab_new.restype = vp; L.orc_tab_new.argtypes = [sz]
        L.orc_tab_free.argtypes = [vp]
        L.orc_tab_get.argtypes = [vp, vp, vp, vp]; L.orc_tab_set.argtypes = [vp, vp, vp, vp]
        L.orc_tab_rowsum.restype = C.c_int; L.orc_tab_rowsum.argtypes = [vp, sz, sz]
        L.orc_tab_sim.restype = C.c_int; L.orc_tab_sim.argtypes = [vp, vp, sz, u64, C.c_int, vp, vp, u64]
        L.orc_tab_counters.argtypes = [vp, vp]
        L.orc_surface_code.restype = u64; L.orc_surface_code.argtypes = [C.c_uint32, C.c_uint32, C.c_int, vp, C.POINTER(sz), vp, C.POINTER(sz)]
        L.orc_transpile.restype = vp; L.orc_transpile.argtypes = [sz, vp, sz]
        L.orc_pbc_free.argtypes = [vp]
        L.orc_pbc_status.restype = C.c_int; L.orc_pbc_status.argtypes = [vp]
        L.orc_pbc_stats.argtypes = [vp, vp]
        L.orc_pbc_layer_rows.restype = sz; L.orc_pbc_layer_rows.argtypes = [vp, sz]
        L.orc_pbc_layer_get.argtypes = [vp, sz, vp, vp, vp]
        L.orc_pbc_mtab.restype = vp; L.orc_pbc_mtab.argtypes = [vp]
        L.orc_build_ttab.restype = vp; L.orc_build_ttab.argtypes = [sz, vp, sz, vp, C.POINTER(C.c_int)]
        L.orc_t_separate_ids.restype = sz; L.orc_t_separate_ids.argtypes = [vp, vp]
        _lib = L
    return _lib


def ref():
    """The compiled reference (None when oracle/_ref was never built)."""
    global _ref
    if _ref is None:
        if not os.path.exists(REFLIB):
            return None
        R = C.CDLL(REFLIB)
        vp, u64, sz = C.c_void_p, C.c_uint64, C.c_size_t
        R.ref_splitmix64.restype = u64; R.ref_splitmix64.argtypes = [u64]
        R.ref_counter_bit.restype = C.c_int; R.ref_counter_bit.argtypes = [u64, u64]
        R.ref_seq_fill.argtypes = [u64, vp, sz]
        R.ref_seq_unit.restype = C.c_double; R.ref_seq_unit.argtypes = [u64, sz]
        R.ref_g_sum.restype = C.c_int64; R.ref_g_sum.argtypes = [vp, vp, vp, vp, sz]
        R.ref_commutes.restype = C.c_int; R.ref_commutes.argtypes = [sz, vp, vp, vp, vp]
        R.ref_qw_commutes.restype = C.c_int; R.ref_qw_commutes.argtypes = [sz, vp, vp, vp, vp]
        R.ref_weight.restype = u64; R.ref_weight.argtypes = [sz, vp, vp]
        R.ref_conj.argtypes = [sz, vp, vp, C.POINTER(C.c_int), C.c_int, sz, sz]
        R.ref_rowsum_plus_i.restype = C.c_int; R.ref_rowsum_plus_i.argtypes = [sz, vp, vp, C.POINTER(C.c_int), vp, vp, C.c_int]
        R.ref_commutation_vector.argtypes = [sz, vp, vp, vp, vp, sz, vp]
        R.ref_parse_str.restype = C.c_int; R.ref_parse_str.argtypes = [C.c_char_p, C.c_char_p, sz]
        _ref = R
    return _ref


def words_for(n):
    return (n + 63) // 64


def gates_array(gates):
    if isinstance(gates, np.ndarray) and gates.dtype == GATE_DTYPE:
        return np.ascontiguousarray(gates)
    out = np.zeros(len(gates), dtype=GATE_DTYPE)
    for i, g in enumerate(gates):
        out[i]["kind"] = g[0]; out[i]["q0"] = g[1]; out[i]["q1"] = g[2] if len(g) > 2 else 0
    return out


# ---- Pauli text helpers (pauli.hpp:39-41, 62-63: leftmost char = qubit 0) ---------------
def pauli_from_text(text: str):
    sign = 0
    if text[0] in "+-":
        sign = int(text[0] == "-"); text = text[1:]
    n = len(text); W = words_for(n)
    x = np.zeros(W, np.uint64); z = np.zeros(W, np.uint64)
    for q, ch in enumerate(text):
        if ch in "XY": x[q >> 6] |= np.uint64(1 << (q & 63))
        if ch in "ZY": z[q >> 6] |= np.uint64(1 << (q & 63))
    return n, x, z, sign


def pauli_to_text(n, x, z, sign) -> str:
    s = "-" if sign else "+"
    for q in range(n):
        xb = (int(x[q >> 6]) >> (q & 63)) & 1; zb = (int(z[q >> 6]) >> (q & 63)) & 1
        s += "IXZY"[xb + 2 * zb]
    return s


class Rows:
    """Row-major block of signed Pauli rows in the oracle."""

    def __init__(self, n, x=None, z=None, r=None, m=None):
        self.n, self.W = n, words_for(n)
        if x is not None:
            x = np.ascontiguousarray(x, np.uint64).reshape(-1, self.W); m = x.shape[0]
        self.h = lib().orc_rows_new(n, m or 0)
        if x is not None and m:
            z = np.ascontiguousarray(z, np.uint64).reshape(-1, self.W)
            r = np.ascontiguousarray(r if r is not None else np.zeros(m), np.uint8)
            lib().orc_rows_set(self.h, _p(x), _p(z), _p(r))

    @classmethod
    def from_text(cls, texts):
        ps = [pauli_from_text(t) for t in texts]
        n = ps[0][0]
        return cls(n, np.stack([p[1] for p in ps]), np.stack([p[2] for p in ps]), np.array([p[3] for p in ps], np.uint8))

    def __del__(self):
        try: lib().orc_rows_free(self.h)
        except Exception: pass

    @property
    def m(self): return int(lib().orc_rows_count(self.h))

    def get(self):
        m = self.m
        x = np.zeros((m, self.W), np.uint64); z = np.zeros_like(x); r = np.zeros(m, np.uint8)
        if m: lib().orc_rows_get(self.h, _p(x), _p(z), _p(r))
        return x, z, r

    def texts(self):
        x, z, r = self.get()
        return [pauli_to_text(self.n, x[i], z[i], r[i]) for i in range(self.m)]

    def apply(self, gates):
        g = gates_array(gates); lib().orc_rows_apply(self.h, _p(g), len(g))

    def commutation_vector(self, px, pz):
        out = np.zeros(max(1, words_for(self.m)), np.uint64)
        lib().orc_commutation_vector(self.h, _p(np.ascontiguousarray(px, np.uint64)), _p(np.ascontiguousarray(pz, np.uint64)), _p(out))
        return out

    def rowsum_plus_i(self, i, px, pz, pr):
        return lib().orc_rowsum_plus_i(self.h, i, _p(np.ascontiguousarray(px, np.uint64)), _p(np.ascontiguousarray(pz, np.uint64)), int(pr))

    def weight_sum(self): return int(lib().orc_weight_sum(self.h))

    def first_duplicate(self):
        i, j = C.c_uint64(), C.c_uint64()
        return (int(i.value), int(j.value)) if lib().orc_first_duplicate(self.h, C.byref(i), C.byref(j)) else None

    def group_first_fit(self, mode):
        out = np.zeros(max(1, self.m), np.uint32); calls = C.c_uint64()
        ng = lib().orc_group_first_fit(self.h, mode, _p(out), C.byref(calls))
        return out[:self.m], int(ng), int(calls.value)

    def verify_grouping(self, mode, group):
        return int(lib().orc_verify_grouping(self.h, mode, _p(np.ascontiguousarray(group, np.uint32))))


def surface_code(d: int, rounds: int, final_data_measure: bool = False):
    """SPEC:375-383 surface_code_circuit, the oracle's own generator (independent of the product's):
    -> (n, gates GATE_DTYPE[], chunk_marks u32[]).  Lets bench.py's reference arm and the tests build their
    input without loading the CUDA library, and pins the product's generator gate for gate."""
    L = lib()
    ng, nm = C.c_size_t(), C.c_size_t()
    n = L.orc_surface_code(d, rounds, int(final_data_measure), None, C.byref(ng), None, C.byref(nm))
    if n == 0:
        raise ValueError(f"surface_code(d={d}, rounds={rounds}): d must be odd >= 3, rounds >= 1 (SPEC:379)")
    gates = np.zeros(ng.value, dtype=GATE_DTYPE); marks = np.zeros(max(nm.value, 1), dtype=np.uint32)
    L.orc_surface_code(d, rounds, int(final_data_measure), _p(gates), C.byref(ng), _p(marks), C.byref(nm))
    return int(n), gates, marks[:nm.value]


class Tableau:
    def __init__(self, n, _h=None, _owner=None):
        self.n, self.W = n, words_for(n)
        self._owner = _owner
        self.h = _h if _h is not None else lib().orc_tab_new(n)

    def __del__(self):
        try:
            if self._owner is None: lib().orc_tab_free(self.h)
        except Exception: pass

    def get(self):
        x = np.zeros((2 * self.n, self.W), np.uint64); z = np.zeros_like(x); r = np.zeros(2 * self.n, np.uint8)
        lib().orc_tab_get(self.h, _p(x), _p(z), _p(r)); return x, z, r

    def set(self, x, z, r):
        lib().orc_tab_set(self.h, _p(np.ascontiguousarray(x, np.uint64)), _p(np.ascontiguousarray(z, np.uint64)), _p(np.ascontiguousarray(r, np.uint8)))

    def texts(self):
        x, z, r = self.get()
        return [pauli_to_text(self.n, x[i], z[i], r[i]) for i in range(2 * self.n)]

    def rowsum(self, h, i): return lib().orc_tab_rowsum(self.h, h, i)

    def sim(self, gates, seed, workers=1, ordinal0=0):
        """Runs gates (Clifford + M) from the current state. -> (outcomes, deterministic, status)."""
        g = gates_array(gates)
        nm = int((g["kind"] == 9).sum())
        o = np.zeros(max(nm, 1), np.uint8); d = np.zeros(max(nm, 1), np.uint8)
        rc = lib().orc_tab_sim(self.h, _p(g), len(g), seed, workers, _p(o), _p(d), ordinal0)
        return o[:nm], d[:nm], rc

    def counters(self):
        c = np.zeros(16, np.uint64); lib().orc_tab_counters(self.h, _p(c))
        return {"n_rand": int(c[0]), "n_det": int(c[1]), "k_rand": int(c[2]), "k_det": int(c[3]), "gate_hist": [int(v) for v in c[4:16]]}


class Pbc:
    def __init__(self, n, gates, exact=False):
        """exact=False: Algorithms 2-3 as published; exact=True: the unitary-exact variant (flags bit 0)."""
        g = gates_array(gates); self.n, self.W = n, words_for(n)
        self.h = lib().orc_transpile_ex(n, _p(g), len(g), 1 if exact else 0)
        self.status = lib().orc_pbc_status(self.h)

    def __del__(self):
        try: lib().orc_pbc_free(self.h)
        except Exception: pass

    def stats(self):
        s = np.zeros(5, np.uint64); lib().orc_pbc_stats(self.h, _p(s))
        return dict(zip(["initial_t", "final_rotations_rowcount", "final_rotations_pauliweight", "layers", "passes"], map(int, s)))

    def layer(self, k):
        m = int(lib().orc_pbc_layer_rows(self.h, k))
        x = np.zeros((m, self.W), np.uint64); z = np.zeros_like(x); r = np.zeros(m, np.uint8)
        if m: lib().orc_pbc_layer_get(self.h, k, _p(x), _p(z), _p(r))
        return x, z, r

    def mtab(self): return Tableau(self.n, _h=lib().orc_pbc_mtab(self.h), _owner=self)


def algorithmic_bytes(n: int, counters: dict, fused_layers: int | None = None) -> float:
    """layout-independent byte count of a CHP run on the bit-packed tableau.
    R = 2n rows; one column = R/8 bytes; W = ceil(n/64) words per half row."""
    R = 2 * n; col = R / 8.0; W = words_for(n)
    h = counters["gate_hist"]
    # fused-layer form: columns read+written per gate; the sign column is charged once per layer
    per_gate = {0: 4, 1: 3, 2: 3, 3: 1, 4: 2, 5: 1, 6: 6, 7: 6, 8: 8}
    b = sum(h[k] * per_gate[k] for k in per_gate) * col
    if fused_layers:
        b += fused_layers * 2 * col
    b += counters["n_rand"] * (col + 16 * W + 32 * W) + counters["k_rand"] * 32 * W
    b += counters["n_det"] * col + counters["k_det"] * 16 * W
    return b
