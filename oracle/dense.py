"""TEST INFRASTRUCTURE ONLY -- dense statevector oracle (SPEC.md [MODULE] oracle, lines 606-676; n <= 12).

An INDEPENDENT pin of the sign conventions the reference ships only as prose: nothing here knows about
tableaux.  tests/test_oracle_dense.py uses it to check, by physics,
  * the CHP restatement (oracle/stab_oracle.cpp): after any Clifford circuit with measurements every stabilizer
    row has expectation +1 on the dense state, deterministic outcomes have probability 1 and random ones 1/2
    ("Clifford-gate action agrees with the tableau module on stabilizer expectation values");
  * the transpiler restatement: verify_transpile -- the Z-outcome distribution of the circuit
    equals the joint outcome distribution of measurement_rows after the pi/8 Pauli rotations, TV < 1e-9.
Never imported by the product.
"""
from __future__ import annotations

import numpy as np

H, S, SDG, X, Y, Z, CX, CZ, SWAP, M, T, TDG = range(12)
MAX_QUBITS = 12


def zero_state(n: int) -> np.ndarray:
    if n > MAX_QUBITS:
        raise ValueError(f"n={n} over the dense oracle limit {MAX_QUBITS} (SPEC:659)")
    s = np.zeros(1 << n, np.complex128); s[0] = 1.0
    return s


def _idx(n):
    return np.arange(1 << n)


_PAR = np.array([bin(v).count("1") & 1 for v in range(1 << MAX_QUBITS)], np.int8)


def pauli_apply(state: np.ndarray, n: int, x: int, z: int, sign: int) -> np.ndarray:
    """P|psi> for P = (-1)^sign * prod_q {I,X,Y,Z}; bit q of x/z as in pauli.hpp:28-31 (Y = iXZ)."""
    b = _idx(n)
    ph = np.where(_PAR[b & z] == 1, -1.0, 1.0).astype(np.complex128)
    ph *= (1j) ** (bin(x & z).count("1") % 4)
    if sign:
        ph = -ph
    out = np.zeros_like(state)
    out[b ^ x] = ph * state[b]
    return out


def pauli_rotation(state, n, x, z, sign, angle):
    """exp(-i * angle * P) |psi>."""
    return np.cos(angle) * state - 1j * np.sin(angle) * pauli_apply(state, n, x, z, sign)


def expectation(state, n, x, z, sign) -> float:
    return float(np.real(np.vdot(state, pauli_apply(state, n, x, z, sign))))


def apply_gate(state, n, kind, a, b=0):
    """standard unitary action."""
    i = _idx(n)
    ba = (i >> a) & 1
    if kind == H:
        out = np.zeros_like(state)
        lo = i[ba == 0]
        s0, s1 = state[lo], state[lo | (1 << a)]
        out[lo] = (s0 + s1) / np.sqrt(2); out[lo | (1 << a)] = (s0 - s1) / np.sqrt(2)
        return out
    if kind in (S, SDG, Z, T, TDG):
        ph = {S: 1j, SDG: -1j, Z: -1.0, T: np.exp(1j * np.pi / 4), TDG: np.exp(-1j * np.pi / 4)}[kind]
        return np.where(ba == 1, ph * state, state)
    if kind == X:
        return state[i ^ (1 << a)]
    if kind == Y:                      # Y|0> = i|1>, Y|1> = -i|0>
        src = i ^ (1 << a)
        return np.where(ba == 1, 1j, -1j) * state[src]
    bb = (i >> b) & 1
    if kind == CX:                     # a control, b target
        return state[np.where(ba == 1, i ^ (1 << b), i)]
    if kind == CZ:
        return np.where((ba & bb) == 1, -state, state)
    if kind == SWAP:
        return state[np.where(ba != bb, i ^ (1 << a) ^ (1 << b), i)]
    raise ValueError(f"gate kind {kind}")


def measure_z_forced(state, n, q, outcome):
    """Projects on Z_q = (-1)^outcome; returns (probability of that outcome, normalised post-state)."""
    mask = ((_idx(n) >> q) & 1) == outcome
    p = float(np.sum(np.abs(state[mask]) ** 2))
    out = np.where(mask, state, 0)
    return p, (out / np.sqrt(p) if p > 1e-15 else out)


def z_distribution(state):
    return np.abs(state) ** 2


def pauli_distribution(state, n, rows):
    """Joint outcome distribution of pairwise-commuting Hermitian rows [(x, z, sign), ...] by sequential projection
    P_+- = (I +- P)/2; outcome bit 1 = eigenvalue -1; bit k of the index = row k."""
    dist = np.zeros(1 << len(rows))

    def rec(st, k, idx):
        if float(np.vdot(st, st).real) < 1e-18:
            return
        if k == len(rows):
            dist[idx] += float(np.vdot(st, st).real); return
        x, z, sg = rows[k]
        ps = pauli_apply(st, n, x, z, sg)
        rec((st + ps) / 2, k + 1, idx)
        rec((st - ps) / 2, k + 1, idx | (1 << k))

    rec(state, 0, 0)
    return dist


def run_circuit(n, gates):
    """Unitary part of a circuit (no M) on |0..0>."""
    st = zero_state(n)
    for k, a, b in gates:
        st = apply_gate(st, n, int(k), int(a), int(b))
    return st


def verify_transpile(n, gates, layers, measurement_rows):
    """SPEC:563-573.  gates: Clifford+T without measurements (every qubit measured in Z at the end);
    layers: [[(x, z, sign), ...], ...] each row a rotation exp(-i pi/8 (-1)^sign P), applied in order;
    measurement_rows: n rows, row q <-> original Z_q.  -> total-variation distance of the two distributions."""
    a = z_distribution(run_circuit(n, gates))
    st = zero_state(n)
    for layer in layers:
        for x, z, sg in layer:
            st = pauli_rotation(st, n, x, z, sg, np.pi / 8)
    b = pauli_distribution(st, n, measurement_rows)
    return 0.5 * float(np.sum(np.abs(a - b)))
