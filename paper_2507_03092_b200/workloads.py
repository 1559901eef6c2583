"""Synthetic inputs of the BASELINE configs C4 and C5 exactly as SURVEY.md section 8d defines them (the surface-code
configs C1-C3 come from `surface_code_circuit`).  Pure numpy: the generator is the reference's sequential SplitMix64
(proj/include/stabkit/rng.hpp:42-65), restated in vector form -- output k is mix(seed + (k+1) * golden) -- so a million
draws cost milliseconds.  tests/test_host_logic.py pins the stream against the compiled reference."""
from __future__ import annotations

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)


def splitmix_stream(seed: int, count: int) -> np.ndarray:
    """The first `count` outputs of SplitMix64(seed).next() (rng.hpp:46-52)."""
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + _GOLDEN * np.arange(1, count + 1, dtype=np.uint64)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def unit(v: np.ndarray) -> np.ndarray:
    """SplitMix64::unit (rng.hpp:61-63): uniform double in [0, 1)."""
    return (v >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def c4_terms(N: int, seed: int = 20250703):
    """C4: N random Pauli strings on 128 qubits with coefficients: per term x0, x1, z0, z1 = next() x 4,
    coeff = 2 * unit() - 1; sorted by |coeff| descending, ties by input order.  A term that is all identity
    or has coefficient 0 would be redrawn (probability 2^-256 / 2^-53: asserted absent instead).
    -> (x [N, 2] u64, z [N, 2] u64, coeff [N] f64), already in first-fit order."""
    v = splitmix_stream(seed, 5 * N).reshape(N, 5)
    x = np.ascontiguousarray(v[:, 0:2]); z = np.ascontiguousarray(v[:, 2:4])
    coeff = 2.0 * unit(v[:, 4]) - 1.0
    assert ((x | z).any(axis=1)).all() and (coeff != 0).all()
    order = np.argsort(-np.abs(coeff), kind="stable")
    return np.ascontiguousarray(x[order]), np.ascontiguousarray(z[order]), coeff[order]


def c5_gates(n: int = 1000, G: int = 100_000, seed: int = 20250704, gate_dtype=None, kinds=None) -> np.ndarray:
    """C5: random Clifford+T circuit: per gate u = unit(): u < 0.05 t q | < 0.10 tdg q | < 0.40 h q | < 0.70 s q | else
    cx c t, with q, c = below(n) and t redrawn until != c.  Sequential draws (the redraw makes the stream data dependent)."""
    H, S, CX, T, TDG = kinds
    raw = splitmix_stream(seed, 4 * G + 64)
    gates = np.zeros(G, gate_dtype)
    k = 0
    rawl = raw.tolist()
    kind = np.zeros(G, np.uint8); q0 = np.zeros(G, np.uint32); q1 = np.zeros(G, np.uint32)
    for i in range(G):
        u = (rawl[k] >> 11) * 2.0 ** -53; k += 1
        if u < 0.70:
            kind[i] = T if u < 0.05 else TDG if u < 0.10 else H if u < 0.40 else S
            q0[i] = rawl[k] % n; k += 1
        else:
            c = rawl[k] % n; k += 1
            t = rawl[k] % n; k += 1
            while t == c:
                t = rawl[k] % n; k += 1
            kind[i] = CX; q0[i] = c; q1[i] = t
    gates["kind"] = kind; gates["q0"] = q0; gates["q1"] = q1
    return gates
