"""stabkit-b200: ctypes plumbing over the C ABI in include/stabkit_b200.h.

This module is NOT the product; it only lets tests/ and bench.py reach the C ABI
(libstabkit_b200.so: hand-written sm_100a kernels + C++ host code).  There is no CPU
fallback: if the shared library is missing, or no CUDA device is usable, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libstabkit_b200.so")

# gate kinds (include/stabkit_b200.h, sk_gate_kind)
H, S, SDG, X, Y, Z, CX, CZ, SWAP, M, T, TDG = range(12)
KIND_NAMES = ["h", "s", "sdg", "x", "y", "z", "cx", "cz", "swap", "m", "t", "tdg"]
GATE_DTYPE = np.dtype([("kind", "u1"), ("pad", "u1", (3,)), ("q0", "<u4"), ("q1", "<u4")])
assert GATE_DTYPE.itemsize == 12

SK_OK, SK_EDIM, SK_EUNSUPPORTED, SK_EINVARIANT, SK_ECUDA, SK_ENCCL, SK_EPARSE, SK_EARG = range(8)


class StabkitError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[sk_status {code}] {msg}")
        self.code = code


class DimensionError(StabkitError): ...
class UnsupportedError(StabkitError): ...
class InvariantError(StabkitError): ...
class ParseError(StabkitError): ...
class CudaError(StabkitError): ...


_ERR = {SK_EDIM: DimensionError, SK_EUNSUPPORTED: UnsupportedError, SK_EINVARIANT: InvariantError,
        SK_EPARSE: ParseError, SK_ECUDA: CudaError}


class Counters(C.Structure):
    _fields_ = [("n_rand", C.c_uint64), ("n_det", C.c_uint64), ("k_rand", C.c_uint64), ("k_det", C.c_uint64),
                ("gate_hist", C.c_uint64 * 12), ("layers", C.c_uint64), ("waves", C.c_uint64),
                ("transposes", C.c_uint64), ("kernel_launches", C.c_uint64), ("meas_phase_ns", C.c_uint64 * 8),
                ("pred_evals", C.c_uint64), ("algorithmic_bytes", C.c_double), ("class_ms", C.c_double * 4)]


_lib = None


def lib() -> C.CDLL:
    """Load libstabkit_b200.so; raise (loudly) if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2507_03092_b200._build` "
                "(nvcc, sm_100a). There is no CPU fallback for the stabilizer hot path.")
        L = C.CDLL(LIB_PATH)
        vp, u64, u32, sz, i32 = C.c_void_p, C.c_uint64, C.c_uint32, C.c_size_t, C.c_int32
        P = C.POINTER
        sig = {
            "sk_version": (C.c_char_p, []),
            "sk_ctx_create": (i32, [C.c_int, vp, P(vp)]),
            "sk_ctx_destroy": (None, [vp]),
            "sk_last_error": (C.c_char_p, [vp]),
            "sk_ctx_stream": (vp, [vp]),
            "sk_ctx_sync": (i32, [vp]),
            "sk_get_counters": (i32, [vp, P(Counters)]),
            "sk_reset_counters": (i32, [vp]),
            "sk_tableau_create": (i32, [vp, u64, P(vp)]),
            "sk_tableau_destroy": (None, [vp]),
            "sk_tableau_reset": (i32, [vp]),
            "sk_tableau_qubits": (u64, [vp]),
            "sk_tableau_upload": (i32, [vp, vp, vp, vp]),
            "sk_tableau_download": (i32, [vp, vp, vp, vp]),
            "sk_apply_layer": (i32, [vp, vp, sz]),
            "sk_apply_gates": (i32, [vp, vp, sz]),
            "sk_measure_z": (i32, [vp, u32, u64, u64, vp, vp]),
            "sk_measure_batch": (i32, [vp, vp, sz, u64, u64, vp, vp]),
            "sk_tableau_rowsum": (i32, [vp, u64, u64]),
            "sk_program_create": (i32, [vp, u64, vp, sz, vp, sz, C.c_int, P(vp), P(u32)]),
            "sk_program_destroy": (None, [vp]),
            "sk_program_measurements": (u64, [vp]),
            "sk_program_run": (i32, [vp, vp, u64]),
            "sk_program_run_profiled": (i32, [vp, vp, u64, P(C.c_float)]),
            "sk_program_read_record": (i32, [vp, vp, vp]),
            "sk_program_run_shots": (i32, [vp, vp, u64, u64, vp, vp]),
            "sk_sim": (i32, [vp, u64, vp, sz, vp, sz, C.c_int, u64, P(vp), vp, vp, P(u32)]),
            "sk_free": (None, [vp]),
            "sk_circuit_surface_code": (i32, [u32, u32, C.c_int, P(u64), P(vp), P(sz), P(vp), P(sz)]),
            "sk_circuit_random_layered": (i32, [u64, u64, P(vp), P(sz), P(vp), P(sz)]),
            "sk_circuit_parse_native": (i32, [C.c_char_p, sz, P(u64), P(vp), P(sz), P(vp), P(sz), P(sz), C.c_char_p, sz]),
            "sk_circuit_parse_qasm2": (i32, [C.c_char_p, sz, P(u64), P(vp), P(sz), P(vp), P(sz), P(sz), C.c_char_p, sz]),
            "sk_circuit_validate_chunks": (i32, [u64, vp, sz, vp, sz, P(vp), P(vp), P(vp), P(sz)]),
            "sk_circuit_validate_chunks_ex": (i32, [u64, vp, sz, vp, sz, u32, P(vp), P(vp), P(vp), P(sz)]),
            "sk_rows_create": (i32, [vp, u64, u64, P(vp)]),
            "sk_rows_destroy": (None, [vp]),
            "sk_rows_count": (u64, [vp]),
            "sk_rows_upload": (i32, [vp, vp, vp, vp, u64]),
            "sk_rows_download": (i32, [vp, vp, vp, vp]),
            "sk_rows_append": (i32, [vp, vp, vp, vp, u64]),
            "sk_commute_matrix_tile": (i32, [vp, C.c_int, u64, u64, u64, u64, vp]),
            "sk_tableau_audit": (i32, [vp, P(u64)]),
            "sk_shard_export_words": (u64, [vp]),
            "sk_shard_export_rows": (i32, [vp, vp]),
            "sk_shard_import_rows": (i32, [vp, vp]),
            "sk_tableau_import_block": (i32, [vp, u64, u64, vp]),
            "sk_tableau_commit_blocks": (i32, [vp]),
            "sk_tableau_export_block": (i32, [vp, u64, u64, vp]),
            "sk_group_shard_create": (i32, [vp, C.c_int, u32, u32, P(vp)]),
            "sk_group_shard_destroy": (None, [vp]),
            "sk_group_shard_blocks": (u64, [vp]),
            "sk_group_shard_bitmap_words": (u64, [vp]),
            "sk_group_shard_conflicts": (i32, [vp, u64, vp]),
            "sk_group_shard_resolve": (i32, [vp, u64, vp]),
            "sk_group_shard_result": (i32, [vp, vp, P(u64)]),
            "sk_rows_conj_layer": (i32, [vp, vp, sz]),
            "sk_commutation_vector": (i32, [vp, vp, vp, vp]),
            "sk_rowsum_plus_i_where_anticommuting": (i32, [vp, vp, vp, C.c_uint8, P(u64)]),
            "sk_find_first_duplicate": (i32, [vp, P(C.c_int), P(u64), P(u64)]),
            "sk_weight_sum": (i32, [vp, P(u64)]),
            "sk_group_first_fit": (i32, [vp, C.c_int, vp, P(u64)]),
            "sk_verify_grouping": (i32, [vp, C.c_int, vp, P(u64)]),
            "sk_transpile": (i32, [vp, u64, vp, sz, P(vp)]),
            "sk_transpile_ex": (i32, [vp, u64, vp, sz, u32, P(vp)]),
            "sk_pbc_destroy": (None, [vp]),
            "sk_pbc_stats": (i32, [vp, P(u64)]),
            "sk_pbc_layer_rows": (u64, [vp, u64]),
            "sk_pbc_layer_download": (i32, [vp, u64, vp, vp, vp]),
            "sk_pbc_mtab_download": (i32, [vp, vp, vp, vp]),
            "sk_shard_create": (i32, [vp, u64, u64, u64, P(vp)]),
            "sk_shard_destroy": (None, [vp]),
            "sk_shard_reset": (i32, [vp]),
            "sk_shard_apply_gates": (i32, [vp, vp, sz]),
            "sk_shard_pivot_search": (i32, [vp, vp, sz, vp]),
            "sk_shard_partial_words": (u64, [vp]),
            "sk_shard_det_partial": (i32, [vp, vp, sz, vp]),
            "sk_shard_det_combine": (i32, [vp, vp, u32, sz, vp]),
            "sk_shard_pivot_row": (i32, [vp, u64, vp]),
            "sk_shard_random_update": (i32, [vp, u32, u64, vp, C.c_uint8]),
            "sk_shard_download": (i32, [vp, vp, vp, vp]),
            "sk_shard_counters": (i32, [vp, P(u64)]),
            "sk_dev_alloc": (i32, [vp, sz, P(vp)]),
            "sk_dev_free": (None, [vp, vp]),
            "sk_dev_copy": (i32, [vp, vp, vp, sz, C.c_int]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)      # AttributeError here == header/library mismatch: fail loudly
            fn.restype, fn.argtypes = res, args
        _lib = L
    return _lib


EXPORTS = [
    "sk_version", "sk_ctx_create", "sk_ctx_destroy", "sk_last_error", "sk_ctx_stream", "sk_ctx_sync",
    "sk_get_counters", "sk_reset_counters", "sk_tableau_create", "sk_tableau_destroy", "sk_tableau_reset",
    "sk_tableau_qubits", "sk_tableau_upload", "sk_tableau_download", "sk_apply_layer", "sk_apply_gates",
    "sk_measure_z", "sk_measure_batch", "sk_tableau_rowsum", "sk_program_create", "sk_program_destroy",
    "sk_program_measurements", "sk_program_run", "sk_program_run_profiled", "sk_program_read_record", "sk_program_run_shots", "sk_sim", "sk_free",
    "sk_circuit_surface_code", "sk_circuit_random_layered", "sk_circuit_parse_native", "sk_circuit_parse_qasm2",
    "sk_circuit_validate_chunks", "sk_circuit_validate_chunks_ex", "sk_rows_create", "sk_rows_destroy", "sk_rows_count", "sk_rows_upload",
    "sk_rows_download", "sk_rows_append", "sk_commute_matrix_tile", "sk_tableau_audit", "sk_shard_export_words", "sk_shard_export_rows", "sk_shard_import_rows",
    "sk_tableau_import_block", "sk_tableau_commit_blocks", "sk_tableau_export_block",
    "sk_group_shard_create", "sk_group_shard_destroy", "sk_group_shard_blocks", "sk_group_shard_bitmap_words", "sk_group_shard_conflicts",
    "sk_group_shard_resolve", "sk_group_shard_result", "sk_rows_conj_layer", "sk_commutation_vector",
    "sk_rowsum_plus_i_where_anticommuting", "sk_find_first_duplicate", "sk_weight_sum",
    "sk_group_first_fit", "sk_verify_grouping", "sk_transpile", "sk_transpile_ex", "sk_pbc_destroy", "sk_pbc_stats",
    "sk_pbc_layer_rows", "sk_pbc_layer_download", "sk_pbc_mtab_download",
    "sk_shard_create", "sk_shard_destroy", "sk_shard_reset", "sk_shard_apply_gates", "sk_shard_pivot_search",
    "sk_shard_partial_words", "sk_shard_det_partial", "sk_shard_det_combine", "sk_shard_pivot_row",
    "sk_shard_random_update", "sk_shard_download", "sk_shard_counters", "sk_dev_alloc", "sk_dev_free", "sk_dev_copy",
]


def words_for(n: int) -> int:
    return (n + 63) // 64


def algorithmic_bytes(n: int, counters: dict, fused_layers: float | None = None) -> float:
    """layout-independent byte count of a CHP run on the bit-packed tableau, from the device's
    counters (Context.counters(): gate histogram, n_rand / n_det, k_rand / k_det).  R = 2n rows; one column = R/8 bytes;
    W = ceil(n/64) words per half row.  Used by bench.py for the roofline line."""
    R = 2 * n; col = R / 8.0; W = words_for(n)
    h = counters["gate_hist"]
    # fused-layer form: columns read + written per gate; the sign column is charged once per layer
    per_gate = {H: 4, S: 3, SDG: 3, X: 1, Y: 2, Z: 1, CX: 6, CZ: 6, SWAP: 8}
    b = sum(h[k] * c for k, c in per_gate.items()) * col
    if fused_layers:
        b += fused_layers * 2 * col
    b += counters["n_rand"] * (col + 16 * W + 32 * W) + counters["k_rand"] * 32 * W
    b += counters["n_det"] * col + counters["k_det"] * 16 * W
    return b


def gates_array(gates) -> np.ndarray:
    """[(kind, q0[, q1]), ...] or an existing GATE_DTYPE array -> contiguous GATE_DTYPE array."""
    if isinstance(gates, np.ndarray) and gates.dtype == GATE_DTYPE:
        return np.ascontiguousarray(gates)
    out = np.zeros(len(gates), dtype=GATE_DTYPE)
    for i, g in enumerate(gates):
        out[i]["kind"] = g[0]
        out[i]["q0"] = g[1]
        out[i]["q1"] = g[2] if len(g) > 2 else 0
    return out


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _take(ptr: C.c_void_p, count: int, dtype) -> np.ndarray:
    """Copy a library-malloc'ed array into numpy and free it."""
    n = int(count)
    if n == 0 or not ptr.value:
        if ptr.value:
            lib().sk_free(ptr)
        return np.zeros(0, dtype=dtype)
    buf = (C.c_char * (n * np.dtype(dtype).itemsize)).from_address(ptr.value)
    arr = np.frombuffer(buf, dtype=dtype, count=n).copy()
    lib().sk_free(ptr)
    return arr


class Circuit:
    """Circuit IR: qubit count, GATE_DTYPE gate array, chunk marks."""

    def __init__(self, n: int, gates, chunk_marks=None):
        self.n = int(n)
        self.gates = gates_array(gates)
        self.chunk_marks = np.ascontiguousarray(np.asarray(chunk_marks if chunk_marks is not None else [], dtype=np.uint32))

    @property
    def num_measurements(self) -> int:
        if getattr(self, "_nm", None) is None:             # counted once: a pass over the gate array costs milliseconds at d=71
            self._nm = int((self.gates["kind"] == M).sum())
        return self._nm

    def emit_native(self) -> str:
        """.stab text (SPEC:273 round trip)."""
        marks = set(int(m) for m in self.chunk_marks)
        lines = [f"qubits {self.n}"]
        for i, g in enumerate(self.gates):
            if i in marks:
                lines.append("chunk")
            k = int(g["kind"])
            lines.append(f"{KIND_NAMES[k]} {int(g['q0'])}" + (f" {int(g['q1'])}" if k in (CX, CZ, SWAP) else ""))
        return "\n".join(lines) + "\n"


def _check_noctx(rc: int, what: str):
    if rc != SK_OK:
        raise _ERR.get(rc, StabkitError)(rc, what)


def surface_code_circuit(d: int, rounds: int, final_data_measure: bool = False) -> Circuit:
    L = lib()
    n, g, ng, mk, nmk = C.c_uint64(), C.c_void_p(), C.c_size_t(), C.c_void_p(), C.c_size_t()
    rc = L.sk_circuit_surface_code(d, rounds, int(final_data_measure), C.byref(n), C.byref(g), C.byref(ng), C.byref(mk), C.byref(nmk))
    _check_noctx(rc, f"surface_code_circuit(d={d}, rounds={rounds}): d must be odd >= 3, rounds >= 1 (SPEC:377)")
    return Circuit(n.value, _take(g, ng.value, GATE_DTYPE), _take(mk, nmk.value, np.uint32))


def random_layered_circuit(n: int, seed: int) -> Circuit:
    L = lib()
    g, ng, mk, nmk = C.c_void_p(), C.c_size_t(), C.c_void_p(), C.c_size_t()
    rc = L.sk_circuit_random_layered(n, seed, C.byref(g), C.byref(ng), C.byref(mk), C.byref(nmk))
    _check_noctx(rc, f"random_layered_circuit(n={n}): n must be even >= 4 (SPEC:387)")
    return Circuit(n, _take(g, ng.value, GATE_DTYPE), _take(mk, nmk.value, np.uint32))


def parse_native(text: str) -> Circuit:
    L = lib()
    raw = text.encode()
    n, g, ng, mk, nmk, line = C.c_uint64(), C.c_void_p(), C.c_size_t(), C.c_void_p(), C.c_size_t(), C.c_size_t()
    msg = C.create_string_buffer(256)
    rc = L.sk_circuit_parse_native(raw, len(raw), C.byref(n), C.byref(g), C.byref(ng), C.byref(mk), C.byref(nmk), C.byref(line), msg, 256)
    if rc == SK_EPARSE:
        e = ParseError(rc, f"line {line.value}: {msg.value.decode()}")
        e.line = line.value
        raise e
    _check_noctx(rc, "parse_native")
    return Circuit(n.value, _take(g, ng.value, GATE_DTYPE), _take(mk, nmk.value, np.uint32))


def parse_qasm2_subset(text: str) -> Circuit:
    """SPEC:252-260.  Unsupported constructs raise UnsupportedError, malformed text ParseError (both carry .line)."""
    L = lib()
    raw = text.encode()
    n, g, ng, mk, nmk, line = C.c_uint64(), C.c_void_p(), C.c_size_t(), C.c_void_p(), C.c_size_t(), C.c_size_t()
    msg = C.create_string_buffer(256)
    rc = L.sk_circuit_parse_qasm2(raw, len(raw), C.byref(n), C.byref(g), C.byref(ng), C.byref(mk), C.byref(nmk), C.byref(line), msg, 256)
    if rc in (SK_EPARSE, SK_EUNSUPPORTED):
        e = (ParseError if rc == SK_EPARSE else UnsupportedError)(rc, f"line {line.value}: {msg.value.decode()}")
        e.line = line.value
        raise e
    _check_noctx(rc, "parse_qasm2_subset")
    return Circuit(n.value, _take(g, ng.value, GATE_DTYPE), _take(mk, nmk.value, np.uint32))


def validate_chunks(c: Circuit, strict: bool = False):
    """-> list of (chunk index, gate index, kind) with kind 'collision' | 'measurement'.  Chunks that hold only
    measurements are barrier regions and are not reported; strict=True reports them too (third example)."""
    L = lib()
    vc, vg, vk, nv = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_size_t()
    rc = L.sk_circuit_validate_chunks_ex(c.n, _ptr(c.gates), len(c.gates), _ptr(c.chunk_marks), len(c.chunk_marks), 1 if strict else 0,
                                         C.byref(vc), C.byref(vg), C.byref(vk), C.byref(nv))
    _check_noctx(rc, "validate_chunks")
    a, b, k = _take(vc, nv.value, np.uint32), _take(vg, nv.value, np.uint32), _take(vk, nv.value, np.uint8)
    return [(int(x), int(y), "collision" if z == 1 else "measurement") for x, y, z in zip(a, b, k)]


class Context:
    def __init__(self, device: int = 0, stream: int | None = None):
        self._h = C.c_void_p()
        rc = lib().sk_ctx_create(device, C.c_void_p(stream) if stream else None, C.byref(self._h))
        if rc != SK_OK:
            raise CudaError(rc, f"sk_ctx_create(device={device}) failed: no usable CUDA device; there is no CPU fallback")

    def check(self, rc: int):
        if rc != SK_OK:
            msg = lib().sk_last_error(self._h).decode()
            raise _ERR.get(rc, StabkitError)(rc, msg)

    def close(self):
        if self._h:
            lib().sk_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return int(lib().sk_ctx_stream(self._h) or 0)

    def sync(self):
        self.check(lib().sk_ctx_sync(self._h))

    def counters(self) -> dict:
        c = Counters()
        self.check(lib().sk_get_counters(self._h, C.byref(c)))
        d = {k: int(getattr(c, k)) for k in ("n_rand", "n_det", "k_rand", "k_det", "layers", "waves", "transposes", "kernel_launches")}
        d["gate_hist"] = [int(v) for v in c.gate_hist]
        d["meas_phase_ns"] = [int(v) for v in c.meas_phase_ns]
        d["pred_evals"] = int(c.pred_evals); d["algorithmic_bytes"] = float(c.algorithmic_bytes); d["class_ms"] = [float(v) for v in c.class_ms]
        return d

    def reset_counters(self):
        self.check(lib().sk_reset_counters(self._h))

    def sim(self, circ: Circuit, seed: int, mode: int = 0):
        """SPEC:310-328.  -> (Tableau, outcomes u8[], deterministic u8[], warnings)."""
        nm = circ.num_measurements
        out, det = np.zeros(max(nm, 1), np.uint8), np.zeros(max(nm, 1), np.uint8)
        th, warn = C.c_void_p(), C.c_uint32()
        self.check(lib().sk_sim(self._h, circ.n, _ptr(circ.gates), len(circ.gates), _ptr(circ.chunk_marks), len(circ.chunk_marks),
                                mode, seed, C.byref(th), _ptr(out), _ptr(det), C.byref(warn)))
        return Tableau(self, circ.n, _h=th), out[:nm], det[:nm], warn.value


class Tableau:
    """Device CHP tableau."""

    def __init__(self, ctx: Context, n: int, _h=None):
        self.ctx, self.n, self.W = ctx, int(n), words_for(int(n))
        if _h is None:
            _h = C.c_void_p()
            ctx.check(lib().sk_tableau_create(ctx._h, n, C.byref(_h)))
        self._h = _h

    def close(self):
        if self._h and self.ctx._h:
            lib().sk_tableau_destroy(self._h)
        self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def audit(self) -> int:
        """sk_tableau_audit (EngineConfig.audit): row pairs that violate the CHP symplectic form; 0 = valid."""
        v = C.c_uint64(0)
        self.ctx.check(lib().sk_tableau_audit(self._h, C.byref(v)))
        return int(v.value)

    def reset(self):
        self.ctx.check(lib().sk_tableau_reset(self._h))

    def download(self):
        """-> x[2n, W] u64, z[2n, W] u64, sign[2n] u8 (row-major, SPEC:110 row order)."""
        x = np.zeros((2 * self.n, self.W), np.uint64); z = np.zeros_like(x); r = np.zeros(2 * self.n, np.uint8)
        self.ctx.check(lib().sk_tableau_download(self._h, _ptr(x), _ptr(z), _ptr(r)))
        return x, z, r

    def upload(self, x, z, r):
        x = np.ascontiguousarray(x, np.uint64); z = np.ascontiguousarray(z, np.uint64); r = np.ascontiguousarray(r, np.uint8)
        assert x.shape == (2 * self.n, self.W) and z.shape == x.shape and r.shape == (2 * self.n,)
        self.ctx.check(lib().sk_tableau_upload(self._h, _ptr(x), _ptr(z), _ptr(r)))

    def apply_layer(self, gates):
        g = gates_array(gates)
        self.ctx.check(lib().sk_apply_layer(self._h, _ptr(g), len(g)))

    def apply_gates(self, gates):
        g = gates_array(gates)
        self.ctx.check(lib().sk_apply_gates(self._h, _ptr(g), len(g)))

    def measure_z(self, q: int, seed: int, ordinal: int):
        o, d = C.c_uint8(), C.c_uint8()
        self.ctx.check(lib().sk_measure_z(self._h, q, seed, ordinal, C.byref(o), C.byref(d)))
        return o.value, d.value

    def measure_batch(self, qubits, seed: int, ordinal0: int = 0):
        q = np.ascontiguousarray(qubits, np.uint32)
        o, d = np.zeros(max(len(q), 1), np.uint8), np.zeros(max(len(q), 1), np.uint8)
        self.ctx.check(lib().sk_measure_batch(self._h, _ptr(q), len(q), seed, ordinal0, _ptr(o), _ptr(d)))
        return o[:len(q)], d[:len(q)]

    def rowsum(self, h: int, i: int):
        self.ctx.check(lib().sk_tableau_rowsum(self._h, h, i))


class Program:
    """A compiled circuit resident on the device (sk_program_*)."""

    def __init__(self, ctx: Context, circ: Circuit, mode: int = 0):
        self.ctx, self.n = ctx, circ.n
        self._h, warn = C.c_void_p(), C.c_uint32()
        ctx.check(lib().sk_program_create(ctx._h, circ.n, _ptr(circ.gates), len(circ.gates), _ptr(circ.chunk_marks),
                                          len(circ.chunk_marks), mode, C.byref(self._h), C.byref(warn)))
        self.warnings = warn.value
        self.num_measurements = int(lib().sk_program_measurements(self._h))

    def run(self, t: Tableau, seed: int):
        self.ctx.check(lib().sk_program_run(self._h, t._h, seed))

    def run_profiled(self, t: Tableau, seed: int) -> dict:
        ms = (C.c_float * 4)()
        self.ctx.check(lib().sk_program_run_profiled(self._h, t._h, seed, ms))
        return {"layer_ms": float(ms[0]), "transpose_ms": float(ms[1]), "measure_ms": float(ms[2]), "wave_ms": float(ms[3])}

    def run_shots(self, t: Tableau, shots: int, seed: int, records: bool = False):
        """SPEC:330-338.  -> (ones[nm] u32, records[shots, nm] u8 or None); shot s uses seed ^ s."""
        nm = self.num_measurements
        ones = np.zeros(max(nm, 1), np.uint32)
        rec = np.zeros((shots, max(nm, 1)), np.uint8) if records else None
        self.ctx.check(lib().sk_program_run_shots(self._h, t._h, shots, seed, _ptr(ones), _ptr(rec)))
        return ones[:nm], (rec[:, :nm] if records else None)

    def read_record(self):
        nm = self.num_measurements
        o, d = np.zeros(max(nm, 1), np.uint8), np.zeros(max(nm, 1), np.uint8)
        self.ctx.check(lib().sk_program_read_record(self._h, _ptr(o), _ptr(d)))
        return o[:nm], d[:nm]

    def close(self):
        if self._h and self.ctx._h:
            lib().sk_program_destroy(self._h)
        self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Rows:
    """Device block of signed n-qubit Pauli rows (sk_rows_*): term lists, T_tab, layers."""

    def __init__(self, ctx: Context, n: int, x=None, z=None, sign=None, capacity: int | None = None):
        self.ctx, self.n, self.W = ctx, int(n), words_for(int(n))
        m = 0 if x is None else int(np.asarray(x).reshape(-1, self.W).shape[0])
        self._h = C.c_void_p()
        ctx.check(lib().sk_rows_create(ctx._h, n, max(capacity or m, 1), C.byref(self._h)))
        if x is not None:
            self.upload(x, z, sign if sign is not None else np.zeros(m, np.uint8))

    def close(self):
        if self._h and self.ctx._h:
            lib().sk_rows_destroy(self._h)
        self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def count(self) -> int:
        return int(lib().sk_rows_count(self._h))

    def upload(self, x, z, sign):
        x = np.ascontiguousarray(x, np.uint64).reshape(-1, self.W); z = np.ascontiguousarray(z, np.uint64).reshape(-1, self.W)
        s = np.ascontiguousarray(sign, np.uint8)
        self.ctx.check(lib().sk_rows_upload(self._h, _ptr(x), _ptr(z), _ptr(s), x.shape[0]))

    def download(self):
        m = self.count
        x = np.zeros((m, self.W), np.uint64); z = np.zeros_like(x); s = np.zeros(m, np.uint8)
        if m:
            self.ctx.check(lib().sk_rows_download(self._h, _ptr(x), _ptr(z), _ptr(s)))
        return x, z, s

    def append(self, x, z, sign):
        """sk_rows_append: m more rows behind the current ones (up to the capacity given at creation)."""
        x = np.ascontiguousarray(x, np.uint64).reshape(-1, self.W); z = np.ascontiguousarray(z, np.uint64).reshape(-1, self.W)
        s = np.ascontiguousarray(sign, np.uint8)
        self.ctx.check(lib().sk_rows_append(self._h, _ptr(x), _ptr(z), _ptr(s), x.shape[0]))

    def commute_tile(self, mode: int, i0: int, ni: int, j0: int, nj: int) -> np.ndarray:
        """sk_commute_matrix_tile -> bool [ni, nj]: True where rows i0+a and j0+b conflict (mode 0: anticommute, 1: not qubit-wise commuting)."""
        words = (nj + 63) // 64
        out = np.zeros((ni, max(words, 1)), np.uint64)
        self.ctx.check(lib().sk_commute_matrix_tile(self._h, mode, i0, ni, j0, nj, _ptr(out)))
        bits = np.unpackbits(out.view(np.uint8).reshape(ni, -1), axis=1, bitorder="little")
        return bits[:, :nj].astype(bool)

    def conj_layer(self, gates):
        g = gates_array(gates)
        self.ctx.check(lib().sk_rows_conj_layer(self._h, _ptr(g), len(g)))

    def commutation_vector(self, px, pz) -> np.ndarray:
        out = np.zeros(max(1, words_for(self.count)), np.uint64)
        px = np.ascontiguousarray(px, np.uint64); pz = np.ascontiguousarray(pz, np.uint64)
        self.ctx.check(lib().sk_commutation_vector(self._h, _ptr(px), _ptr(pz), _ptr(out)))
        return out

    def rowsum_plus_i_where_anticommuting(self, px, pz, psign) -> int:
        n = C.c_uint64()
        px = np.ascontiguousarray(px, np.uint64); pz = np.ascontiguousarray(pz, np.uint64)
        self.ctx.check(lib().sk_rowsum_plus_i_where_anticommuting(self._h, _ptr(px), _ptr(pz), int(psign), C.byref(n)))
        return int(n.value)

    def find_first_duplicate(self):
        f, i, j = C.c_int(), C.c_uint64(), C.c_uint64()
        self.ctx.check(lib().sk_find_first_duplicate(self._h, C.byref(f), C.byref(i), C.byref(j)))
        return (int(i.value), int(j.value)) if f.value else None

    def weight_sum(self) -> int:
        o = C.c_uint64()
        self.ctx.check(lib().sk_weight_sum(self._h, C.byref(o)))
        return int(o.value)

    def group_first_fit(self, mode: int):
        g = np.zeros(max(1, self.count), np.uint32); ng = C.c_uint64()
        self.ctx.check(lib().sk_group_first_fit(self._h, mode, _ptr(g), C.byref(ng)))
        return g[:self.count], int(ng.value)

    def verify_grouping(self, mode: int, group_of) -> int:
        g = np.ascontiguousarray(group_of, np.uint32); nv = C.c_uint64()
        self.ctx.check(lib().sk_verify_grouping(self._h, mode, _ptr(g), C.byref(nv)))
        return int(nv.value)


class Pbc:
    """Result of sk_transpile (PbcProgram)."""

    def __init__(self, ctx: Context, circ: Circuit, exact: bool = True):
        """exact=True (default, sk_transpile): the unitary-exact form; exact=False: SK_TRANSPILE_PUBLISHED, Algorithms 2-3
        verbatim (stabkit_b200.h explains why they are not the default)."""
        self.ctx, self.n, self.W = ctx, circ.n, words_for(circ.n)
        self._h = C.c_void_p()
        ctx.check(lib().sk_transpile_ex(ctx._h, circ.n, _ptr(circ.gates), len(circ.gates), 0 if exact else 2, C.byref(self._h)))

    def close(self):
        if self._h:
            lib().sk_pbc_destroy(self._h)
        self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def stats(self) -> dict:
        s = (C.c_uint64 * 5)()
        self.ctx.check(lib().sk_pbc_stats(self._h, s))
        return dict(zip(["initial_t", "final_rotations_rowcount", "final_rotations_pauliweight", "layers", "passes"], map(int, s)))

    def layer(self, k: int):
        m = int(lib().sk_pbc_layer_rows(self._h, k))
        x = np.zeros((m, self.W), np.uint64); z = np.zeros_like(x); s = np.zeros(m, np.uint8)
        if m:
            self.ctx.check(lib().sk_pbc_layer_download(self._h, k, _ptr(x), _ptr(z), _ptr(s)))
        return x, z, s

    def mtab(self):
        x = np.zeros((2 * self.n, self.W), np.uint64); z = np.zeros_like(x); s = np.zeros(2 * self.n, np.uint8)
        self.ctx.check(lib().sk_pbc_mtab_download(self._h, _ptr(x), _ptr(z), _ptr(s)))
        return x, z, s
