// stabkit/circuit.hpp -- circuit IR, native .stab text format, chunk validation, generators.
// SPEC:226-292 (circuit_io) and SPEC:364-416 (qec_gen); the reference ships these as
// specification only.  Host logic lives behind the C ABI (csrc/circuit_host.cpp).
#pragma once
#include <cstdint>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "stabkit/error.hpp"
#include "stabkit_b200.h"

namespace stabkit {

enum class GateKind : uint8_t { H = SK_H, S = SK_S, SDG = SK_SDG, X = SK_X, Y = SK_Y, Z = SK_Z, CX = SK_CX, CZ = SK_CZ, SWAP = SK_SWAP, M = SK_M, T = SK_T, TDG = SK_TDG };

// SPEC:231-234.  Layout-compatible with sk_gate so a gate vector crosses the C ABI without copying.
struct Gate {
    GateKind kind = GateKind::H;
    uint8_t pad_[3] = {0, 0, 0};
    uint32_t q0 = 0, q1 = 0;
    Gate() = default;
    Gate(GateKind k, uint32_t a, uint32_t b = 0) : kind(k), q0(a), q1(b) {}
    bool two_qubit() const { return kind == GateKind::CX || kind == GateKind::CZ || kind == GateKind::SWAP; }
    bool operator==(const Gate& o) const { return kind == o.kind && q0 == o.q0 && q1 == o.q1; }
};
static_assert(sizeof(Gate) == sizeof(sk_gate), "Gate must match sk_gate");

// SPEC:236-239
struct Circuit {
    uint64_t n = 0;
    std::vector<Gate> gates;
    std::vector<uint32_t> chunk_marks;
    size_t num_measurements() const { size_t m = 0; for (const Gate& g : gates) m += g.kind == GateKind::M; return m; }
    const sk_gate* raw() const { return reinterpret_cast<const sk_gate*>(gates.data()); }
};

struct ChunkViolation { uint32_t chunk, gate; bool collision, measurement; };

namespace detail {
inline Circuit take_circuit(uint64_t n, sk_gate* g, size_t ng, uint32_t* marks, size_t nm) {
    Circuit c; c.n = n;
    c.gates.resize(ng);
    for (size_t i = 0; i < ng; ++i) c.gates[i] = Gate(static_cast<GateKind>(g[i].kind), g[i].q0, g[i].q1);
    c.chunk_marks.assign(marks, marks + nm);
    sk_free(g); sk_free(marks);
    return c;
}
}  // namespace detail

// SPEC:242-250.  Throws ParseError carrying the 1-based line.
inline Circuit parse_native(std::string_view text) {
    uint64_t n = 0; sk_gate* g = nullptr; size_t ng = 0; uint32_t* marks = nullptr; size_t nm = 0, line = 0;
    char msg[256] = {0};
    const int rc = sk_circuit_parse_native(text.data(), text.size(), &n, &g, &ng, &marks, &nm, &line, msg, sizeof msg);
    if (rc == SK_EPARSE) throw ParseError(line, msg);
    if (rc != SK_OK) throw Error("parse_native failed");
    return detail::take_circuit(n, g, ng, marks, nm);
}

// SPEC:252-260
inline Circuit parse_qasm2_subset(std::string_view text) {
    uint64_t n = 0; sk_gate* g = nullptr; size_t ng = 0, nm = 0, line = 0; uint32_t* marks = nullptr; char msg[256] = {0};
    const int rc = sk_circuit_parse_qasm2(text.data(), text.size(), &n, &g, &ng, &marks, &nm, &line, msg, sizeof msg);
    if (rc == SK_EPARSE) throw ParseError(line, msg);
    if (rc == SK_EUNSUPPORTED) throw UnsupportedError(msg);
    if (rc != SK_OK) throw Error("parse_qasm2_subset failed");
    return detail::take_circuit(n, g, ng, marks, nm);
}

// inverse of parse_native
inline std::string emit_native(const Circuit& c) {
    static const char* names[] = {"h", "s", "sdg", "x", "y", "z", "cx", "cz", "swap", "m", "t", "tdg"};
    std::string out = "qubits " + std::to_string(c.n) + "\n";
    size_t next_mark = 0;
    for (size_t i = 0; i < c.gates.size(); ++i) {
        if (next_mark < c.chunk_marks.size() && c.chunk_marks[next_mark] == i) { out += "chunk\n"; ++next_mark; }
        const Gate& g = c.gates[i];
        out += names[static_cast<int>(g.kind)];
        out += " " + std::to_string(g.q0);
        if (g.two_qubit()) out += " " + std::to_string(g.q1);
        out += "\n";
    }
    return out;
}

// SPEC:262-270.  Measurement-only chunks are barrier regions and are not reported; strict = true reports them
// too (third example).
inline std::vector<ChunkViolation> validate_chunks(const Circuit& c, bool strict = false) {
    uint32_t *vc = nullptr, *vg = nullptr; uint8_t* vk = nullptr; size_t nv = 0;
    const int rc = sk_circuit_validate_chunks_ex(c.n, c.raw(), c.gates.size(), c.chunk_marks.data(), c.chunk_marks.size(),
                                                 strict ? SK_CHUNKS_STRICT : 0u, &vc, &vg, &vk, &nv);
    if (rc == SK_EDIM) throw DimensionError("validate_chunks: gate qubit out of range");
    if (rc != SK_OK) throw Error("validate_chunks failed");
    std::vector<ChunkViolation> out(nv);
    for (size_t i = 0; i < nv; ++i) out[i] = {vc[i], vg[i], vk[i] == 1, vk[i] == 2};
    sk_free(vc); sk_free(vg); sk_free(vk);
    return out;
}

// SPEC:375-383.  final_data_measure appends `m` on the d*d data qubits (BASELINE configs 1-3).
inline Circuit surface_code_circuit(uint32_t d, uint32_t rounds, bool final_data_measure = false) {
    uint64_t n = 0; sk_gate* g = nullptr; size_t ng = 0; uint32_t* marks = nullptr; size_t nm = 0;
    if (sk_circuit_surface_code(d, rounds, final_data_measure, &n, &g, &ng, &marks, &nm) != SK_OK)
        throw Error("surface_code_circuit: distance must be odd and >= 3, rounds >= 1 (SPEC:377-379)");
    return detail::take_circuit(n, g, ng, marks, nm);
}
// SPEC:385-393
inline Circuit random_layered_circuit(uint64_t n, uint64_t seed) {
    sk_gate* g = nullptr; size_t ng = 0; uint32_t* marks = nullptr; size_t nm = 0;
    if (sk_circuit_random_layered(n, seed, &g, &ng, &marks, &nm) != SK_OK)
        throw Error("random_layered_circuit: qubit count must be even and >= 4 (SPEC:387-389)");
    return detail::take_circuit(n, g, ng, marks, nm);
}

}  // namespace stabkit
