// stabkit/pbc.hpp -- Clifford+T -> Pauli-based-computing transpiler (Algorithms 2-4).
// build_tableaus / t_separate / t_optimize run on the device inside sk_transpile.
#pragma once
#include <sstream>
#include <string>
#include <vector>

#include "stabkit/circuit.hpp"
#include "stabkit/device.hpp"
#include "stabkit/pauli.hpp"

namespace stabkit {

struct PbcStats { uint64_t initial_t = 0, final_rotations_rowcount = 0, final_rotations_pauliweight = 0, layers = 0, passes = 0; };

// SPEC:509-512
struct PbcProgram {
    size_t n = 0;
    std::vector<std::vector<PauliString>> layers;     // forward time order; sign = T (false) / T-dagger (true)
    std::vector<PauliString> measurement_rows;        // the n stabilizer rows of the final M_tab
    std::vector<PauliString> destabilizer_rows;       // its destabilizers (kept for parity checks)
    PbcStats stats;
};

// SPEC:545-553.  Mid-circuit measurement throws UnsupportedError.
// The default is the unitary-exact form (inverse-gate backward walk + order-preserving separation: the one that passes the
// dense-statevector equivalence check SPEC:563-573 names as arbiter); published = true selects Algorithms 2-3 verbatim
// (SK_TRANSPILE_PUBLISHED), which are not unitarily equivalent in general -- see include/stabkit_b200.h.
inline PbcProgram transpile(const Circuit& c, bool published = false) {
    Device& dev = Device::instance();
    sk_pbc* p = nullptr;
    dev.check(sk_transpile_ex(dev.ctx(), c.n, c.raw(), c.gates.size(), published ? SK_TRANSPILE_PUBLISHED : 0u, &p));
    PbcProgram out; out.n = c.n;
    uint64_t st[5];
    sk_pbc_stats(p, st);
    out.stats = {st[0], st[1], st[2], st[3], st[4]};
    const size_t W = words_for_bits(c.n);
    for (uint64_t k = 0; k < st[3]; ++k) {
        const size_t m = sk_pbc_layer_rows(p, k);
        std::vector<uint64_t> x(m * W), z(m * W); std::vector<uint8_t> s(m);
        sk_pbc_layer_download(p, k, x.data(), z.data(), s.data());
        out.layers.push_back(unpack_rows(c.n, m, x.data(), z.data(), s.data()));
    }
    std::vector<uint64_t> x(2 * c.n * W), z(2 * c.n * W); std::vector<uint8_t> s(2 * c.n);
    sk_pbc_mtab_download(p, x.data(), z.data(), s.data());
    auto rows = unpack_rows(c.n, 2 * c.n, x.data(), z.data(), s.data());
    out.measurement_rows.assign(rows.begin(), rows.begin() + c.n);
    out.destabilizer_rows.assign(rows.begin() + c.n, rows.end());
    sk_pbc_destroy(p);
    return out;
}

// SPEC:555-561 emit_pbc: `PBC v1` / `qubits <n>` / `t_initial <k>` / `t_final <k'>`, `layer <i>:` blocks with one signed Pauli
// per line, then a `measure:` block with one signed Pauli per original qubit index.  Host-only text plumbing.
inline std::string emit_pbc(const PbcProgram& p) {
    std::ostringstream o;
    o << "PBC v1\nqubits " << p.n << "\nt_initial " << p.stats.initial_t << "\nt_final " << p.stats.final_rotations_rowcount << "\n";
    for (size_t i = 0; i < p.layers.size(); ++i) {
        o << "layer " << i << ":\n";
        for (const PauliString& r : p.layers[i]) o << r.str() << "\n";
    }
    o << "measure:\n";
    for (const PauliString& r : p.measurement_rows) o << r.str() << "\n";
    return o.str();
}
// inverse of emit_pbc (SPEC:561 round trip).  Throws ParseError with the 1-based line.
inline PbcProgram parse_pbc(std::string_view text) {
    PbcProgram p;
    std::istringstream in{std::string(text)};
    std::string line; size_t ln = 0; int section = 0;          // 0 header, 1 inside a layer, 2 measure block
    bool have_n = false;
    auto fail = [&](const std::string& what) -> void { throw ParseError(ln, what); };
    auto number = [&](const std::string& s) -> uint64_t {
        if (s.empty() || s.size() > 18) fail("expected a number");
        uint64_t v = 0; for (char c : s) { if (c < '0' || c > '9') fail("expected a number"); v = v * 10 + uint64_t(c - '0'); }
        return v;
    };
    while (std::getline(in, line)) {
        ++ln;
        while (!line.empty() && (line.back() == '\r' || line.back() == ' ')) line.pop_back();
        if (line.empty()) continue;
        if (ln == 1) { if (line != "PBC v1") fail("expected header 'PBC v1'"); continue; }
        if (line.rfind("qubits ", 0) == 0) { p.n = size_t(number(line.substr(7))); have_n = true; continue; }
        if (line.rfind("t_initial ", 0) == 0) { p.stats.initial_t = number(line.substr(10)); continue; }
        if (line.rfind("t_final ", 0) == 0) { p.stats.final_rotations_rowcount = number(line.substr(8)); continue; }
        if (line.rfind("layer ", 0) == 0 && line.back() == ':') {
            if (number(line.substr(6, line.size() - 7)) != p.layers.size()) fail("layers must be numbered consecutively from 0");
            p.layers.emplace_back(); section = 1; continue;
        }
        if (line == "measure:") { section = 2; continue; }
        if (!have_n || section == 0) fail("Pauli row outside a 'layer <i>:' or 'measure:' block");
        PauliString r = PauliString::parse(line);
        if (r.num_qubits() != p.n) fail("Pauli row has " + std::to_string(r.num_qubits()) + " qubits, expected " + std::to_string(p.n));
        (section == 1 ? p.layers.back() : p.measurement_rows).push_back(std::move(r));
    }
    if (!have_n) { ln = 0; fail("missing 'qubits <n>'"); }
    if (p.measurement_rows.size() != p.n) fail("the measure block needs one row per qubit");
    p.stats.layers = p.layers.size();
    for (const auto& L : p.layers) for (const PauliString& r : L) p.stats.final_rotations_pauliweight += r.weight();
    return p;
}

}  // namespace stabkit
