// stabkit/pbc.hpp -- Clifford+T -> Pauli-based-computing transpiler (Algorithms 2-4).
// build_tableaus / t_separate / t_optimize run on the device inside sk_transpile.
#pragma once
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
// exact = true selects SK_TRANSPILE_EXACT (inverse-gate backward walk + order-preserving separation: the variant that
// passes the dense-statevector equivalence check of SPEC:563-573); false keeps Algorithms 2-3 as published.
inline PbcProgram transpile(const Circuit& c, bool exact = false) {
    Device& dev = Device::instance();
    sk_pbc* p = nullptr;
    dev.check(sk_transpile_ex(dev.ctx(), c.n, c.raw(), c.gates.size(), exact ? SK_TRANSPILE_EXACT : 0u, &p));
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

}  // namespace stabkit
