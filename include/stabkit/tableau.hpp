// stabkit/tableau.hpp -- CHP stabilizer/destabilizer tableau, device resident.
// Rows 0..n-1 stabilizers, n..2n-1 destabilizers; the scratch row never leaves the
// chip.  Every operation is a call into the C ABI (stabkit_b200.h); rows come back as
// PauliString values.  Single-owner during mutation.
#pragma once
#include <memory>
#include <string>
#include <vector>

#include "stabkit/circuit.hpp"
#include "stabkit/device.hpp"
#include "stabkit/pauli.hpp"
#include "stabkit/rng.hpp"

namespace stabkit {

// SPEC:119-122
struct MeasResult { bool outcome = false; bool deterministic = false; };

class Tableau {
  public:
    // SPEC:125-133; n == 0 throws DimensionError
    static Tableau new_identity(size_t n) { return Tableau(n); }
    explicit Tableau(size_t n) : n_(n) {
        Device& d = Device::instance();
        sk_tableau* t = nullptr;
        d.check(sk_tableau_create(d.ctx(), n, &t));
        h_.reset(t, [](sk_tableau* p) { sk_tableau_destroy(p); });
    }
    // adopts a handle produced by sk_sim
    Tableau(size_t n, sk_tableau* adopted) : n_(n), h_(adopted, [](sk_tableau* p) { sk_tableau_destroy(p); }) {}

    size_t num_qubits() const { return n_; }
    sk_tableau* handle() const { return h_.get(); }

    // SPEC:135-163 (row rules ref: proj/src/pauli.cpp:146-187)
    void apply_h(size_t q) { one(GateKind::H, q); }
    void apply_s(size_t q) { one(GateKind::S, q); }
    void apply_cx(size_t c, size_t t) { one(GateKind::CX, c, t); }
    // SPEC:187-195; T/TDG throw UnsupportedError, M is not a gate here
    void apply_gate(const Gate& g) {
        if (g.kind == GateKind::M) throw UnsupportedError("apply_gate: use measure_z for measurements");
        Device::instance().check(sk_apply_gates(h_.get(), reinterpret_cast<const sk_gate*>(&g), 1));
    }
    // a whole validated chunk as one fused pass over the tableau
    void apply_layer(const std::vector<Gate>& gates) {
        Device::instance().check(sk_apply_layer(h_.get(), reinterpret_cast<const sk_gate*>(gates.data()), gates.size()));
    }
    // SPEC:165-173
    void rowsum(size_t h, size_t i) { Device::instance().check(sk_tableau_rowsum(h_.get(), h, i)); }
    // SPEC:175-185; the random bit is CounterRng{seed}.bit(ordinal)
    MeasResult measure_z(size_t q, const CounterRng& rng, uint64_t ordinal) {
        uint8_t o = 0, d = 0;
        Device::instance().check(sk_measure_z(h_.get(), uint32_t(q), rng.seed, ordinal, &o, &d));
        return {o != 0, d != 0};
    }
    std::vector<MeasResult> measure_batch(const std::vector<uint32_t>& qubits, const CounterRng& rng, uint64_t ordinal0) {
        std::vector<uint8_t> o(qubits.size() + 1), d(qubits.size() + 1);
        Device::instance().check(sk_measure_batch(h_.get(), qubits.data(), qubits.size(), rng.seed, ordinal0, o.data(), d.data()));
        std::vector<MeasResult> out(qubits.size());
        for (size_t i = 0; i < qubits.size(); ++i) out[i] = {o[i] != 0, d[i] != 0};
        return out;
    }

    // all 2n rows, SPEC:110 order
    std::vector<PauliString> rows() const {
        const size_t W = words_for_bits(n_);
        std::vector<uint64_t> x(2 * n_ * W), z(2 * n_ * W); std::vector<uint8_t> s(2 * n_);
        Device::instance().check(sk_tableau_download(h_.get(), x.data(), z.data(), s.data()));
        return unpack_rows(n_, 2 * n_, x.data(), z.data(), s.data());
    }
    PauliString stabilizer(size_t i) const { return rows().at(i); }
    PauliString destabilizer(size_t i) const { return rows().at(n_ + i); }
    // SPEC:216 debug dump: "S<i>: <sign><pauli>" / "D<i>: ..."
    std::string dump() const {
        std::string out; const auto r = rows();
        for (size_t i = 0; i < 2 * n_; ++i)
            out += (i < n_ ? "S" + std::to_string(i) : "D" + std::to_string(i - n_)) + ": " + r[i].str() + "\n";
        return out;
    }

  private:
    void one(GateKind k, size_t a, size_t b = 0) { Gate g(k, uint32_t(a), uint32_t(b)); apply_gate(g); }
    size_t n_ = 0;
    std::shared_ptr<sk_tableau> h_;
};

}  // namespace stabkit
