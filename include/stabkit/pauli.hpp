// stabkit/pauli.hpp -- signed n-qubit Pauli operator in binary symplectic form.
// Public API identical to the reference class (ref: proj/include/stabkit/pauli.hpp:32-123):
// same member and free-function names, argument meaning and error behaviour.  Single-operator
// arithmetic is host code (it is the value type that travels across the API); everything that
// sweeps MANY rows -- commutation_vector over a span, tableau updates, grouping, the Clifford+T
// pass -- runs on the device through the C ABI (stabkit_b200.h).
// Encoding per qubit: I=(0,0) X=(1,0) Z=(0,1) Y=(1,1); sign true == -1; padding bits zero.
#pragma once
#include <bit>
#include <cstdint>
#include <span>
#include <string>
#include <string_view>
#include <vector>

#include "stabkit/bitvec.hpp"
#include "stabkit/device.hpp"
#include "stabkit/error.hpp"

namespace stabkit {

class PauliString {
  public:
    PauliString() = default;
    explicit PauliString(size_t n) : n_(n), x_(words_for_bits(n), 0), z_(words_for_bits(n), 0) {}

    // "[+|-]?[IXYZ]+", leftmost character = qubit 0 (ref: proj/src/pauli.cpp:26-57)
    static PauliString parse(std::string_view text) {
        size_t at = 0; bool negative = false;
        if (!text.empty() && (text.front() == '+' || text.front() == '-')) { negative = text.front() == '-'; at = 1; }
        if (at == text.size()) throw ParseError(0, "empty Pauli string");
        PauliString out(text.size() - at);
        out.sign_ = negative;
        for (size_t q = 0; at < text.size(); ++at, ++q) {
            const char c = text[at];
            if (c == 'I') continue;
            if (c == 'X') out.set_pauli(q, true, false);
            else if (c == 'Y') out.set_pauli(q, true, true);
            else if (c == 'Z') out.set_pauli(q, false, true);
            else throw ParseError(0, std::string("invalid Pauli character '") + c + "' at position " + std::to_string(at + 1));
        }
        return out;
    }
    static PauliString z_at(size_t n, size_t q) { PauliString p(n); p.set_pauli(q, false, true); return p; }
    static PauliString x_at(size_t n, size_t q) { PauliString p(n); p.set_pauli(q, true, false); return p; }

    size_t num_qubits() const { return n_; }
    bool sign() const { return sign_; }
    void set_sign(bool s) { sign_ = s; }
    void flip_sign() { sign_ = !sign_; }

    bool x_bit(size_t q) const { return ((x_[q / 64] >> (q % 64)) & 1u) != 0; }
    bool z_bit(size_t q) const { return ((z_[q / 64] >> (q % 64)) & 1u) != 0; }
    void set_pauli(size_t q, bool x, bool z) {
        require_qubit(q);
        const uint64_t bit = uint64_t{1} << (q % 64);
        x_[q / 64] = x ? (x_[q / 64] | bit) : (x_[q / 64] & ~bit);
        z_[q / 64] = z ? (z_[q / 64] | bit) : (z_[q / 64] & ~bit);
    }
    char pauli_at(size_t q) const { require_qubit(q); return "IXZY"[int(x_bit(q)) + 2 * int(z_bit(q))]; }
    std::string str() const {
        std::string s(1, sign_ ? '-' : '+');
        for (size_t q = 0; q < n_; ++q) s.push_back(pauli_at(q));
        return s;
    }
    size_t weight() const {
        size_t total = 0;
        for (size_t w = 0; w < x_.size(); ++w) total += size_t(std::popcount(x_[w] | z_[w]));
        return total;
    }
    bool is_identity() const {
        uint64_t any = 0;
        for (size_t w = 0; w < x_.size(); ++w) any |= x_[w] | z_[w];
        return any == 0;
    }
    // group-wise: even number of anticommuting positions (ref: proj/src/pauli.cpp:117-127)
    bool commutes_with(const PauliString& o) const {
        same_length(o);
        int parity = 0;
        for (size_t w = 0; w < x_.size(); ++w) parity ^= std::popcount((x_[w] & o.z_[w]) ^ (o.x_[w] & z_[w]));
        return (parity & 1) == 0;
    }
    // qubit-wise: commute at every position (ref: proj/src/pauli.cpp:129-140)
    bool qubitwise_commutes_with(const PauliString& o) const {
        same_length(o);
        uint64_t any = 0;
        for (size_t w = 0; w < x_.size(); ++w) any |= (x_[w] & o.z_[w]) ^ (o.x_[w] & z_[w]);
        return any == 0;
    }
    bool same_axis(const PauliString& o) const { return n_ == o.n_ && x_ == o.x_ && z_ == o.z_; }
    bool operator==(const PauliString&) const = default;

    // conjugation by one Clifford generator (tableau row rules, ref: proj/src/pauli.cpp:146-187)
    void conj_h(size_t q) {
        require_qubit(q);
        const bool x = x_bit(q), z = z_bit(q);
        sign_ ^= (x && z);
        set_pauli(q, z, x);
    }
    void conj_s(size_t q) {
        require_qubit(q);
        const bool x = x_bit(q), z = z_bit(q);
        sign_ ^= (x && z);
        set_pauli(q, x, z != x);
    }
    void conj_sdg(size_t q) {
        require_qubit(q);
        const bool x = x_bit(q), z = z_bit(q);
        sign_ ^= (x && !z);
        set_pauli(q, x, z != x);
    }
    void conj_cx(size_t c, size_t t) {
        require_qubit(c); require_qubit(t);
        const bool xc = x_bit(c), zc = z_bit(c), xt = x_bit(t), zt = z_bit(t);
        sign_ ^= (xc && zt && (xt == zc));
        set_pauli(t, xt != xc, zt);
        set_pauli(c, x_bit(c), zc != zt);
    }

    const std::vector<uint64_t>& x_words() const { return x_; }
    const std::vector<uint64_t>& z_words() const { return z_; }
    std::vector<uint64_t>& x_words() { return x_; }
    std::vector<uint64_t>& z_words() { return z_; }

  private:
    void require_qubit(size_t q) const {
        if (q >= n_) throw DimensionError("qubit index " + std::to_string(q) + " out of range for " + std::to_string(n_) + " qubits");
    }
    void same_length(const PauliString& o) const {
        if (o.n_ != n_) throw DimensionError("Pauli length mismatch: " + std::to_string(n_) + " vs " + std::to_string(o.n_));
    }
    size_t n_ = 0;
    bool sign_ = false;
    std::vector<uint64_t> x_, z_;
};

// i-exponent sum of a*b over raw words, a the left factor (ref: proj/src/pauli.cpp:189-205).
inline int64_t product_g_sum(const uint64_t* xa, const uint64_t* za, const uint64_t* xb, const uint64_t* zb, size_t nwords) {
    int64_t total = 0;
    for (size_t w = 0; w < nwords; ++w) {
        const uint64_t aX = xa[w] & ~za[w], aY = xa[w] & za[w], aZ = ~xa[w] & za[w];
        const uint64_t bX = xb[w] & ~zb[w], bY = xb[w] & zb[w], bZ = ~xb[w] & zb[w];
        total += std::popcount((aX & bY) | (aY & bZ) | (aZ & bX));
        total -= std::popcount((aX & bZ) | (aY & bX) | (aZ & bY));
    }
    return total;
}
inline int64_t product_g_sum(const PauliString& a, const PauliString& b) {
    if (a.num_qubits() != b.num_qubits()) throw DimensionError("Pauli length mismatch in product");
    return product_g_sum(a.x_words().data(), a.z_words().data(), b.x_words().data(), b.z_words().data(), a.x_words().size());
}

// target := i * pushed * target for anticommuting operands (ref: proj/src/pauli.cpp:239-254)
inline void rowsum_plus_i(PauliString& target, const PauliString& pushed) {
    const int64_t sum = 2 * int64_t(target.sign()) + 2 * int64_t(pushed.sign()) + product_g_sum(pushed, target) + 1;
    const int64_t mod = ((sum % 4) + 4) % 4;
    if (mod == 1 || mod == 3) throw InvariantError("rowsum+i on commuting rows produced a non-Hermitian product");
    target.set_sign(mod == 2);
    for (size_t w = 0; w < target.x_words().size(); ++w) {
        target.x_words()[w] ^= pushed.x_words()[w];
        target.z_words()[w] ^= pushed.z_words()[w];
    }
}

// pack a span of rows into row-major word arrays (host ABI of stabkit_b200.h)
inline void pack_rows(std::span<const PauliString> rows, size_t n, std::vector<uint64_t>& x, std::vector<uint64_t>& z, std::vector<uint8_t>& s) {
    const size_t W = words_for_bits(n);
    x.assign(rows.size() * W, 0); z.assign(rows.size() * W, 0); s.assign(rows.size(), 0);
    for (size_t i = 0; i < rows.size(); ++i) {
        if (rows[i].num_qubits() != n)
            throw DimensionError("row " + std::to_string(i) + " has length " + std::to_string(rows[i].num_qubits()) + ", expected " + std::to_string(n));
        for (size_t w = 0; w < W; ++w) { x[i * W + w] = rows[i].x_words()[w]; z[i * W + w] = rows[i].z_words()[w]; }
        s[i] = rows[i].sign();
    }
}
inline std::vector<PauliString> unpack_rows(size_t n, size_t m, const uint64_t* x, const uint64_t* z, const uint8_t* s) {
    const size_t W = words_for_bits(n);
    std::vector<PauliString> out(m, PauliString(n));
    for (size_t i = 0; i < m; ++i) {
        for (size_t w = 0; w < W; ++w) { out[i].x_words()[w] = x[i * W + w]; out[i].z_words()[w] = z[i * W + w]; }
        out[i].set_sign(s[i] != 0);
    }
    return out;
}

// bit i set iff p anticommutes with rows[i] (ref: proj/src/pauli.cpp:215-237).  Device kernel
// k_commutation_vector through sk_commutation_vector; throws Error when no GPU is usable.
inline BitVec commutation_vector(const PauliString& p, std::span<const PauliString> rows) {
    BitVec out(rows.size());
    if (rows.empty()) return out;
    std::vector<uint64_t> x, z; std::vector<uint8_t> s;
    pack_rows(rows, p.num_qubits(), x, z, s);
    Device& dev = Device::instance();
    sk_rows* r = nullptr;
    dev.check(sk_rows_create(dev.ctx(), p.num_qubits(), rows.size(), &r));
    int rc = sk_rows_upload(r, x.data(), z.data(), s.data(), rows.size());
    if (!rc) rc = sk_commutation_vector(r, p.x_words().data(), p.z_words().data(), out.words.data());
    const std::string msg = rc ? sk_last_error(dev.ctx()) : "";
    sk_rows_destroy(r);
    if (rc) throw_status(rc, msg);
    return out;
}

// A row set that stays on the device: upload once, then any number of commutation_vector calls (Algorithm 3 asks for one per
// rotation: the free function above re-uploads the rows every time).  append() grows it within the capacity given up front.
class DeviceRows {
  public:
    DeviceRows(size_t n, std::span<const PauliString> rows, size_t capacity = 0) : n_(n) {
        Device& dev = Device::instance();
        dev.check(sk_rows_create(dev.ctx(), n, std::max(capacity, rows.size()), &r_));
        std::vector<uint64_t> x, z; std::vector<uint8_t> s;
        pack_rows(rows, n, x, z, s);
        const int rc = rows.empty() ? 0 : sk_rows_upload(r_, x.data(), z.data(), s.data(), rows.size());
        if (rc) { const std::string msg = sk_last_error(dev.ctx()); sk_rows_destroy(r_); r_ = nullptr; throw_status(rc, msg); }
    }
    ~DeviceRows() { if (r_) sk_rows_destroy(r_); }
    DeviceRows(const DeviceRows&) = delete;
    DeviceRows& operator=(const DeviceRows&) = delete;
    size_t size() const { return size_t(sk_rows_count(r_)); }
    void append(std::span<const PauliString> rows) {
        std::vector<uint64_t> x, z; std::vector<uint8_t> s;
        pack_rows(rows, n_, x, z, s);
        Device::instance().check(sk_rows_append(r_, x.data(), z.data(), s.data(), rows.size()));
    }
    // ref: proj/src/pauli.cpp:215-237
    BitVec commutation_vector(const PauliString& p) const {
        if (p.num_qubits() != n_) throw DimensionError("commutation_vector: Pauli has length " + std::to_string(p.num_qubits()) + ", rows have " + std::to_string(n_));
        BitVec out(size());
        if (size()) Device::instance().check(sk_commutation_vector(r_, p.x_words().data(), p.z_words().data(), out.words.data()));
        return out;
    }
    sk_rows* handle() const { return r_; }
  private:
    size_t n_; sk_rows* r_ = nullptr;
};

}  // namespace stabkit
