// ref_shim.cpp -- C shim over the UNMODIFIED reference translation unit.
//
// TEST INFRASTRUCTURE ONLY.  Built by oracle/Makefile together with
// /root/reference/proj/src/pauli.cpp (compiled where it lies; nothing is
// copied) into oracle/_ref/libstabkit_ref.so.  It lets the tests check the
// oracle restatement (stab_oracle.cpp) against the real reference arithmetic
// and regenerate tests/golden/*.json (tests/golden/make_golden.py).
//
// The shim converts raw word arrays to stabkit::PauliString through the
// reference's own public API (pauli.hpp:32-123) and back.

#include <cstdint>
#include <cstring>
#include <span>
#include <string>
#include <vector>

#include "stabkit/error.hpp"
#include "stabkit/pauli.hpp"
#include "stabkit/rng.hpp"

using stabkit::PauliString;

static PauliString make(size_t n, const uint64_t* x, const uint64_t* z, int sign) {
    PauliString p(n);
    size_t W = stabkit::words_for_bits(n);
    for (size_t w = 0; w < W; ++w) { p.x_words()[w] = x[w]; p.z_words()[w] = z[w]; }
    p.set_sign(sign != 0);
    return p;
}
static void dump(const PauliString& p, uint64_t* x, uint64_t* z, int* sign) {
    size_t W = stabkit::words_for_bits(p.num_qubits());
    for (size_t w = 0; w < W; ++w) { x[w] = p.x_words()[w]; z[w] = p.z_words()[w]; }
    *sign = p.sign();
}

extern "C" {

uint64_t ref_splitmix64(uint64_t x) { return stabkit::splitmix64(x); }
int ref_counter_bit(uint64_t seed, uint64_t ord) { return stabkit::CounterRng{seed}.bit(ord); }
void ref_seq_fill(uint64_t seed, uint64_t* out, size_t k) { stabkit::SplitMix64 g(seed); for (size_t i = 0; i < k; ++i) out[i] = g.next(); }
double ref_seq_unit(uint64_t seed, size_t skip) { stabkit::SplitMix64 g(seed); for (size_t i = 0; i < skip; ++i) g.next(); return g.unit(); }

int64_t ref_g_sum(const uint64_t* ax, const uint64_t* az, const uint64_t* bx, const uint64_t* bz, size_t W) {
    return stabkit::product_g_sum(ax, az, bx, bz, W);
}
int ref_commutes(size_t n, const uint64_t* ax, const uint64_t* az, const uint64_t* bx, const uint64_t* bz) {
    return make(n, ax, az, 0).commutes_with(make(n, bx, bz, 0));
}
int ref_qw_commutes(size_t n, const uint64_t* ax, const uint64_t* az, const uint64_t* bx, const uint64_t* bz) {
    return make(n, ax, az, 0).qubitwise_commutes_with(make(n, bx, bz, 0));
}
uint64_t ref_weight(size_t n, const uint64_t* x, const uint64_t* z) { return make(n, x, z, 0).weight(); }

// kind: 0 H, 1 S, 2 SDG, 6 CX (same numbering as the oracle / sk_gate)
void ref_conj(size_t n, uint64_t* x, uint64_t* z, int* sign, int kind, size_t q0, size_t q1) {
    PauliString p = make(n, x, z, *sign);
    switch (kind) {
        case 0: p.conj_h(q0); break;
        case 1: p.conj_s(q0); break;
        case 2: p.conj_sdg(q0); break;
        case 6: p.conj_cx(q0, q1); break;
        default: break;
    }
    dump(p, x, z, sign);
}
// returns 0 ok, 3 InvariantError
int ref_rowsum_plus_i(size_t n, uint64_t* tx, uint64_t* tz, int* tsign, const uint64_t* px, const uint64_t* pz, int psign) {
    PauliString t = make(n, tx, tz, *tsign), p = make(n, px, pz, psign);
    try { stabkit::rowsum_plus_i(t, p); } catch (const stabkit::InvariantError&) { return 3; }
    dump(t, tx, tz, tsign);
    return 0;
}
// rows: m rows of W words each, row-major
void ref_commutation_vector(size_t n, const uint64_t* px, const uint64_t* pz, const uint64_t* rx, const uint64_t* rz,
                            size_t m, uint64_t* out_bits) {
    size_t W = stabkit::words_for_bits(n);
    std::vector<PauliString> rows;
    for (size_t i = 0; i < m; ++i) rows.push_back(make(n, rx + i * W, rz + i * W, 0));
    stabkit::BitVec v = stabkit::commutation_vector(make(n, px, pz, 0), std::span<const PauliString>(rows));
    for (size_t w = 0; w < v.words.size(); ++w) out_bits[w] = v.words[w];
}
// parse -> str round trip; returns length written, or -(position) style error text in buf with rc<0
int ref_parse_str(const char* text, char* buf, size_t cap) {
    try {
        std::string s = PauliString::parse(text).str();
        std::strncpy(buf, s.c_str(), cap - 1); buf[cap - 1] = 0; return int(s.size());
    } catch (const stabkit::ParseError& e) {
        std::strncpy(buf, e.what(), cap - 1); buf[cap - 1] = 0; return -1;
    }
}

}  // extern "C"
