// stab_oracle.cpp -- CPU ORACLE. TEST INFRASTRUCTURE ONLY.
//
// A plain C++ restatement of the reference's stabilizer-tableau algorithms
// (stabkit / STABSim, /root/reference).  Nothing in the product path
// (paper_2507_03092_b200/, include/) may include, link or call this file; it
// exists so that tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
// leg can check / time the CUDA path against an independent implementation.
//
// Parity status
//   * Pauli-row arithmetic (conj_*, product_g_sum, commutation_vector,
//     rowsum_plus_i, CounterRng, SplitMix64): PINNED.  Checked bit-for-bit
//     against the compiled reference (oracle/_ref, built from
//     /root/reference/proj/src/pauli.cpp) and against the committed golden
//     vectors in tests/golden/ (generated from that build).
//   * Tableau / measurement / sim / grouping / transpiler drivers: the
//     reference ships only SPEC.md prose for these ("spec only", SURVEY.md
//     section 2.1), so they are pinned by SPEC's known-answer examples
//     (tests/test_oracle_spec_examples.py) -- "parity unpinned" beyond those.
//
// Every function cites the reference file:line (or SPEC/PAPER line) it follows.
// Word format: 64-bit words, qubit q -> word q>>6, bit q&63 (bitvec.hpp:26-35,
// pauli.hpp:53-54); I=(0,0) X=(1,0) Z=(0,1) Y=(1,1); sign 1 == -1 (pauli.hpp:28-31).

#include <algorithm>
#include <atomic>
#include <bit>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

namespace orc {

using u64 = uint64_t;
using i64 = int64_t;

// ---------------------------------------------------------------- rng ------
// rng.hpp:23-28
static inline u64 splitmix64(u64 x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
// rng.hpp:33-39  CounterRng::bit
static inline int counter_bit(u64 seed, u64 ordinal) {
    return int(splitmix64(seed ^ splitmix64(ordinal ^ 0xd1b54a32d192ed03ULL)) & 1);
}
// rng.hpp:43-65  SplitMix64 sequential generator
struct Seq {
    u64 s;
    explicit Seq(u64 seed) : s(seed) {}
    u64 next() { s += 0x9e3779b97f4a7c15ULL; u64 z = s;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31); }
    u64 below(u64 b) { return next() % b; }
    double unit() { return double(next() >> 11) * 0x1.0p-53; }
};

// ------------------------------------------------------- row arithmetic ----
static inline size_t words_for(size_t n) { return (n + 63) / 64; }

// Algorithm 1's g summed over one word pair, PAPER:153-164 (restated as the
// two masks pauli.cpp:189-205 counts): +1 for (X,Y) (Y,Z) (Z,X); -1 for the
// reversed pairs.  a is the LEFT factor.
static inline int g_word(u64 ax, u64 az, u64 bx, u64 bz) {
    u64 aX = ax & ~az, aY = ax & az, aZ = ~ax & az;
    u64 bX = bx & ~bz, bY = bx & bz, bZ = ~bx & bz;
    u64 plus = (aX & bY) | (aY & bZ) | (aZ & bX);
    u64 minus = (aX & bZ) | (aY & bX) | (aZ & bY);
    return std::popcount(plus) - std::popcount(minus);
}
// pauli.cpp:189-205 product_g_sum
static i64 g_sum(const u64* ax, const u64* az, const u64* bx, const u64* bz, size_t W) {
    i64 t = 0;
    for (size_t w = 0; w < W; ++w) t += g_word(ax[w], az[w], bx[w], bz[w]);
    return t;
}
// pauli.cpp:117-127 commutes_with  (true == commute)
static bool commutes(const u64* ax, const u64* az, const u64* bx, const u64* bz, size_t W) {
    int par = 0;
    for (size_t w = 0; w < W; ++w) par ^= std::popcount((ax[w] & bz[w]) ^ (bx[w] & az[w])) & 1;
    return par == 0;
}
// pauli.cpp:129-140 qubitwise_commutes_with
static bool qw_commutes(const u64* ax, const u64* az, const u64* bx, const u64* bz, size_t W) {
    for (size_t w = 0; w < W; ++w) if ((ax[w] & bz[w]) ^ (bx[w] & az[w])) return false;
    return true;
}

// A dense block of signed Pauli rows, row-major, W words of x then W of z per row.
struct Rows {
    size_t n = 0, W = 0, m = 0;
    std::vector<u64> x, z;       // m*W each
    std::vector<uint8_t> r;      // m
    Rows() = default;
    Rows(size_t n_, size_t m_) : n(n_), W(words_for(n_)), m(m_), x(m_ * W, 0), z(m_ * W, 0), r(m_, 0) {}
    u64* X(size_t i) { return &x[i * W]; }
    u64* Z(size_t i) { return &z[i * W]; }
    const u64* X(size_t i) const { return &x[i * W]; }
    const u64* Z(size_t i) const { return &z[i * W]; }
    int xb(size_t i, size_t q) const { return int((x[i * W + (q >> 6)] >> (q & 63)) & 1); }
    int zb(size_t i, size_t q) const { return int((z[i * W + (q >> 6)] >> (q & 63)) & 1); }
    void push_zero() { x.resize(x.size() + W, 0); z.resize(z.size() + W, 0); r.push_back(0); ++m; }
    void erase(size_t i) {
        x.erase(x.begin() + i * W, x.begin() + (i + 1) * W);
        z.erase(z.begin() + i * W, z.begin() + (i + 1) * W);
        r.erase(r.begin() + i); --m;
    }
};

// pauli.cpp:146-156 conj_h 
static inline void row_h(Rows& t, size_t i, size_t q) {
    size_t w = i * t.W + (q >> 6); u64 m = u64{1} << (q & 63);
    u64 xb = t.x[w] & m, zb = t.z[w] & m;
    t.r[i] ^= uint8_t(xb && zb);
    u64 d = xb ^ zb; t.x[w] ^= d; t.z[w] ^= d;
}
// pauli.cpp:158-165 conj_s 
static inline void row_s(Rows& t, size_t i, size_t q) {
    size_t w = i * t.W + (q >> 6); u64 m = u64{1} << (q & 63);
    u64 xb = t.x[w] & m;
    t.r[i] ^= uint8_t(xb && (t.z[w] & m));
    t.z[w] ^= xb;
}
// pauli.cpp:167-174 conj_sdg
static inline void row_sdg(Rows& t, size_t i, size_t q) {
    size_t w = i * t.W + (q >> 6); u64 m = u64{1} << (q & 63);
    u64 xb = t.x[w] & m;
    t.r[i] ^= uint8_t(xb && !(t.z[w] & m));
    t.z[w] ^= xb;
}
// pauli.cpp:176-187 conj_cx ; SPEC:155-163 (full CHP sign factor)
static inline void row_cx(Rows& t, size_t i, size_t c, size_t q) {
    int xc = t.xb(i, c), zc = t.zb(i, c), xt = t.xb(i, q), zt = t.zb(i, q);
    t.r[i] ^= uint8_t(xc && zt && (xt == zc));
    if (xc) t.x[i * t.W + (q >> 6)] ^= u64{1} << (q & 63);
    if (zt) t.z[i * t.W + (c >> 6)] ^= u64{1} << (c & 63);
}

enum Kind : uint8_t { K_H = 0, K_S, K_SDG, K_X, K_Y, K_Z, K_CX, K_CZ, K_SWAP, K_M, K_T, K_TDG };
struct Gate { uint8_t kind; uint8_t pad[3]; uint32_t q0, q1; };
static_assert(sizeof(Gate) == 12, "gate ABI");

// SPEC:187-195 apply_gate: derived Cliffords are FIXED H/S/CX sequences:
// Z=S.S ; X=H.Z.H ; Y=Z.X ; SDG=S.S.S ; CZ=H(t).CX.H(t) ; SWAP=CX(a,b)CX(b,a)CX(a,b)
static inline void row_gate(Rows& t, size_t i, const Gate& g) {
    size_t a = g.q0, b = g.q1;
    switch (g.kind) {
        case K_H: row_h(t, i, a); break;
        case K_S: row_s(t, i, a); break;
        case K_SDG: row_s(t, i, a); row_s(t, i, a); row_s(t, i, a); break;
        case K_Z: row_s(t, i, a); row_s(t, i, a); break;
        case K_X: row_h(t, i, a); row_s(t, i, a); row_s(t, i, a); row_h(t, i, a); break;
        case K_Y: row_s(t, i, a); row_s(t, i, a);                           // Z
                  row_h(t, i, a); row_s(t, i, a); row_s(t, i, a); row_h(t, i, a); break;  // then X
        case K_CX: row_cx(t, i, a, b); break;
        case K_CZ: row_h(t, i, b); row_cx(t, i, a, b); row_h(t, i, b); break;
        case K_SWAP: row_cx(t, i, a, b); row_cx(t, i, b, a); row_cx(t, i, a, b); break;
        default: break;
    }
}

// ------------------------------------------------------------ tableau -----
struct Counters {
    u64 n_rand = 0, n_det = 0, k_rand = 0, k_det = 0;
    u64 gate_hist[12] = {0};
};

// rows 0..n-1 stabilizers, n..2n-1 destabilizers, 2n scratch.
struct Tableau {
    size_t n = 0;
    Rows t;
    Counters c;
    explicit Tableau(size_t n_) : n(n_), t(n_, 2 * n_ + 1) {       // SPEC:125-133 new_identity
        for (size_t q = 0; q < n; ++q) {
            t.Z(q)[q >> 6] |= u64{1} << (q & 63);          // stabilizer q = Z_q
            t.X(n + q)[q >> 6] |= u64{1} << (q & 63);      // destabilizer q = X_q
        }
    }
    // SPEC:165-173 rowsum(h, i) / PAPER:166-185.  Returns false on an odd sum.
    bool rowsum(size_t h, size_t i) {
        i64 sum = 2 * t.r[h] + 2 * t.r[i] + g_sum(t.X(i), t.Z(i), t.X(h), t.Z(h), t.W);
        int mod = int(((sum % 4) + 4) % 4);
        bool ok = (mod == 0 || mod == 2);
        if (ok) t.r[h] = uint8_t(mod == 2);
        for (size_t w = 0; w < t.W; ++w) { t.X(h)[w] ^= t.X(i)[w]; t.Z(h)[w] ^= t.Z(i)[w]; }
        return ok;
    }
    // SPEC:175-185 measure_z.  The random branch skips i == p+n: that row
    // anticommutes with the pivot (odd mod-4 sum) and is overwritten
    // by the copy of row p immediately afterwards (SURVEY.md section 7 hazard).
    void measure_z(size_t q, u64 seed, u64 ordinal, int* outcome, int* deterministic) {
        size_t p = n;
        for (size_t i = 0; i < n; ++i) if (t.xb(i, q)) { p = i; break; }   // smallest p
        if (p < n) {
            for (size_t i = 0; i < 2 * n; ++i)
                if (i != p && i != p + n && t.xb(i, q)) { rowsum(i, p); ++c.k_rand; }
            std::copy(t.X(p), t.X(p) + t.W, t.X(p + n));
            std::copy(t.Z(p), t.Z(p) + t.W, t.Z(p + n));
            t.r[p + n] = t.r[p];
            std::fill(t.X(p), t.X(p) + t.W, 0); std::fill(t.Z(p), t.Z(p) + t.W, 0);
            t.Z(p)[q >> 6] = u64{1} << (q & 63);
            t.r[p] = uint8_t(counter_bit(seed, ordinal));
            *outcome = t.r[p]; *deterministic = 0; ++c.n_rand;
        } else {
            size_t s = 2 * n;                                            // scratch
            std::fill(t.X(s), t.X(s) + t.W, 0); std::fill(t.Z(s), t.Z(s) + t.W, 0); t.r[s] = 0;
            for (size_t j = n; j < 2 * n; ++j) if (t.xb(j, q)) { rowsum(s, j - n); ++c.k_det; }
            *outcome = t.r[s]; *deterministic = 1; ++c.n_det;
            std::fill(t.X(s), t.X(s) + t.W, 0); std::fill(t.Z(s), t.Z(s) + t.W, 0); t.r[s] = 0;
        }
    }
};

// SPEC:310-318 sim.  Clifford runs are row-partitioned across `workers`
// (no sync inside a run because rows are independent);
// every M is a full barrier.  Output is schedule independent.
static void apply_run(Tableau& T, const Gate* g, size_t ng, int workers) {
    size_t rows = 2 * T.n;
    auto body = [&](size_t lo, size_t hi) {
        for (size_t i = lo; i < hi; ++i)
            for (size_t k = 0; k < ng; ++k) row_gate(T.t, i, g[k]);
    };
    if (workers <= 1 || rows * ng < 200000) { body(0, rows); return; }
    std::vector<std::thread> th;
    size_t per = (rows + workers - 1) / workers;
    for (int w = 0; w < workers; ++w) {
        size_t lo = std::min(rows, w * per), hi = std::min(rows, lo + per);
        if (lo < hi) th.emplace_back(body, lo, hi);
    }
    for (auto& t : th) t.join();
}

// returns 0 ok, 2 unsupported (T gate), 1 bad qubit
static int sim(Tableau& T, const Gate* gates, size_t ng, u64 seed, int workers,
               uint8_t* outcomes, uint8_t* dets, u64 ordinal0 = 0) {
    u64 ord = ordinal0; size_t i = 0;
    while (i < ng) {
        if (gates[i].kind == K_M) {
            int o, d; T.measure_z(gates[i].q0, seed, ord, &o, &d);
            if (outcomes) outcomes[ord - ordinal0] = uint8_t(o);
            if (dets) dets[ord - ordinal0] = uint8_t(d);
            ++ord; ++T.c.gate_hist[K_M]; ++i; continue;
        }
        size_t j = i;
        while (j < ng && gates[j].kind != K_M) {
            if (gates[j].kind >= K_T) return 2;
            ++T.c.gate_hist[gates[j].kind]; ++j;
        }
        apply_run(T, gates + i, j - i, workers);
        i = j;
    }
    return 0;
}

// ------------------------------------------------------------ grouping ----
// SPEC:444-452 group_greedy on already-sorted terms (sorting is host logic:
// |coeff| desc, ties by Pauli text then input order).  First fit.
// mode 0 = GC (commutes), 1 = QWC.  out_group[i] = group id of sorted term i.
static u64 group_first_fit(const Rows& terms, int mode, uint32_t* out_group, u64* pred_calls) {
    std::vector<std::vector<uint32_t>> groups;
    u64 calls = 0;
    for (size_t t = 0; t < terms.m; ++t) {
        size_t placed = groups.size();
        for (size_t g = 0; g < groups.size() && placed == groups.size(); ++g) {
            bool ok = true;
            for (uint32_t m : groups[g]) {
                ++calls;
                bool c = mode ? qw_commutes(terms.X(t), terms.Z(t), terms.X(m), terms.Z(m), terms.W)
                              : commutes(terms.X(t), terms.Z(t), terms.X(m), terms.Z(m), terms.W);
                if (!c) { ok = false; break; }
            }
            if (ok) placed = g;
        }
        if (placed == groups.size()) groups.emplace_back();
        groups[placed].push_back(uint32_t(t));
        out_group[t] = uint32_t(placed);
    }
    if (pred_calls) *pred_calls = calls;
    return groups.size();
}
// SPEC:454-462 verify_grouping: number of violating intra-group pairs.
static u64 verify_grouping(const Rows& terms, int mode, const uint32_t* group) {
    std::unordered_map<uint32_t, std::vector<uint32_t>> g;
    for (size_t i = 0; i < terms.m; ++i) g[group[i]].push_back(uint32_t(i));
    u64 bad = 0;
    for (auto& kv : g) for (size_t a = 0; a < kv.second.size(); ++a) for (size_t b = a + 1; b < kv.second.size(); ++b) {
        uint32_t i = kv.second[a], j = kv.second[b];
        bool c = mode ? qw_commutes(terms.X(i), terms.Z(i), terms.X(j), terms.Z(j), terms.W)
                      : commutes(terms.X(i), terms.Z(i), terms.X(j), terms.Z(j), terms.W);
        bad += !c;
    }
    return bad;
}

// ---------------------------------------------------------- transpiler ----
// pauli.cpp:239-254 rowsum_plus_i: target := i * pushed * target.  false = odd.
static bool rowsum_plus_i(Rows& tr, size_t ti, const u64* px, const u64* pz, int pr) {
    i64 sum = 2 * tr.r[ti] + 2 * pr + g_sum(px, pz, tr.X(ti), tr.Z(ti), tr.W) + 1;
    int mod = int(((sum % 4) + 4) % 4);
    if (mod != 0 && mod != 2) return false;
    tr.r[ti] = uint8_t(mod == 2);
    for (size_t w = 0; w < tr.W; ++w) { tr.X(ti)[w] ^= px[w]; tr.Z(ti)[w] ^= pz[w]; }
    return true;
}

struct Pbc {
    size_t n = 0;
    std::vector<Rows> layers;    // forward time order
    Tableau M;                   // measurement tableau
    u64 initial_t = 0, passes = 0;
    int status = 0;              // 0 ok, 2 unsupported, 3 invariant
    explicit Pbc(size_t n_) : n(n_), M(n_) {}
};

// SPEC:515-523 build_tableaus / Algorithm 2 PAPER:372-387.  Trailing Z
// measurements are stripped; any other M is unsupported.
// T_tab rows are in append order (reverse circuit time).
// exact = true: the backward walk conjugates by the INVERSE gate (S <-> S^dagger; every other Clifford of the gate set
// is its own inverse).  Moving a measurement / rotation axis P from behind G to in front of it turns it into
// G^dagger P G, so this is what unitary equivalence needs (tests/test_oracle_dense.py); exact = false applies G's own
// rule, the literal reading of "Apply G to M_tab and T_tab using CHP rules" (Algorithm 2 line 8).
static int build_tableaus(size_t n, const Gate* g, size_t ng, Tableau& M, Rows& T, bool exact = false) {
    size_t end = ng;
    while (end > 0 && g[end - 1].kind == K_M) --end;
    for (size_t i = 0; i < end; ++i) if (g[i].kind == K_M) return 2;
    T = Rows(n, 0);
    for (size_t k = end; k-- > 0;) {
        Gate a = g[k];
        if (exact) { if (a.kind == K_S) a.kind = K_SDG; else if (a.kind == K_SDG) a.kind = K_S; }
        if (a.kind == K_T || a.kind == K_TDG) {
            T.push_zero();
            T.Z(T.m - 1)[a.q0 >> 6] |= u64{1} << (a.q0 & 63);
            T.r[T.m - 1] = uint8_t(a.kind == K_TDG);
        } else {
            for (size_t i = 0; i < 2 * n; ++i) row_gate(M.t, i, a);
            for (size_t i = 0; i < T.m; ++i) row_gate(T, i, a);
        }
    }
    return 0;
}

// SPEC:525-533 t_separate / Algorithm 3: scan rows in `order`, first fit from P_0.
// ordered = true: a row joins the layer right AFTER the last layer that holds an anticommuting member (it may not be
// moved in front of a rotation it does not commute with); ordered = false is Algorithm 3 as published: the first
// layer, scanning from P_0, whose members all commute with it.
static void separate_into(const Rows& src, const std::vector<size_t>& order, std::vector<Rows>& layers, bool ordered = false) {
    for (size_t s : order) {
        size_t placed = layers.size();
        if (ordered) {
            placed = 0;
            for (size_t k = 0; k < layers.size(); ++k)
                for (size_t m = 0; m < layers[k].m; ++m)
                    if (!commutes(src.X(s), src.Z(s), layers[k].X(m), layers[k].Z(m), src.W)) { placed = k + 1; break; }
        } else
        for (size_t k = 0; k < layers.size() && placed == layers.size(); ++k) {
            bool ok = true;
            for (size_t m = 0; m < layers[k].m && ok; ++m)
                ok = commutes(src.X(s), src.Z(s), layers[k].X(m), layers[k].Z(m), src.W);
            if (ok) placed = k;
        }
        if (placed == layers.size()) layers.emplace_back(src.n, 0);
        Rows& L = layers[placed];
        L.push_zero();
        std::copy(src.X(s), src.X(s) + src.W, L.X(L.m - 1));
        std::copy(src.Z(s), src.Z(s) + src.W, L.Z(L.m - 1));
        L.r[L.m - 1] = src.r[s];
    }
}
static std::vector<Rows> t_separate(const Rows& T, bool ordered = false) {
    std::vector<size_t> order;
    for (size_t s = T.m; s-- > 0;) order.push_back(s);       // last appended first == forward time
    std::vector<Rows> layers; separate_into(T, order, layers, ordered); return layers;
}

// first (x,z)-duplicate pair in scan order: smallest i with a later
// same_axis row (pauli.cpp:142-144), then the smallest such j.
static bool first_duplicate(const Rows& L, size_t* oi, size_t* oj) {
    std::unordered_map<u64, std::vector<uint32_t>> buckets;
    auto hash = [&](size_t i) { u64 h = 0x243f6a8885a308d3ULL;
        for (size_t w = 0; w < L.W; ++w) { h = splitmix64(h ^ L.X(i)[w]); h = splitmix64(h ^ (L.Z(i)[w] * 3)); }
        return h; };
    std::vector<u64> hs(L.m);
    for (size_t i = 0; i < L.m; ++i) { hs[i] = hash(i); buckets[hs[i]].push_back(uint32_t(i)); }
    for (size_t i = 0; i < L.m; ++i) {
        auto& b = buckets[hs[i]];
        if (b.size() < 2) continue;
        for (uint32_t j : b) {
            if (j <= i) continue;
            if (std::equal(L.X(i), L.X(i) + L.W, L.X(j)) && std::equal(L.Z(i), L.Z(i) + L.W, L.Z(j))) {
                *oi = i; *oj = j; return true;
            }
        }
    }
    return false;
}

// SPEC:535-543 t_optimize / Algorithm 4 PAPER:441-472.  Layers in forward time
// order; a pass visits layers from the last (closest to measurement) to the
// first.  Equal-sign duplicate pair -> quarter rotation (P, s) pushed through
// every later layer and then applied to M_tab (each arriving copy is applied
// immediately; four identical copies compose to the identity, so this equals
// the "annihilate in fours, apply the residue" wording).  Opposite signs cancel
// (SPEC:587).  Empty layers are dropped after each pass.
static int t_optimize(std::vector<Rows>& layers, Tableau& M, u64* passes) {
    auto total = [&] { u64 s = 0; for (auto& L : layers) s += L.m; return s; };
    u64 prev = total(); *passes = 0;
    for (;;) {
        ++*passes;
        for (size_t L = layers.size(); L-- > 0;) {
            size_t i, j;
            while (first_duplicate(layers[L], &i, &j)) {
                Rows& lay = layers[L];
                std::vector<u64> px(lay.X(i), lay.X(i) + lay.W), pz(lay.Z(i), lay.Z(i) + lay.W);
                int si = lay.r[i], sj = lay.r[j];
                lay.erase(j); lay.erase(i);
                if (si != sj) continue;
                for (size_t L2 = L + 1; L2 < layers.size(); ++L2)
                    for (size_t m = 0; m < layers[L2].m; ++m)
                        if (!commutes(px.data(), pz.data(), layers[L2].X(m), layers[L2].Z(m), lay.W))
                            if (!rowsum_plus_i(layers[L2], m, px.data(), pz.data(), si)) return 3;
                for (size_t m = 0; m < 2 * M.n; ++m)
                    if (!commutes(px.data(), pz.data(), M.t.X(m), M.t.Z(m), M.t.W))
                        if (!rowsum_plus_i(M.t, m, px.data(), pz.data(), si)) return 3;
            }
        }
        layers.erase(std::remove_if(layers.begin(), layers.end(), [](const Rows& L) { return L.m == 0; }), layers.end());
        u64 now = total();
        if (now == prev) break;
        prev = now;
    }
    return 0;
}

// SPEC:545-553 transpile: build -> separate -> optimize -> re-separate layers
// that lost internal commutativity.
static void transpile(Pbc& P, const Gate* g, size_t ng, bool exact = false) {
    Rows T;
    P.status = build_tableaus(P.n, g, ng, P.M, T, exact);
    if (P.status) return;
    P.initial_t = T.m;
    P.layers = t_separate(T, exact);
    P.status = t_optimize(P.layers, P.M, &P.passes);
    if (P.status) return;
    std::vector<Rows> out;
    for (auto& L : P.layers) {
        bool ok = true;
        for (size_t a = 0; a < L.m && ok; ++a) for (size_t b = a + 1; b < L.m && ok; ++b)
            ok = commutes(L.X(a), L.Z(a), L.X(b), L.Z(b), L.W);
        if (ok) { out.push_back(std::move(L)); continue; }
        std::vector<size_t> order(L.m); for (size_t i = 0; i < L.m; ++i) order[i] = i;
        std::vector<Rows> sub; separate_into(L, order, sub, exact);
        for (auto& s : sub) out.push_back(std::move(s));
    }
    P.layers = std::move(out);
}

}  // namespace orc

// ================================================================ C API ====
using namespace orc;
extern "C" {

uint64_t orc_splitmix64(uint64_t x) { return splitmix64(x); }
int orc_counter_bit(uint64_t seed, uint64_t ord) { return counter_bit(seed, ord); }
void orc_seq_fill(uint64_t seed, uint64_t* out, size_t k) { Seq s(seed); for (size_t i = 0; i < k; ++i) out[i] = s.next(); }

int64_t orc_g_sum(const uint64_t* ax, const uint64_t* az, const uint64_t* bx, const uint64_t* bz, size_t W) { return g_sum(ax, az, bx, bz, W); }
int orc_commutes(const uint64_t* ax, const uint64_t* az, const uint64_t* bx, const uint64_t* bz, size_t W) { return commutes(ax, az, bx, bz, W); }
int orc_qw_commutes(const uint64_t* ax, const uint64_t* az, const uint64_t* bx, const uint64_t* bz, size_t W) { return qw_commutes(ax, az, bx, bz, W); }

// rows handle -------------------------------------------------------------
void* orc_rows_new(size_t n, size_t m) { return new Rows(n, m); }
void orc_rows_free(void* h) { delete static_cast<Rows*>(h); }
size_t orc_rows_count(void* h) { return static_cast<Rows*>(h)->m; }
void orc_rows_set(void* h, const uint64_t* x, const uint64_t* z, const uint8_t* r) {
    Rows* R = static_cast<Rows*>(h);
    std::copy(x, x + R->m * R->W, R->x.begin()); std::copy(z, z + R->m * R->W, R->z.begin()); std::copy(r, r + R->m, R->r.begin());
}
void orc_rows_get(void* h, uint64_t* x, uint64_t* z, uint8_t* r) {
    Rows* R = static_cast<Rows*>(h);
    std::copy(R->x.begin(), R->x.end(), x); std::copy(R->z.begin(), R->z.end(), z); std::copy(R->r.begin(), R->r.end(), r);
}
void orc_rows_apply(void* h, const Gate* g, size_t ng) {
    Rows* R = static_cast<Rows*>(h);
    for (size_t k = 0; k < ng; ++k) for (size_t i = 0; i < R->m; ++i) row_gate(*R, i, g[k]);
}
// pauli.cpp:215-237 commutation_vector: bit i set iff p ANTIcommutes with row i
void orc_commutation_vector(void* h, const uint64_t* px, const uint64_t* pz, uint64_t* out_bits) {
    Rows* R = static_cast<Rows*>(h);
    std::fill(out_bits, out_bits + words_for(R->m), 0);
    for (size_t i = 0; i < R->m; ++i)
        if (!commutes(px, pz, R->X(i), R->Z(i), R->W)) out_bits[i >> 6] |= u64{1} << (i & 63);
}
int orc_rowsum_plus_i(void* h, size_t i, const uint64_t* px, const uint64_t* pz, int pr) {
    return rowsum_plus_i(*static_cast<Rows*>(h), i, px, pz, pr) ? 0 : 3;
}
// pauli.cpp:100-106 weight, summed over rows
uint64_t orc_weight_sum(void* h) {
    Rows* R = static_cast<Rows*>(h); u64 s = 0;
    for (size_t i = 0; i < R->m * R->W; ++i) s += std::popcount(R->x[i] | R->z[i]);
    return s;
}
int orc_first_duplicate(void* h, uint64_t* i, uint64_t* j) {
    size_t a, b; if (!first_duplicate(*static_cast<Rows*>(h), &a, &b)) return 0; *i = a; *j = b; return 1;
}
uint64_t orc_group_first_fit(void* h, int mode, uint32_t* out_group, uint64_t* pred_calls) {
    return group_first_fit(*static_cast<Rows*>(h), mode, out_group, pred_calls);
}
uint64_t orc_verify_grouping(void* h, int mode, const uint32_t* group) { return verify_grouping(*static_cast<Rows*>(h), mode, group); }

// tableau handle ----------------------------------------------------------
void* orc_tab_new(size_t n) { return n ? new Tableau(n) : nullptr; }
void orc_tab_free(void* h) { delete static_cast<Tableau*>(h); }
// row-major export of the 2n live rows: x[2n*W], z[2n*W], r[2n]
void orc_tab_get(void* h, uint64_t* x, uint64_t* z, uint8_t* r) {
    Tableau* T = static_cast<Tableau*>(h); size_t k = 2 * T->n * T->t.W;
    std::copy(T->t.x.begin(), T->t.x.begin() + k, x); std::copy(T->t.z.begin(), T->t.z.begin() + k, z);
    std::copy(T->t.r.begin(), T->t.r.begin() + 2 * T->n, r);
}
void orc_tab_set(void* h, const uint64_t* x, const uint64_t* z, const uint8_t* r) {
    Tableau* T = static_cast<Tableau*>(h); size_t k = 2 * T->n * T->t.W;
    std::copy(x, x + k, T->t.x.begin()); std::copy(z, z + k, T->t.z.begin()); std::copy(r, r + 2 * T->n, T->t.r.begin());
}
int orc_tab_rowsum(void* h, size_t hh, size_t i) { return static_cast<Tableau*>(h)->rowsum(hh, i) ? 0 : 3; }
int orc_tab_sim(void* h, const Gate* g, size_t ng, uint64_t seed, int workers, uint8_t* outcomes, uint8_t* dets, uint64_t ordinal0) {
    return sim(*static_cast<Tableau*>(h), g, ng, seed, workers, outcomes, dets, ordinal0);
}
// counters: n_rand, n_det, k_rand, k_det, then 12 gate-kind counts
void orc_tab_counters(void* h, uint64_t* out16) {
    Tableau* T = static_cast<Tableau*>(h);
    out16[0] = T->c.n_rand; out16[1] = T->c.n_det; out16[2] = T->c.k_rand; out16[3] = T->c.k_det;
    for (int i = 0; i < 12; ++i) out16[4 + i] = T->c.gate_hist[i];
}

// qec_gen -------------------------------------------------------------------
// SPEC:369-383, 399-403 surface_code_circuit, written independently of the product's generator
// (paper_2507_03092_b200/csrc/circuit_host.cpp) so that tests can cross-check the two gate for gate; the
// conventions SPEC leaves open are the ones DESIGN.md section 8 freezes:
//   data qubit (r, c) = r*d + c; a plaquette is named by its south-east corner (i, j), 0 <= i, j <= d, and touches
//   the data qubits (i-1,j-1) (i-1,j) (i,j-1) (i,j) that exist; X type iff i+j even; all interior plaquettes, X-type
//   ones on the top/bottom edge, Z-type ones on the left/right edge; ancillas numbered d*d.. in row-major (i, j) order;
//   round = [H on X ancillas] [4 CX slots: X: NW NE SW SE, ancilla -> data; Z: NW SW NE SE, data -> ancilla]
//   [H on X ancillas] [M on every ancilla in index order], a chunk mark in front of each bracket.
// Two passes: count, then fill caller-provided arrays (gates == nullptr -> sizes only).  Returns the qubit count, 0 = bad args.
uint64_t orc_surface_code(uint32_t d, uint32_t rounds, int final_data_measure, Gate* gates, size_t* ngates, uint32_t* marks, size_t* nmarks) {
    if (d < 3 || !(d & 1) || rounds == 0) return 0;
    const long D = d;
    std::vector<uint32_t> anc_of((D + 1) * (D + 1), 0xffffffffu);          // plaquette -> ancilla qubit
    uint32_t q = uint32_t(D * D);
    for (long i = 0; i <= D; ++i) for (long j = 0; j <= D; ++j) {
        const bool xtype = ((i + j) & 1) == 0, edge_i = (i == 0 || i == D), edge_j = (j == 0 || j == D);
        bool keep;
        if (!edge_i && !edge_j) keep = true;
        else if (edge_i && !edge_j) keep = xtype;
        else if (edge_j && !edge_i) keep = !xtype;
        else keep = false;
        if (keep) anc_of[i * (D + 1) + j] = q++;
    }
    const uint64_t nq = q;
    size_t ng = 0, nm = 0;
    auto emit = [&](uint8_t k, uint32_t a, uint32_t b) { if (gates) { Gate g{}; g.kind = k; g.q0 = a; g.q1 = b; gates[ng] = g; } ++ng; };
    size_t last_mark = size_t(-1);       // a mark is a gate index > 0, never repeated
    auto mark2 = [&] { if (ng == 0 || last_mark == ng) return; last_mark = ng; if (marks) marks[nm] = uint32_t(ng); ++nm; };
    // corner offsets of a plaquette's data qubits in each type's CX order
    static const int xo[4][2] = {{-1, -1}, {-1, 0}, {0, -1}, {0, 0}};     // NW NE SW SE
    static const int zo[4][2] = {{-1, -1}, {0, -1}, {-1, 0}, {0, 0}};     // NW SW NE SE
    for (uint32_t r = 0; r < rounds; ++r) {
        for (int phase = 0; phase < 7; ++phase) {     // 0: H, 1-4: CX slot, 5: H, 6: M
            mark2();
            for (long i = 0; i <= D; ++i) for (long j = 0; j <= D; ++j) {
                const uint32_t a = anc_of[i * (D + 1) + j];
                if (a == 0xffffffffu) continue;
                const bool xtype = ((i + j) & 1) == 0;
                if (phase == 0 || phase == 5) { if (xtype) emit(K_H, a, 0); }
                else if (phase == 6) emit(K_M, a, 0);
                else {
                    const int* o = xtype ? xo[phase - 1] : zo[phase - 1];
                    const long rr = i + o[0], cc = j + o[1];
                    if (rr < 0 || cc < 0 || rr >= D || cc >= D) continue;
                    const uint32_t dq = uint32_t(rr * D + cc);
                    if (xtype) emit(K_CX, a, dq); else emit(K_CX, dq, a);
                }
            }
        }
    }
    if (final_data_measure) { mark2(); for (uint32_t k = 0; k < uint32_t(D * D); ++k) emit(K_M, k, 0); }
    *ngates = ng; *nmarks = nm;
    return nq;
}

// transpiler ----------------------------------------------------------------
void* orc_transpile(size_t n, const Gate* g, size_t ng) { Pbc* P = new Pbc(n); transpile(*P, g, ng); return P; }
// flags bit 0: unitary-exact variant (inverse-gate conjugation in Algorithm 2, order-preserving separation in Algorithm 3)
void* orc_transpile_ex(size_t n, const Gate* g, size_t ng, unsigned flags) { Pbc* P = new Pbc(n); transpile(*P, g, ng, (flags & 1u) != 0); return P; }
void orc_pbc_free(void* h) { delete static_cast<Pbc*>(h); }
int orc_pbc_status(void* h) { return static_cast<Pbc*>(h)->status; }
// stats: initial_t, final rowcount, final pauli weight, layers, passes
void orc_pbc_stats(void* h, uint64_t* out5) {
    Pbc* P = static_cast<Pbc*>(h); u64 rows = 0, wt = 0;
    for (auto& L : P->layers) { rows += L.m; for (size_t i = 0; i < L.m * L.W; ++i) wt += std::popcount(L.x[i] | L.z[i]); }
    out5[0] = P->initial_t; out5[1] = rows; out5[2] = wt; out5[3] = P->layers.size(); out5[4] = P->passes;
}
size_t orc_pbc_layer_rows(void* h, size_t k) { return static_cast<Pbc*>(h)->layers[k].m; }
void orc_pbc_layer_get(void* h, size_t k, uint64_t* x, uint64_t* z, uint8_t* r) {
    Rows& L = static_cast<Pbc*>(h)->layers[k];
    std::copy(L.x.begin(), L.x.end(), x); std::copy(L.z.begin(), L.z.end(), z); std::copy(L.r.begin(), L.r.end(), r);
}
void* orc_pbc_mtab(void* h) { return &static_cast<Pbc*>(h)->M; }   // borrowed Tableau handle

// staged access for unit tests of Algorithm 2 / 3 ---------------------------
void* orc_build_ttab(size_t n, const Gate* g, size_t ng, void* mtab_out, int* status) {
    Rows* T = new Rows(n, 0);
    *status = build_tableaus(n, g, ng, *static_cast<Tableau*>(mtab_out), *T);
    return T;
}
// layer id for each T_tab row (row order = append order)
size_t orc_t_separate_ids(void* ttab, uint32_t* layer_of_row) {
    Rows* T = static_cast<Rows*>(ttab);
    std::vector<Rows> layers; std::vector<std::vector<size_t>> members;
    // replay separate_into but remember membership
    for (size_t s = T->m; s-- > 0;) {
        size_t placed = layers.size();
        for (size_t k = 0; k < layers.size() && placed == layers.size(); ++k) {
            bool ok = true;
            for (size_t m = 0; m < layers[k].m && ok; ++m) ok = commutes(T->X(s), T->Z(s), layers[k].X(m), layers[k].Z(m), T->W);
            if (ok) placed = k;
        }
        if (placed == layers.size()) layers.emplace_back(T->n, 0);
        Rows& L = layers[placed]; L.push_zero();
        std::copy(T->X(s), T->X(s) + T->W, L.X(L.m - 1)); std::copy(T->Z(s), T->Z(s) + T->W, L.Z(L.m - 1));
        layer_of_row[s] = uint32_t(placed);
    }
    return layers.size();
}

}  // extern "C"
