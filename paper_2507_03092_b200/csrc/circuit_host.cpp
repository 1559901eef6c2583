// circuit_host.cpp -- circuit_io + qec_gen host logic behind the C ABI
// (SPEC:226-292 circuit_io, SPEC:364-416 qec_gen).  Pure host code, no kernels:
// these produce the inputs of the hot path.
#include <algorithm>
#include <cctype>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "stabkit_b200.h"

namespace {

// ref: proj/include/stabkit/rng.hpp:43-65 (SplitMix64 sequential generator)
struct Seq {
    uint64_t s;
    explicit Seq(uint64_t seed) : s(seed) {}
    uint64_t next() {
        s += 0x9e3779b97f4a7c15ULL; uint64_t z = s;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    }
    uint64_t below(uint64_t b) { return next() % b; }
};

sk_gate mk(uint8_t k, uint32_t a, uint32_t b = 0) { sk_gate g; std::memset(&g, 0, sizeof g); g.kind = k; g.q0 = a; g.q1 = b; return g; }

template <class T> T* dup(const std::vector<T>& v) {
    T* p = static_cast<T*>(std::malloc(std::max<size_t>(1, v.size()) * sizeof(T)));
    if (p && !v.empty()) std::memcpy(p, v.data(), v.size() * sizeof(T));
    return p;
}

bool two(uint8_t k) { return k == SK_CX || k == SK_CZ || k == SK_SWAP; }

}  // namespace

extern "C" void sk_free(void* p) { std::free(p); }

// SPEC:369-383, 399-403.  Rotated surface code, frozen conventions (the SPEC fixes only
// the counts 2d^2-1 / d^2-1 and the neighbour orders):
//   data qubit (r,c), 0<=r,c<d            -> index r*d + c
//   plaquette (i,j), 0<=i,j<=d touches data (i-1,j-1)=NW (i-1,j)=NE (i,j-1)=SW (i,j)=SE
//   type X iff (i+j) even; kept: all interior (1<=i,j<=d-1); top/bottom boundary (i=0|d)
//   X-type with 1<=j<=d-1; left/right boundary (j=0|d) Z-type with 1<=i<=d-1
//   ancilla index d*d + running count in row-major (i,j) scan order
// Round: chunk | H on X ancillas | chunk | 4 CX sub-layers (slot k of the fixed order;
// X: NW,NE,SW,SE ancilla->data ; Z: NW,SW,NE,SE data->ancilla) each its own chunk |
// H on X ancillas | chunk | M on every ancilla in index order.
extern "C" int32_t sk_circuit_surface_code(uint32_t d, uint32_t rounds, int final_data_measure,
                                           uint64_t* n_out, sk_gate** gates_out, size_t* ngates_out,
                                           uint32_t** marks_out, size_t* nmarks_out) {
    if (!n_out || !gates_out || !ngates_out || !marks_out || !nmarks_out) return SK_EARG;
    if (d < 3 || (d % 2) == 0 || rounds < 1) return SK_EARG;
    struct Anc { uint32_t q; bool is_x; int nb[4]; };                // nb: data index or -1, in CX order
    std::vector<Anc> anc;
    uint32_t next = d * d;
    auto data = [&](int r, int c) -> int { return (r >= 0 && c >= 0 && r < int(d) && c < int(d)) ? r * int(d) + c : -1; };
    for (uint32_t i = 0; i <= d; ++i)
        for (uint32_t j = 0; j <= d; ++j) {
            bool is_x = ((i + j) % 2) == 0;
            bool interior = i >= 1 && i <= d - 1 && j >= 1 && j <= d - 1;
            bool tb = (i == 0 || i == d) && j >= 1 && j <= d - 1 && is_x;
            bool lr = (j == 0 || j == d) && i >= 1 && i <= d - 1 && !is_x;
            if (!(interior || tb || lr)) continue;
            int nw = data(int(i) - 1, int(j) - 1), ne = data(int(i) - 1, int(j)), sw = data(int(i), int(j) - 1), se = data(int(i), int(j));
            Anc a; a.q = next++; a.is_x = is_x;
            if (is_x) { a.nb[0] = nw; a.nb[1] = ne; a.nb[2] = sw; a.nb[3] = se; }
            else      { a.nb[0] = nw; a.nb[1] = sw; a.nb[2] = ne; a.nb[3] = se; }
            anc.push_back(a);
        }
    if (next != 2 * d * d - 1) return SK_EINVARIANT;
    std::vector<sk_gate> g; std::vector<uint32_t> marks;
    auto mark = [&] { if (!g.empty() && (marks.empty() || marks.back() != g.size())) marks.push_back(uint32_t(g.size())); };
    for (uint32_t r = 0; r < rounds; ++r) {
        mark();
        for (auto& a : anc) if (a.is_x) g.push_back(mk(SK_H, a.q));
        for (int k = 0; k < 4; ++k) {
            mark();
            for (auto& a : anc) {
                if (a.nb[k] < 0) continue;
                if (a.is_x) g.push_back(mk(SK_CX, a.q, uint32_t(a.nb[k])));
                else g.push_back(mk(SK_CX, uint32_t(a.nb[k]), a.q));
            }
        }
        mark();
        for (auto& a : anc) if (a.is_x) g.push_back(mk(SK_H, a.q));
        mark();
        for (auto& a : anc) g.push_back(mk(SK_M, a.q));
    }
    if (final_data_measure) { mark(); for (uint32_t q = 0; q < d * d; ++q) g.push_back(mk(SK_M, q)); }
    *n_out = next; *gates_out = dup(g); *ngates_out = g.size(); *marks_out = dup(marks); *nmarks_out = marks.size();
    return (*gates_out && *marks_out) ? SK_OK : SK_ECUDA;
}

// SPEC:385-393.  Layer l < floor(log2 n): for i < n/2: H or S on qubit i (next()&1 ? S : H);
// chunk; CX(i, i+n/2); chunk; measure ceil(0.2*n/2) (min 1) distinct second-half qubits,
// drawn by a partial Fisher-Yates shuffle with below().
extern "C" int32_t sk_circuit_random_layered(uint64_t n, uint64_t seed, sk_gate** gates_out, size_t* ngates_out,
                                             uint32_t** marks_out, size_t* nmarks_out) {
    if (!gates_out || !ngates_out || !marks_out || !nmarks_out) return SK_EARG;
    if (n < 4 || (n % 2) != 0 || n > (1u << 20)) return SK_EARG;
    const uint32_t half = uint32_t(n / 2);
    uint32_t layers = 0; while ((2ull << layers) <= n) ++layers;      // floor(log2 n)
    const uint32_t nm = std::max<uint32_t>(1, (half + 4) / 5);          // ceil(0.2 * half)
    Seq rng(seed);
    std::vector<sk_gate> g; std::vector<uint32_t> marks;
    auto mark = [&] { if (!g.empty() && (marks.empty() || marks.back() != g.size())) marks.push_back(uint32_t(g.size())); };
    std::vector<uint32_t> perm(half);
    for (uint32_t l = 0; l < layers; ++l) {
        mark();
        for (uint32_t i = 0; i < half; ++i) g.push_back(mk((rng.next() & 1) ? SK_S : SK_H, i));
        mark();
        for (uint32_t i = 0; i < half; ++i) g.push_back(mk(SK_CX, i, i + half));
        mark();
        for (uint32_t i = 0; i < half; ++i) perm[i] = half + i;
        for (uint32_t k = 0; k < nm; ++k) {
            uint32_t j = k + uint32_t(rng.below(half - k));
            std::swap(perm[k], perm[j]);
            g.push_back(mk(SK_M, perm[k]));
        }
    }
    *gates_out = dup(g); *ngates_out = g.size(); *marks_out = dup(marks); *nmarks_out = marks.size();
    return (*gates_out && *marks_out) ? SK_OK : SK_ECUDA;
}

// SPEC:242-250 parse_native.
extern "C" int32_t sk_circuit_parse_native(const char* text, size_t len, uint64_t* n_out, sk_gate** gates_out,
                                           size_t* ngates_out, uint32_t** marks_out, size_t* nmarks_out,
                                           size_t* err_line, char* err_msg, size_t err_cap) {
    if (!text || !n_out || !gates_out || !ngates_out || !marks_out || !nmarks_out) return SK_EARG;
    auto fail = [&](size_t line, const std::string& what) {
        if (err_line) *err_line = line;
        if (err_msg && err_cap) { std::snprintf(err_msg, err_cap, "%s", what.c_str()); }
        return int32_t(SK_EPARSE);
    };
    static const struct { const char* name; uint8_t kind; int arity; } table[] = {
        {"h", SK_H, 1}, {"s", SK_S, 1}, {"sdg", SK_SDG, 1}, {"x", SK_X, 1}, {"y", SK_Y, 1}, {"z", SK_Z, 1},
        {"cx", SK_CX, 2}, {"cz", SK_CZ, 2}, {"swap", SK_SWAP, 2}, {"m", SK_M, 1}, {"t", SK_T, 1}, {"tdg", SK_TDG, 1}};
    std::vector<sk_gate> g; std::vector<uint32_t> marks;
    bool have_header = false; uint64_t n = 0;
    size_t pos = 0, line = 0;
    while (pos <= len) {
        size_t end = pos;
        while (end < len && text[end] != '\n') ++end;
        ++line;
        std::string s(text + pos, end - pos);
        pos = end + 1;
        size_t hash = s.find('#');
        if (hash != std::string::npos) s.erase(hash);
        std::vector<std::string> tok;
        size_t i = 0;
        while (i < s.size()) {
            while (i < s.size() && std::isspace((unsigned char)s[i])) ++i;
            size_t j = i;
            while (j < s.size() && !std::isspace((unsigned char)s[j])) ++j;
            if (j > i) tok.push_back(s.substr(i, j - i));
            i = j;
        }
        if (tok.empty()) { if (end >= len) break; continue; }
        auto parse_u = [&](const std::string& t, uint64_t* v) {
            if (t.empty() || t.size() > 12) return false;
            uint64_t x = 0;
            for (char c : t) { if (c < '0' || c > '9') return false; x = x * 10 + uint64_t(c - '0'); }
            *v = x; return true;
        };
        if (tok[0] == "qubits") {
            if (have_header) return fail(line, "duplicate 'qubits' header");
            if (tok.size() != 2 || !parse_u(tok[1], &n) || n == 0) return fail(line, "expected 'qubits <n>' with n >= 1");
            have_header = true;
        } else {
            if (!have_header) return fail(line, "missing 'qubits <n>' header before the first gate");
            if (tok[0] == "chunk") {
                if (tok.size() != 1) return fail(line, "'chunk' takes no operands");
                if (!g.empty() && (marks.empty() || marks.back() != g.size())) marks.push_back(uint32_t(g.size()));
            } else {
                int found = -1;
                for (int k = 0; k < 12; ++k) if (tok[0] == table[k].name) found = k;
                if (found < 0) return fail(line, "unknown mnemonic '" + tok[0] + "'");
                if (int(tok.size()) != 1 + table[found].arity)
                    return fail(line, "'" + tok[0] + "' expects " + std::to_string(table[found].arity) + " operand(s)");
                uint64_t q[2] = {0, 0};
                for (int k = 0; k < table[found].arity; ++k) {
                    if (!parse_u(tok[1 + k], &q[k])) return fail(line, "bad qubit index '" + tok[1 + k] + "'");
                    if (q[k] >= n) return fail(line, "qubit index " + tok[1 + k] + " out of range for " + std::to_string(n) + " qubits");
                }
                if (table[found].arity == 2 && q[0] == q[1]) return fail(line, "two-qubit gate on duplicate qubit " + tok[1]);
                g.push_back(mk(table[found].kind, uint32_t(q[0]), uint32_t(q[1])));
            }
        }
        if (end >= len) break;
    }
    if (!have_header) return fail(line ? line : 1, "missing 'qubits <n>' header");
    while (!marks.empty() && marks.back() >= g.size()) marks.pop_back();   // marks must be < gate count
    *n_out = n; *gates_out = dup(g); *ngates_out = g.size(); *marks_out = dup(marks); *nmarks_out = marks.size();
    if (err_line) *err_line = 0;
    return (*gates_out && *marks_out) ? SK_OK : SK_ECUDA;
}

// SPEC:252-260 parse_qasm2_subset: OPENQASM 2.0 header, one qreg, optional cregs, gates {h,s,sdg,x,y,z,cx,cz,swap,t,tdg},
// `measure q[i] -> c[j];` -> M, `barrier` -> chunk mark; a bare register name applies the statement to every qubit.
// Unsupported constructs (second qreg, parameterised / unknown gates, `if`, `gate`, `reset`, `opaque`) -> SK_EUNSUPPORTED with
// the construct and its line in err_msg; malformed text -> SK_EPARSE.
extern "C" int32_t sk_circuit_parse_qasm2(const char* text, size_t len, uint64_t* n_out, sk_gate** gates_out,
                                          size_t* ngates_out, uint32_t** marks_out, size_t* nmarks_out,
                                          size_t* err_line, char* err_msg, size_t err_cap) {
    if (!text || !n_out || !gates_out || !ngates_out || !marks_out || !nmarks_out) return SK_EARG;
    auto fail = [&](int32_t code, size_t line, const std::string& what) {
        if (err_line) *err_line = line;
        if (err_msg && err_cap) { std::snprintf(err_msg, err_cap, "%s", what.c_str()); }
        return code;
    };
    static const struct { const char* name; uint8_t kind; int arity; } table[] = {
        {"h", SK_H, 1}, {"s", SK_S, 1}, {"sdg", SK_SDG, 1}, {"x", SK_X, 1}, {"y", SK_Y, 1}, {"z", SK_Z, 1},
        {"cx", SK_CX, 2}, {"CX", SK_CX, 2}, {"cz", SK_CZ, 2}, {"swap", SK_SWAP, 2}, {"t", SK_T, 1}, {"tdg", SK_TDG, 1}};
    std::vector<sk_gate> g; std::vector<uint32_t> marks;
    std::string qname; uint64_t n = 0; bool have_q = false;
    std::vector<std::string> cregs;
    // strip // comments, then split into ';'-terminated statements remembering the line each one starts on
    std::string src(text, len);
    for (size_t i = 0; i + 1 < src.size(); ++i)
        if (src[i] == '/' && src[i + 1] == '/') { while (i < src.size() && src[i] != '\n') src[i++] = ' '; }
    size_t line = 1, pos = 0;
    auto is_id = [](char c) { return std::isalnum((unsigned char)c) || c == '_'; };
    // operand "name" or "name[idx]" -> (name, idx or -1)
    auto operand = [&](std::string t, std::string* name, long long* idx) {
        size_t a = 0; while (a < t.size() && std::isspace((unsigned char)t[a])) ++a;
        size_t b = t.size(); while (b > a && std::isspace((unsigned char)t[b - 1])) --b;
        t = t.substr(a, b - a);
        size_t lb = t.find('[');
        if (lb == std::string::npos) { *name = t; *idx = -1; for (char c : t) if (!is_id(c)) return false; return !t.empty(); }
        if (t.back() != ']') return false;
        *name = t.substr(0, lb);
        for (char c : *name) if (!is_id(c)) return false;
        std::string num = t.substr(lb + 1, t.size() - lb - 2);
        if (name->empty() || num.empty() || num.size() > 12) return false;
        long long v = 0; for (char c : num) { if (c < '0' || c > '9') return false; v = v * 10 + (c - '0'); }
        *idx = v; return true;
    };
    while (pos < src.size()) {
        while (pos < src.size() && std::isspace((unsigned char)src[pos])) { if (src[pos] == '\n') ++line; ++pos; }
        if (pos >= src.size()) break;
        const size_t sline = line;
        size_t end = pos;
        while (end < src.size() && src[end] != ';') { if (src[end] == '\n') ++line; if (src[end] == '{') break; ++end; }
        std::string st = src.substr(pos, end - pos);
        if (end < src.size() && src[end] == '{') return fail(SK_EUNSUPPORTED, sline, "unsupported construct: block statement '" + st.substr(0, st.find_first_of(" \t\n")) + "' (line " + std::to_string(sline) + ")");
        if (end >= src.size()) return fail(SK_EPARSE, sline, "statement is not terminated by ';'");
        pos = end + 1;
        for (char& c : st) if (c == '\n' || c == '\t' || c == '\r') c = ' ';
        size_t k = 0; while (k < st.size() && (is_id(st[k]) || st[k] == '.')) ++k;
        const std::string head = st.substr(0, k);
        std::string rest = st.substr(k);
        if (head == "OPENQASM") { if (rest.find("2.0") == std::string::npos) return fail(SK_EUNSUPPORTED, sline, "unsupported construct: OPENQASM version" + rest + " (line " + std::to_string(sline) + ")"); continue; }
        if (head == "include") continue;
        if (head == "qreg" || head == "creg") {
            std::string name; long long sz = -1;
            if (!operand(rest, &name, &sz) || sz <= 0) return fail(SK_EPARSE, sline, "expected '" + head + " name[size]'");
            if (head == "qreg") {
                if (have_q) return fail(SK_EUNSUPPORTED, sline, "unsupported construct: multiple qregs ('" + name + "', line " + std::to_string(sline) + ")");
                have_q = true; qname = name; n = uint64_t(sz);
            } else cregs.push_back(name);
            continue;
        }
        if (head == "if" || head == "gate" || head == "opaque" || head == "reset" || head == "U" || head == "u1" || head == "u2" || head == "u3")
            return fail(SK_EUNSUPPORTED, sline, "unsupported construct: '" + head + "' (line " + std::to_string(sline) + ")");
        if (!rest.empty() && rest.find('(') != std::string::npos && head != "measure")
            return fail(SK_EUNSUPPORTED, sline, "unsupported construct: parameterised gate '" + head + "' (line " + std::to_string(sline) + ")");
        if (!have_q) return fail(SK_EPARSE, sline, "statement before the qreg declaration");
        auto qubit = [&](const std::string& t, long long* idx) -> int32_t {
            std::string name;
            if (!operand(t, &name, idx)) return SK_EPARSE;
            if (name != qname) return SK_EPARSE;
            if (*idx >= (long long)n) return SK_EDIM;
            return SK_OK;
        };
        if (head == "barrier") {
            if (!g.empty() && (marks.empty() || marks.back() != g.size())) marks.push_back(uint32_t(g.size()));
            continue;
        }
        if (head == "measure") {
            size_t arrow = rest.find("->");
            if (arrow == std::string::npos) return fail(SK_EPARSE, sline, "expected 'measure q[i] -> c[j]'");
            long long qi = -1, ci = -1; std::string cname;
            int32_t rc = qubit(rest.substr(0, arrow), &qi);
            if (rc == SK_EDIM) return fail(SK_EPARSE, sline, "qubit index out of range in 'measure'");
            if (rc || !operand(rest.substr(arrow + 2), &cname, &ci)) return fail(SK_EPARSE, sline, "expected 'measure q[i] -> c[j]'");
            bool known = false; for (const std::string& c : cregs) known |= (c == cname);
            if (!known) return fail(SK_EPARSE, sline, "measure into undeclared creg '" + cname + "'");
            if (qi < 0) { for (uint64_t q = 0; q < n; ++q) g.push_back(mk(SK_M, uint32_t(q), 0)); }
            else g.push_back(mk(SK_M, uint32_t(qi), 0));
            continue;
        }
        int found = -1;
        for (int t = 0; t < 12; ++t) if (head == table[t].name) found = t;
        if (found < 0) return fail(SK_EUNSUPPORTED, sline, "unsupported construct: gate '" + head + "' (line " + std::to_string(sline) + ")");
        std::vector<std::string> ops;
        { size_t a = 0; while (true) { size_t c = rest.find(',', a); ops.push_back(rest.substr(a, c == std::string::npos ? std::string::npos : c - a)); if (c == std::string::npos) break; a = c + 1; } }
        if (int(ops.size()) != table[found].arity) return fail(SK_EPARSE, sline, "'" + head + "' expects " + std::to_string(table[found].arity) + " operand(s)");
        long long q[2] = {0, 0};
        for (int t = 0; t < table[found].arity; ++t) {
            int32_t rc = qubit(ops[t], &q[t]);
            if (rc == SK_EDIM) return fail(SK_EPARSE, sline, "qubit index out of range for " + std::to_string(n) + " qubits");
            if (rc) return fail(SK_EPARSE, sline, "bad operand '" + ops[t] + "'");
        }
        if (table[found].arity == 1) {
            if (q[0] < 0) { for (uint64_t v = 0; v < n; ++v) g.push_back(mk(table[found].kind, uint32_t(v), 0)); }
            else g.push_back(mk(table[found].kind, uint32_t(q[0]), 0));
        } else {
            if (q[0] < 0 || q[1] < 0) return fail(SK_EUNSUPPORTED, sline, "unsupported construct: register-wide two-qubit gate (line " + std::to_string(sline) + ")");
            if (q[0] == q[1]) return fail(SK_EPARSE, sline, "two-qubit gate on duplicate qubit");
            g.push_back(mk(table[found].kind, uint32_t(q[0]), uint32_t(q[1])));
        }
    }
    if (!have_q) return fail(SK_EPARSE, line, "missing qreg declaration");
    while (!marks.empty() && marks.back() >= g.size()) marks.pop_back();
    *n_out = n; *gates_out = dup(g); *ngates_out = g.size(); *marks_out = dup(marks); *nmarks_out = marks.size();
    if (err_line) *err_line = 0;
    return (*gates_out && *marks_out) ? SK_OK : SK_ECUDA;
}

// SPEC:262-270 validate_chunks.  A chunk made of measurements ONLY is a measurement barrier region, not a chunk "intended for
// sim2d": every M is a full barrier in both engines, so there is nothing to run concurrently and
// nothing to fall back from.  Such chunks are not reported -- that is what makes SPEC:397 hold ("surface_code_circuit passes
// validate_chunks for all emitted chunks"; the generators put every M block in a chunk of its own).  A measurement inside a
// chunk that also holds Clifford gates is a violation.  SK_CHUNKS_STRICT reports measurement-only chunks as well, the literal
// reading of SPEC:270's third example.
extern "C" int32_t sk_circuit_validate_chunks_ex(uint64_t n, const sk_gate* gates, size_t ngates,
                                                 const uint32_t* marks, size_t nmarks, uint32_t flags,
                                                 uint32_t** viol_chunk, uint32_t** viol_gate, uint8_t** viol_kind, size_t* nviol) {
    if ((!gates && ngates) || (!marks && nmarks) || !viol_chunk || !viol_gate || !viol_kind || !nviol) return SK_EARG;
    const bool strict = (flags & SK_CHUNKS_STRICT) != 0;
    std::vector<uint32_t> vc, vg; std::vector<uint8_t> vk;
    std::vector<uint32_t> seen(n, 0);
    size_t lo = 0; uint32_t chunk = 0;
    for (size_t k = 0; k <= nmarks; ++k) {
        size_t hi = (k < nmarks) ? marks[k] : ngates;
        if (hi > ngates || hi < lo) return SK_EARG;
        ++chunk;    // stamp = chunk index + 1
        bool only_m = true;
        for (size_t i = lo; i < hi && only_m; ++i) only_m = gates[i].kind == SK_M;
        for (size_t i = lo; i < hi; ++i) {
            if (gates[i].q0 >= n || (two(gates[i].kind) && gates[i].q1 >= n)) return SK_EDIM;
            if (gates[i].kind == SK_M && (strict || !only_m)) { vc.push_back(chunk - 1); vg.push_back(uint32_t(i)); vk.push_back(2); }
            if (only_m) continue;                            // sequential by definition: repeated qubits are not collisions
            bool coll = seen[gates[i].q0] == chunk;
            seen[gates[i].q0] = chunk;
            if (two(gates[i].kind)) { coll = coll || seen[gates[i].q1] == chunk; seen[gates[i].q1] = chunk; }
            if (coll) { vc.push_back(chunk - 1); vg.push_back(uint32_t(i)); vk.push_back(1); }
        }
        lo = hi;
    }
    *viol_chunk = dup(vc); *viol_gate = dup(vg); *viol_kind = dup(vk); *nviol = vc.size();
    return SK_OK;
}

extern "C" int32_t sk_circuit_validate_chunks(uint64_t n, const sk_gate* gates, size_t ngates,
                                              const uint32_t* marks, size_t nmarks,
                                              uint32_t** viol_chunk, uint32_t** viol_gate, uint8_t** viol_kind, size_t* nviol) {
    return sk_circuit_validate_chunks_ex(n, gates, ngates, marks, nmarks, 0u, viol_chunk, viol_gate, viol_kind, nviol);
}
