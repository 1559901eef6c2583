// stabkit/grouping.hpp -- greedy commuting-group construction.
// Sorting is host logic; the predicate scans and the first-fit run on the device
// (k_conflict_bitmap / k_first_fit_block through sk_group_first_fit).
#pragma once
#include <algorithm>
#include <cmath>
#include <numeric>
#include <vector>

#include "stabkit/device.hpp"
#include "stabkit/pauli.hpp"

namespace stabkit {

enum class GroupMode { GC = 0, QWC = 1 };
struct WeightedPauli { double coeff = 0; PauliString pauli; };
struct GroupedHamiltonian { GroupMode mode = GroupMode::GC; std::vector<std::vector<WeightedPauli>> groups; };
struct GroupViolation { size_t group, a, b; };

// SPEC:444-452
inline GroupedHamiltonian group_greedy(const std::vector<WeightedPauli>& terms, GroupMode mode) {
    if (terms.empty()) throw Error("group_greedy: empty input (SPEC:448)");
    const size_t n = terms[0].pauli.num_qubits();
    std::vector<size_t> order(terms.size());
    std::iota(order.begin(), order.end(), size_t{0});
    std::vector<std::string> text(terms.size());
    for (size_t i = 0; i < terms.size(); ++i) text[i] = terms[i].pauli.str().substr(1);
    std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) {
        const double wa = std::fabs(terms[a].coeff), wb = std::fabs(terms[b].coeff);
        if (wa != wb) return wa > wb;
        return text[a] < text[b];                                              // then input order (stable)
    });
    std::vector<PauliString> sorted; sorted.reserve(terms.size());
    for (size_t i : order) { sorted.push_back(terms[i].pauli); sorted.back().set_sign(false); }
    std::vector<uint64_t> x, z; std::vector<uint8_t> s;
    pack_rows(sorted, n, x, z, s);
    Device& dev = Device::instance();
    sk_rows* r = nullptr;
    dev.check(sk_rows_create(dev.ctx(), n, terms.size(), &r));
    std::vector<uint32_t> gid(terms.size()); uint64_t ng = 0;
    int rc = sk_rows_upload(r, x.data(), z.data(), s.data(), terms.size());
    if (!rc) rc = sk_group_first_fit(r, int(mode), gid.data(), &ng);
    const std::string msg = rc ? sk_last_error(dev.ctx()) : "";
    sk_rows_destroy(r);
    if (rc) throw_status(rc, msg);
    GroupedHamiltonian out; out.mode = mode; out.groups.resize(ng);
    for (size_t k = 0; k < order.size(); ++k) out.groups[gid[k]].push_back(terms[order[k]]);
    return out;
}

// every violating intra-group pair
inline std::vector<GroupViolation> verify_grouping(const GroupedHamiltonian& g) {
    std::vector<GroupViolation> bad;
    for (size_t k = 0; k < g.groups.size(); ++k)
        for (size_t a = 0; a < g.groups[k].size(); ++a)
            for (size_t b = a + 1; b < g.groups[k].size(); ++b) {
                const bool ok = g.mode == GroupMode::GC ? g.groups[k][a].pauli.commutes_with(g.groups[k][b].pauli)
                                                         : g.groups[k][a].pauli.qubitwise_commutes_with(g.groups[k][b].pauli);
                if (!ok) bad.push_back({k, a, b});
            }
    return bad;
}

}  // namespace stabkit
