// stabkit/engine.hpp -- sim / sim2d.  The device engine fuses Clifford runs into
// layers and executes measurement runs in one persistent kernel; results are bit-identical to
// gate-by-gate CHP for every seed (schedule independence).
#pragma once
#include <vector>

#include "stabkit/tableau.hpp"

namespace stabkit {

// SPEC:304-307.  `workers` is kept for API compatibility; the device engine ignores it
// (row parallelism is the GPU's).  `audit` checks the tableau invariants of SPEC:111-116 on the device after the run
// (sk_tableau_audit: every row pair has the symplectic product the CHP form demands) and throws InvariantError otherwise.
struct EngineConfig { size_t workers = 1; uint64_t seed = 0; bool audit = false; };

// SPEC:299-302
struct MeasurementEntry { size_t gate_index; uint32_t qubit; bool outcome; bool deterministic; };
using MeasurementRecord = std::vector<MeasurementEntry>;

struct SimResult { Tableau tableau; MeasurementRecord record; bool chunk_fallback = false; };

namespace detail {
inline SimResult run(const Circuit& c, const EngineConfig& cfg, int mode) {
    if (cfg.workers < 1) throw Error("EngineConfig.workers must be >= 1 (SPEC:306)");
    Device& d = Device::instance();
    const size_t nm = c.num_measurements();
    std::vector<uint8_t> o(nm + 1), det(nm + 1);
    sk_tableau* t = nullptr; uint32_t warn = 0;
    d.check(sk_sim(d.ctx(), c.n, c.raw(), c.gates.size(), c.chunk_marks.data(), c.chunk_marks.size(), mode, cfg.seed, &t, o.data(), det.data(), &warn));
    if (cfg.audit) {
        uint64_t bad = 0;
        const int32_t rc = sk_tableau_audit(t, &bad);
        if (rc || bad) { sk_tableau_destroy(t); d.check(rc); throw InvariantError("audit: " + std::to_string(bad) + " row pairs violate the tableau invariants (SPEC:111-116)"); }
    }
    SimResult r{Tableau(c.n, t), {}, (warn & 1u) != 0};
    r.record.reserve(nm);
    size_t k = 0;
    for (size_t i = 0; i < c.gates.size(); ++i)
        if (c.gates[i].kind == GateKind::M) { r.record.push_back({i, c.gates[i].q0, o[k] != 0, det[k] != 0}); ++k; }
    return r;
}
}  // namespace detail

// SPEC:310-318; T/TDG throw UnsupportedError
inline SimResult sim(const Circuit& c, const EngineConfig& cfg) { return detail::run(c, cfg, 0); }
// SPEC:320-328; chunk_size_hint is advisory
inline SimResult sim2d(const Circuit& c, size_t /*chunk_size_hint*/, const EngineConfig& cfg) { return detail::run(c, cfg, 1); }

// per-measurement-site counts of outcome 1 over `shots` runs, shot s seeded cfg.seed ^ s.
// The circuit is compiled once and stays on the device; counts are accumulated there.
struct ShotHistogram { uint64_t shots = 0; std::vector<uint32_t> ones; std::vector<std::vector<uint8_t>> records; };
inline ShotHistogram run_shots(const Circuit& c, uint64_t shots, const EngineConfig& cfg, bool keep_records = false) {
    if (shots < 1) throw Error("run_shots: shots must be >= 1 (SPEC:332)");
    Device& d = Device::instance();
    sk_program* p = nullptr; sk_tableau* t = nullptr; uint32_t warn = 0;
    d.check(sk_program_create(d.ctx(), c.n, c.raw(), c.gates.size(), c.chunk_marks.data(), c.chunk_marks.size(), 0, &p, &warn));
    const int32_t rc_t = sk_tableau_create(d.ctx(), c.n, &t);
    if (rc_t) { sk_program_destroy(p); d.check(rc_t); }
    const size_t nm = c.num_measurements();
    ShotHistogram h; h.shots = shots; h.ones.assign(nm + 1, 0);
    std::vector<uint8_t> flat(keep_records ? shots * nm + 1 : 0);
    const int32_t rc = sk_program_run_shots(p, t, shots, cfg.seed, h.ones.data(), keep_records ? flat.data() : nullptr);
    sk_tableau_destroy(t); sk_program_destroy(p);
    d.check(rc);
    h.ones.resize(nm);
    if (keep_records) for (uint64_t s = 0; s < shots; ++s) h.records.emplace_back(flat.begin() + s * nm, flat.begin() + (s + 1) * nm);
    return h;
}

}  // namespace stabkit
