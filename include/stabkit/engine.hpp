// stabkit/engine.hpp -- sim / sim2d.  The device engine fuses Clifford runs into
// layers and executes measurement runs in one persistent kernel; results are bit-identical to
// gate-by-gate CHP for every seed (schedule independence).
#pragma once
#include <vector>

#include "stabkit/tableau.hpp"

namespace stabkit {

// SPEC:304-307.  `workers` is kept for API compatibility; the device engine ignores it
// (row parallelism is the GPU's), `audit` is accepted and ignored.
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

}  // namespace stabkit
