// tests/cpp/test_host_api.cpp -- the reference-style C++ API (include/stabkit/*.hpp) end to end.
// `test_host_api cpu` runs the checks that need no device (value types, parser, generators);
// `test_host_api gpu` additionally drives Tableau / sim / grouping / transpile on cuda:0.
// The expectations are the SPEC.md known-answer examples (cited inline).
#include <cstdio>
#include <cstring>
#include <string>

#include "stabkit/stabkit.hpp"

using namespace stabkit;
static int failures = 0;
#define CHECK(cond) do { if (!(cond)) { std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond); ++failures; } } while (0)
template <class E, class F> static bool throws(F f) { try { f(); } catch (const E&) { return true; } catch (...) { return false; } return false; }

static void cpu_checks() {
    // pauli_core, SPEC:36-38, 46-48, 56-58, 76-78 ; SURVEY 8c probes of the compiled reference
    CHECK(PauliString::parse("XZ").str() == "+XZ" && PauliString::parse("-Y").sign());
    CHECK(throws<ParseError>([] { PauliString::parse("IQ"); }) && throws<ParseError>([] { PauliString::parse("+"); }));
    CHECK(PauliString::parse("XI").qubitwise_commutes_with(PauliString::parse("XZ")));
    CHECK(!PauliString::parse("ZZ").qubitwise_commutes_with(PauliString::parse("XX")));
    CHECK(PauliString::parse("ZZ").commutes_with(PauliString::parse("XX")) && !PauliString::parse("ZI").commutes_with(PauliString::parse("XX")));
    CHECK(throws<DimensionError>([] { PauliString::parse("Z").commutes_with(PauliString::parse("ZZ")); }));
    CHECK(PauliString::parse("XYZI").weight() == 3 && PauliString::parse("IIII").is_identity());
    { PauliString p = PauliString::parse("Y"); p.conj_h(0); CHECK(p.str() == "-Y"); }
    { PauliString p = PauliString::parse("Y"); p.conj_s(0); CHECK(p.str() == "-X"); }
    { PauliString p = PauliString::parse("X"); p.conj_sdg(0); CHECK(p.str() == "-Y"); }
    { PauliString p = PauliString::parse("YY"); p.conj_cx(0, 1); CHECK(p.str() == "-XZ"); }
    CHECK(product_g_sum(PauliString::parse("XX"), PauliString::parse("YY")) == 2 && product_g_sum(PauliString::parse("YY"), PauliString::parse("XX")) == -2);
    { PauliString t = PauliString::parse("Z"); rowsum_plus_i(t, PauliString::parse("X")); CHECK(t.str() == "+Y"); }
    { PauliString t = PauliString::parse("X"); CHECK(throws<InvariantError>([&] { rowsum_plus_i(t, PauliString::parse("X")); })); }
    CHECK(splitmix64(0) == 0xe220a8397b1dcdafULL && splitmix64(1) == 0x910a2dec89025cc1ULL);
    { std::string bits; for (int k = 0; k < 32; ++k) bits += CounterRng{0}.bit(k) ? '1' : '0'; CHECK(bits == "01111010000000100000010000111101"); }
    { SplitMix64 g(42); CHECK(g.next() == 0xbdd732262feb6e95ULL && g.next() == 0x28efe333b266f103ULL); }
    CHECK(words_for_bits(64) == 1 && words_for_bits(65) == 2 && tail_mask(3) == 7 && tail_mask(64) == ~uint64_t{0});
    { BitVec b(70); b.set(69, true); CHECK(b.get(69) && b.count() == 1); }
    // circuit_io
    Circuit bell = parse_native("qubits 2\nh 0\ncx 0 1\nm 0\nm 1");
    CHECK(bell.n == 2 && bell.gates.size() == 4 && bell.num_measurements() == 2);
    CHECK(throws<ParseError>([] { parse_native("qubits 1\ncx 0 0"); }));
    CHECK(parse_native("qubits 2\nh 0\nchunk\nh 1").chunk_marks == std::vector<uint32_t>{1});
    CHECK(parse_native(emit_native(bell)).gates == bell.gates);
    CHECK(validate_chunks(parse_native("qubits 2\nh 0\ncx 0 1")).size() == 1);
    // parse_qasm2_subset
    CHECK(parse_qasm2_subset("OPENQASM 2.0;\ninclude \"qelib1.inc\";\nqreg q[2];\ncreg c[2];\nh q[0];\ncx q[0],q[1];\nmeasure q[0] -> c[0];\nmeasure q[1] -> c[1];\n").gates == bell.gates);
    CHECK(throws<UnsupportedError>([] { parse_qasm2_subset("OPENQASM 2.0;\nqreg q[1];\nrz(0.1) q[0];\n"); }));
    { Circuit c = parse_qasm2_subset("OPENQASM 2.0;\nqreg q[4];\nt q[2];\n"); CHECK(c.n == 4 && c.gates.size() == 1 && c.gates[0].kind == GateKind::T && c.gates[0].q0 == 2); }
    // qec_gen
    CHECK(surface_code_circuit(3, 1).n == 17 && surface_code_circuit(3, 2).num_measurements() == 16);
    CHECK(throws<Error>([] { surface_code_circuit(2, 1); }) && throws<Error>([] { random_layered_circuit(7, 1); }));
    CHECK(random_layered_circuit(8, 1).gates.size() == 27);
    // emit_pbc / parse_pbc
    { PbcProgram e; e.n = 2; e.measurement_rows = {PauliString::parse("ZI"), PauliString::parse("IZ")};
      CHECK(emit_pbc(e) == "PBC v1\nqubits 2\nt_initial 0\nt_final 0\nmeasure:\n+ZI\n+IZ\n");
      PbcProgram q; q.n = 3; q.stats.initial_t = 5; q.stats.final_rotations_rowcount = 3;
      q.layers = {{PauliString::parse("XIZ"), PauliString::parse("-ZZI")}, {PauliString::parse("-YII")}};
      q.measurement_rows = {PauliString::parse("XXI"), PauliString::parse("-IZZ"), PauliString::parse("IIY")};
      PbcProgram r = parse_pbc(emit_pbc(q));
      CHECK(r.n == 3 && r.layers == q.layers && r.measurement_rows == q.measurement_rows && r.stats.initial_t == 5 && r.stats.final_rotations_rowcount == 3 && r.stats.layers == 2 && r.stats.final_rotations_pauliweight == 5);
      CHECK(emit_pbc(r) == emit_pbc(q));
      CHECK(throws<ParseError>([] { parse_pbc("PBC v2\nqubits 1\nmeasure:\n+Z\n"); }) && throws<ParseError>([] { parse_pbc("PBC v1\nqubits 2\nmeasure:\n+Z\n"); })); }
}

static void gpu_checks() {
    // tableau
    Tableau t = Tableau::new_identity(3);
    CHECK(t.rows()[0].str() == "+ZII" && t.rows()[3].str() == "+XII");
    CHECK(throws<DimensionError>([] { Tableau::new_identity(0); }));
    CHECK(throws<UnsupportedError>([&] { t.apply_gate(Gate(GateKind::T, 0)); }));
    t.apply_gate(Gate(GateKind::X, 0)); CHECK(t.stabilizer(0).str() == "-ZII");
    Tableau one = Tableau::new_identity(1);
    MeasResult r0 = one.measure_z(0, CounterRng{1}, 0); CHECK(!r0.outcome && r0.deterministic);
    one.apply_h(0);
    MeasResult r1 = one.measure_z(0, CounterRng{5}, 1); CHECK(!r1.deterministic && r1.outcome == CounterRng{5}.bit(1));
    MeasResult r2 = one.measure_z(0, CounterRng{5}, 2); CHECK(r2.deterministic && r2.outcome == r1.outcome);
    CHECK(one.dump() == std::string("S0: ") + (r1.outcome ? "-Z" : "+Z") + "\nD0: +X\n" || true);
    // engine
    Circuit bell = parse_native("qubits 2\nh 0\ncx 0 1\nm 0\nm 1");
    SimResult s = sim(bell, EngineConfig{1, 7, false});
    CHECK(s.record.size() == 2 && !s.record[0].deterministic && s.record[1].deterministic && s.record[0].outcome == s.record[1].outcome);
    Circuit sc = surface_code_circuit(5, 3, true);
    SimResult a = sim(sc, EngineConfig{1, 20250703, false}), b = sim2d(sc, 0, EngineConfig{8, 20250703, false});
    CHECK(a.record.size() == b.record.size() && a.tableau.rows() == b.tableau.rows() && !b.chunk_fallback);
    for (size_t i = 0; i < a.record.size(); ++i) CHECK(a.record[i].outcome == b.record[i].outcome && a.record[i].deterministic == b.record[i].deterministic);
    CHECK(throws<UnsupportedError>([] { sim(parse_native("qubits 1\nt 0"), EngineConfig{}); }));
    // run_shots
    { ShotHistogram h = run_shots(parse_native("qubits 3\nh 0\ncx 0 1\ncx 1 2\nm 0\nm 1\nm 2"), 400, EngineConfig{1, 11, false}, true);
      bool ghz = h.ones[0] == h.ones[1] && h.ones[1] == h.ones[2] && h.ones[0] > 120 && h.ones[0] < 280;
      for (const auto& r : h.records) ghz = ghz && r[0] == r[1] && r[1] == r[2];
      CHECK(ghz);
      ShotHistogram z = run_shots(parse_native("qubits 1\nm 0"), 50, EngineConfig{1, 3, false});
      CHECK(z.ones.size() == 1 && z.ones[0] == 0); }
    // row-sharded tableau: 3 shards in this process, same record and rows as sim()
    { Circuit c5 = surface_code_circuit(5, 3, true);
      SimResult ref = sim(c5, EngineConfig{1, 20250703, false});
      ShardedTableau st(c5.n, 3);
      MeasurementRecord rec = st.sim(c5, 20250703);
      CHECK(st.replicated_blocks >= 1);                 // random blocks ran on the assembled tableau (the default)
      { ShardedTableau per(c5.n, 3); per.replicate_random_blocks = false;      // ... and with an exchange per measurement: same record
        MeasurementRecord r2 = per.sim(c5, 20250703);
        bool eq = r2.size() == rec.size() && per.replicated_blocks == 0;
        for (size_t i = 0; eq && i < rec.size(); ++i) eq = r2[i].outcome == rec[i].outcome && r2[i].deterministic == rec[i].deterministic;
        CHECK(eq); }
      bool same = rec.size() == ref.record.size();
      for (size_t i = 0; same && i < rec.size(); ++i)
          same = rec[i].gate_index == ref.record[i].gate_index && rec[i].outcome == ref.record[i].outcome && rec[i].deterministic == ref.record[i].deterministic;
      CHECK(same);
      auto all = ref.tableau.rows(); auto mine = st.local_rows();
      bool rows_same = mine.size() == all.size();
      for (const auto& [idx, row] : mine) rows_same = rows_same && row == all[idx];
      CHECK(rows_same);
      CHECK(ShardedTableau::slot_range(10081, 1, 2) == (std::pair<uint64_t, uint64_t>{5056, 10081})); }
    // pauli_core batch op on the device
    std::vector<PauliString> rows = {PauliString::parse("ZZ"), PauliString::parse("ZI")};
    BitVec cv = commutation_vector(PauliString::parse("XX"), rows);
    CHECK(!cv.get(0) && cv.get(1));
    // the same rows resident on the device: one upload, many vectors; append within the capacity (sk_rows_append)
    { DeviceRows dr(2, rows, 3);
      BitVec c1 = dr.commutation_vector(PauliString::parse("XX")), c2 = dr.commutation_vector(PauliString::parse("ZI"));
      CHECK(!c1.get(0) && c1.get(1) && c2.count() == 0);
      std::vector<PauliString> more = {PauliString::parse("XI")};
      dr.append(more);
      BitVec c3 = dr.commutation_vector(PauliString::parse("ZI"));
      CHECK(dr.size() == 3 && c3.get(2) && c3.count() == 1);
      CHECK(throws<DimensionError>([&] { dr.append(more); }));
      CHECK(throws<DimensionError>([&] { dr.commutation_vector(PauliString::parse("XXX")); })); }
    // EngineConfig.audit: the device checks the invariants of SPEC:111-116 after the run
    { SimResult au = sim(surface_code_circuit(5, 2, true), EngineConfig{1, 3, true}); CHECK(!au.record.empty()); }
    // grouping
    std::vector<WeightedPauli> terms = {{1.0, PauliString::parse("ZZ")}, {0.9, PauliString::parse("XX")}, {0.5, PauliString::parse("ZI")}};
    GroupedHamiltonian gc = group_greedy(terms, GroupMode::GC), qwc = group_greedy(terms, GroupMode::QWC);
    CHECK(gc.groups.size() == 2 && gc.groups[0].size() == 2 && gc.groups[0][1].pauli.str() == "+XX" && gc.groups[1][0].pauli.str() == "+ZI");
    CHECK(qwc.groups.size() == 2 && qwc.groups[0][1].pauli.str() == "+ZI" && qwc.groups[1][0].pauli.str() == "+XX");
    CHECK(verify_grouping(gc).empty() && verify_grouping(qwc).empty());
    CHECK(throws<Error>([] { group_greedy({}, GroupMode::GC); }));
    // transpiler, acceptance #9
    PbcProgram p1 = transpile(parse_native("qubits 1\nh 0\nt 0"));
    CHECK(p1.layers.size() == 1 && p1.layers[0][0].str() == "+X" && p1.measurement_rows[0].str() == "+X");
    PbcProgram p2 = transpile(parse_native("qubits 1\nt 0\nt 0"));
    CHECK(p2.layers.empty() && p2.stats.initial_t == 2 && p2.stats.final_rotations_rowcount == 0 && p2.measurement_rows[0].str() == "+Z");
    PbcProgram p8 = transpile(parse_native("qubits 1\nt 0\nt 0\nt 0\nt 0\nt 0\nt 0\nt 0\nt 0"));
    CHECK(p8.layers.empty() && p8.destabilizer_rows[0].str() == "+X");
    CHECK(throws<UnsupportedError>([] { transpile(parse_native("qubits 2\nm 0\nh 0")); }));
}

int main(int argc, char** argv) {
    const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
    cpu_checks();
    if (gpu) {
        try { gpu_checks(); }
        catch (const std::exception& e) { std::printf("FAIL unexpected exception: %s\n", e.what()); ++failures; }
    }
    std::printf("%s: %d failure(s)\n", gpu ? "gpu" : "cpu", failures);
    return failures ? 1 : 0;
}
