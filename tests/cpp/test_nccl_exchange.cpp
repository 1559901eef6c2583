// The row-sharded tableau over a real NCCL communicator (stabkit::NcclExchange).  One process per GPU:
//   STABKIT_DEVICE=r RANK=r WORLD_SIZE=N STABKIT_NCCL_ID=/path/shared/by/all/ranks ./test_nccl_exchange [d] [rounds] [local_shards]
// Rank 0 writes the ncclUniqueId to the file, the others wait for it.  WORLD_SIZE=1 (the single-GPU box of this project) still
// goes through ncclAllReduce / ncclBroadcast / ncclAllGather on the library's stream.  Every rank checks its rows and the record
// against the unsharded engine on its own device.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <thread>

#include "stabkit/nccl_exchange.hpp"
#include "stabkit/stabkit.hpp"

using namespace stabkit;

int main(int argc, char** argv) {
    const int rank = std::getenv("RANK") ? std::atoi(std::getenv("RANK")) : 0;
    const int world = std::getenv("WORLD_SIZE") ? std::atoi(std::getenv("WORLD_SIZE")) : 1;
    const char* idfile = std::getenv("STABKIT_NCCL_ID");
    const uint32_t d = argc > 1 ? uint32_t(std::atoi(argv[1])) : 5, rounds = argc > 2 ? uint32_t(std::atoi(argv[2])) : 3;
    const int local = argc > 3 ? std::atoi(argv[3]) : 2;
    try {
        ncclUniqueId id;
        if (rank == 0) {
            id = NcclExchange::make_id();
            if (world > 1) {
                if (!idfile) { std::fprintf(stderr, "STABKIT_NCCL_ID must name a file all ranks can read\n"); return 2; }
                std::ofstream f(std::string(idfile) + ".tmp", std::ios::binary); f.write(reinterpret_cast<const char*>(&id), sizeof id); f.close();
                std::rename((std::string(idfile) + ".tmp").c_str(), idfile);
            }
        } else {
            if (!idfile) { std::fprintf(stderr, "STABKIT_NCCL_ID must name a file all ranks can read\n"); return 2; }
            for (int tries = 0;; ++tries) {
                std::ifstream f(idfile, std::ios::binary);
                if (f && f.read(reinterpret_cast<char*>(&id), sizeof id)) break;
                if (tries > 600) { std::fprintf(stderr, "rank %d: no id file\n", rank); return 2; }
                std::this_thread::sleep_for(std::chrono::milliseconds(100));
            }
        }
        NcclExchange ex(id, rank, world);
        Circuit c = surface_code_circuit(d, rounds, true);
        SimResult ref = sim(c, EngineConfig{1, 20250703, false});
        auto all = ref.tableau.rows();
        for (int per_measurement = 0; per_measurement < 2; ++per_measurement) {
            // 0: random blocks on the tableau assembled by ONE ncclAllGather of the rows (the default); 1: an exchange per measurement
            ShardedTableau st(c.n, local, &ex);
            st.replicate_random_blocks = per_measurement == 0;
            const size_t c0[3] = {ex.calls()[0], ex.calls()[1], ex.calls()[2]};
            const size_t b0 = ex.bytes();
            const auto t0 = std::chrono::steady_clock::now();
            MeasurementRecord rec = st.sim(c, 20250703);
            Device::instance().sync();
            const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
            bool same = rec.size() == ref.record.size();
            for (size_t i = 0; same && i < rec.size(); ++i) same = rec[i].outcome == ref.record[i].outcome && rec[i].deterministic == ref.record[i].deterministic;
            auto mine = st.local_rows();
            bool rows_same = !mine.empty() || world * local > int((c.n + 63) / 64);
            for (const auto& [idx, row] : mine) rows_same = rows_same && row == all[idx];
            const size_t nar = ex.calls()[0] - c0[0], nag = ex.calls()[1] - c0[1], nbc = ex.calls()[2] - c0[2];
            std::printf("rank %d/%d: d=%u rounds=%u local_shards=%d %s: record %s rows %s | ncclAllReduce(min) %zu ncclAllGather %zu ncclBroadcast %zu, %zu payload bytes, %.1f ms\n",
                        rank, world, d, rounds, local, per_measurement ? "exchange per measurement" : "replicated random blocks", same ? "ok" : "DIFFERS", rows_same ? "ok" : "DIFFER",
                        nar, nag, nbc, ex.bytes() - b0, ms);
            if (!same || !rows_same || nar == 0 || nag == 0) return 1;
            if (per_measurement ? nbc == 0 : (nbc != 0 || st.replicated_blocks == 0)) return 1;
        }
        // an NCCL failure surfaces as stabkit::Error with the SK_ENCCL text
        bool threw = false;
        try { std::vector<uint64_t> dummy; ex.broadcast(nullptr, nullptr, 8, world + 7); } catch (const Error& e) { threw = std::strstr(e.what(), "ncclBroadcast") != nullptr; }
        if (!threw) { std::printf("rank %d: invalid root did not raise\n", rank); return 1; }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "rank %d: %s\n", rank, e.what());
        return 1;
    }
    std::printf("rank %d ok\n", rank);
    return 0;
}
