// stabkit/sharded.hpp -- one CHP tableau row-sharded over several shards / GPUs.
// Shard g owns the slots [lo_g, hi_g) = stabilizer i AND destabilizer i (whole 64-row words).  Clifford gates never
// communicate; a measurement is assembled from the sk_shard_* kernels and three exchanges:
// allreduce-MIN of the pivot candidates, broadcast of the pivot row, allgather of the partial products.  Results are
// bit-identical to stabkit::sim.  `ShardExchange` is the communication seam: the default implementation serves several
// shards held by ONE process (device-to-device copies); a multi-process job overrides the three calls with its
// communication library (NCCL: ncclAllReduce(ncclMin) / ncclAllGather / ncclBroadcast on the context's stream -- see
// INTEGRATION.md section 4a; the Python driver paper_2507_03092_b200/sharded.py does exactly that over torch.distributed).
#pragma once
#include <algorithm>
#include <vector>

#include "stabkit/engine.hpp"

namespace stabkit {

struct ShardExchange {
    virtual ~ShardExchange() = default;
    virtual int rank() const { return 0; }
    virtual int world() const { return 1; }
    // element-wise MIN over all ranks of `cand` (host array; pivot candidates are a few bytes per measurement)
    virtual void allreduce_min(std::vector<int32_t>& /*cand*/) {}
    // d_out[world * local][words] <- every rank's d_in[local][words]; the default (world == 1) is one device copy
    virtual void allgather(sk_ctx* ctx, const uint64_t* d_in, uint64_t* d_out, size_t words_per_rank) {
        Device::instance().check(sk_dev_copy(ctx, d_out, d_in, words_per_rank * 8, 2));
    }
    // pivot row from the rank that owns it to everybody (device buffer, in place)
    virtual void broadcast(sk_ctx* /*ctx*/, uint64_t* /*d_row*/, size_t /*words*/, int /*root_rank*/) {}
};

class ShardedTableau {
  public:
    static constexpr int32_t kNone = 0x7f7f7f7f;

    // `local` shards on this process's device; global shard index = rank * local + l
    ShardedTableau(size_t n, int local, ShardExchange* ex = nullptr) : n_(n), local_(local), ex_(ex ? ex : &self_) {
        Device& d = Device::instance();
        const int G = ex_->world() * local_;
        for (int g = 0; g < G; ++g) ranges_.push_back(slot_range(n, g, G));
        for (int l = 0; l < local_; ++l) {
            sk_shard* s = nullptr;
            const auto [lo, hi] = ranges_[size_t(ex_->rank() * local_ + l)];
            d.check(sk_shard_create(d.ctx(), n, lo, hi, &s));
            shards_.push_back(s);
        }
        pw_ = size_t(sk_shard_partial_words(shards_[0]));
        d.check(sk_dev_alloc(d.ctx(), pw_ * 8, reinterpret_cast<void**>(&d_row_)));
    }
    // Random measurement blocks on the tableau assembled from all shards (one allgather of the rows per block; the elimination is
    // replicated on every rank) -- the default; false = an exchange per measurement throughout (tableaux beyond one GPU's memory).
    bool replicate_random_blocks = true;
    size_t replicated_blocks = 0;

    ~ShardedTableau() {
        Device& d = Device::instance();
        if (full_) sk_tableau_destroy(full_);
        sk_dev_free(d.ctx(), d_blk_); sk_dev_free(d.ctx(), d_blks_);
        for (sk_shard* s : shards_) sk_shard_destroy(s);
        sk_dev_free(d.ctx(), d_row_); sk_dev_free(d.ctx(), d_cand_); sk_dev_free(d.ctx(), d_part_); sk_dev_free(d.ctx(), d_all_);
    }
    ShardedTableau(const ShardedTableau&) = delete;
    ShardedTableau& operator=(const ShardedTableau&) = delete;

    // contiguous slots of global shard g out of G, whole 64-row words (same rule as paper_2507_03092_b200/dist.py)
    static std::pair<uint64_t, uint64_t> slot_range(uint64_t n, int g, int G) {
        const uint64_t words = (n + 63) / 64, per = (words + uint64_t(G) - 1) / uint64_t(G);
        const uint64_t lo = std::min(words, uint64_t(g) * per) * 64, hi = std::min(words, (uint64_t(g) + 1) * per) * 64;
        return {std::min(lo, n), std::min(hi, n)};
    }

    void apply_gates(const std::vector<Gate>& gates) {
        Device& d = Device::instance();
        for (sk_shard* s : shards_) d.check(sk_shard_apply_gates(s, reinterpret_cast<const sk_gate*>(gates.data()), gates.size()));
    }

    // m consecutive Z measurements with ordinals ordinal0.. ; bit-identical to sequential measure_z
    std::vector<MeasResult> measure_batch(const std::vector<uint32_t>& qubits, uint64_t seed, uint64_t ordinal0) {
        Device& d = Device::instance();
        sk_ctx* ctx = d.ctx();
        const size_t m = qubits.size();
        std::vector<MeasResult> out(m);
        const int G = ex_->world() * local_, first = ex_->rank() * local_;
        size_t pos = 0;
        while (pos < m) {
            const size_t w = std::min(win_, m - pos);
            reserve(w, size_t(G));
            // pivot candidates: MIN over the local shards on the host, then over the ranks
            std::vector<int32_t> cand(w, kNone), tmp(w);
            for (sk_shard* s : shards_) {
                d.check(sk_shard_pivot_search(s, qubits.data() + pos, w, d_cand_));
                d.check(sk_dev_copy(ctx, tmp.data(), d_cand_, w * 4, 1));
                for (size_t j = 0; j < w; ++j) cand[j] = std::min(cand[j], tmp[j]);
            }
            ex_->allreduce_min(cand);
            size_t r0 = 0;
            while (r0 < w && cand[r0] == kNone) ++r0;
            if (r0 > 0) {                                        // deterministic prefix: one allgather
                for (int l = 0; l < local_; ++l) d.check(sk_shard_det_partial(shards_[size_t(l)], qubits.data() + pos, r0, d_part_ + size_t(l) * r0 * pw_));
                ex_->allgather(ctx, d_part_, d_all_, size_t(local_) * r0 * pw_);
                std::vector<uint8_t> o(r0);
                d.check(sk_shard_det_combine(shards_[0], d_all_, uint32_t(G), r0, o.data()));
                for (size_t j = 0; j < r0; ++j) out[pos + j] = {o[j] != 0, true};
            }
            if (r0 < w && replicate_random_blocks) {            // the rest of the block on the assembled tableau
                const size_t rest = m - (pos + r0);
                std::vector<uint8_t> o(rest + 1), dt(rest + 1);
                replicated_block(qubits.data() + pos + r0, rest, seed, ordinal0 + pos + r0, o.data(), dt.data());
                for (size_t j = 0; j < rest; ++j) out[pos + r0 + j] = {o[j] != 0, dt[j] != 0};
                win_ = 64;
                return out;
            }
            if (r0 < w) {                                        // the first random measurement of the window
                const uint64_t p = uint64_t(cand[r0]);
                int owner = 0;
                while (!(ranges_[size_t(owner)].first <= p && p < ranges_[size_t(owner)].second)) ++owner;
                const int l = owner - first;
                if (l >= 0 && l < local_) d.check(sk_shard_pivot_row(shards_[size_t(l)], p, d_row_));
                ex_->broadcast(ctx, d_row_, pw_, owner / local_);
                const bool bit = CounterRng{seed}.bit(ordinal0 + pos + r0);
                for (sk_shard* s : shards_) d.check(sk_shard_random_update(s, qubits[pos + r0], p, d_row_, bit ? 1 : 0));
                out[pos + r0] = {bit, false};
                pos += r0 + 1;
                win_ = std::max<size_t>(8, std::min(win_, 2 * (r0 + 1)));    // candidates behind a random one are stale
            } else {
                pos += w;
                win_ = std::min<size_t>(8192, win_ * 4);
            }
        }
        return out;
    }

    // SPEC:310-318 on the sharded tableau
    MeasurementRecord sim(const Circuit& c, uint64_t seed) {
        MeasurementRecord rec;
        std::vector<Gate> run; std::vector<uint32_t> mq; std::vector<size_t> mi;
        uint64_t ordinal = 0;
        auto flush_gates = [&] { if (!run.empty()) { apply_gates(run); run.clear(); } };
        auto flush_meas = [&] {
            if (mq.empty()) return;
            const auto r = measure_batch(mq, seed, ordinal);
            for (size_t j = 0; j < mq.size(); ++j) rec.push_back({mi[j], mq[j], r[j].outcome, r[j].deterministic});
            ordinal += mq.size(); mq.clear(); mi.clear();
        };
        for (size_t i = 0; i < c.gates.size(); ++i) {
            const Gate& g = c.gates[i];
            if (g.kind == GateKind::M) { flush_gates(); mq.push_back(g.q0); mi.push_back(i); }
            else { flush_meas(); run.push_back(g); }
        }
        flush_gates(); flush_meas();
        return rec;
    }

    // rows held by this process, SPEC:110 order restricted to its slots: (global row index, row)
    std::vector<std::pair<size_t, PauliString>> local_rows() {
        Device& d = Device::instance();
        std::vector<std::pair<size_t, PauliString>> out;
        const size_t W = words_for_bits(n_);
        for (int l = 0; l < local_; ++l) {
            const auto [lo, hi] = ranges_[size_t(ex_->rank() * local_ + l)];
            const size_t k = size_t(hi - lo);
            std::vector<uint64_t> x(2 * k * W + 1), z(2 * k * W + 1); std::vector<uint8_t> s(2 * k + 1);
            d.check(sk_shard_download(shards_[size_t(l)], x.data(), z.data(), s.data()));
            auto rows = unpack_rows(n_, 2 * k, x.data(), z.data(), s.data());
            for (size_t i = 0; i < k; ++i) out.emplace_back(size_t(lo) + i, rows[i]);
            for (size_t i = 0; i < k; ++i) out.emplace_back(n_ + size_t(lo) + i, rows[k + i]);
        }
        return out;
    }

  private:
    // every shard's rows as one block -> allgather -> full sk_tableau -> sk_measure_batch (identical on every rank) -> rows back
    void replicated_block(const uint32_t* qubits, size_t m, uint64_t seed, uint64_t ordinal0, uint8_t* outcomes, uint8_t* dets) {
        Device& d = Device::instance();
        sk_ctx* ctx = d.ctx();
        const size_t G = ranges_.size();
        const size_t Wp = (words_for_bits(n_) + 1) & ~size_t(1);
        if (!blk_words_) {
            for (const auto& [lo, hi] : ranges_) { const size_t k = size_t(hi - lo); blk_words_ = std::max(blk_words_, 4 * k * Wp + 2 * ((k + 63) / 64)); }
            blk_words_ = std::max<size_t>(blk_words_, 2);
            d.check(sk_dev_alloc(ctx, size_t(local_) * blk_words_ * 8, reinterpret_cast<void**>(&d_blk_)));
            d.check(sk_dev_alloc(ctx, G * blk_words_ * 8, reinterpret_cast<void**>(&d_blks_)));
            d.check(sk_tableau_create(ctx, n_, &full_));
        }
        for (int l = 0; l < local_; ++l) d.check(sk_shard_export_rows(shards_[size_t(l)], d_blk_ + size_t(l) * blk_words_));
        ex_->allgather(ctx, d_blk_, d_blks_, size_t(local_) * blk_words_);
        for (size_t g = 0; g < G; ++g) d.check(sk_tableau_import_block(full_, ranges_[g].first, ranges_[g].second, d_blks_ + g * blk_words_));
        d.check(sk_tableau_commit_blocks(full_));
        d.check(sk_measure_batch(full_, qubits, m, seed, ordinal0, outcomes, dets));
        for (int l = 0; l < local_; ++l) {
            const auto [lo, hi] = ranges_[size_t(ex_->rank() * local_ + l)];
            d.check(sk_tableau_export_block(full_, lo, hi, d_blk_ + size_t(l) * blk_words_));
            d.check(sk_shard_import_rows(shards_[size_t(l)], d_blk_ + size_t(l) * blk_words_));
        }
        ++replicated_blocks;
    }
    void reserve(size_t w, size_t G) {
        if (w <= cap_) return;
        Device& d = Device::instance();
        sk_dev_free(d.ctx(), d_cand_); sk_dev_free(d.ctx(), d_part_); sk_dev_free(d.ctx(), d_all_);
        d_cand_ = nullptr; d_part_ = nullptr; d_all_ = nullptr;
        cap_ = std::max<size_t>(2 * w, 256);
        d.check(sk_dev_alloc(d.ctx(), cap_ * 4, reinterpret_cast<void**>(&d_cand_)));
        d.check(sk_dev_alloc(d.ctx(), size_t(local_) * cap_ * pw_ * 8, reinterpret_cast<void**>(&d_part_)));
        d.check(sk_dev_alloc(d.ctx(), G * cap_ * pw_ * 8, reinterpret_cast<void**>(&d_all_)));
    }
    size_t n_; int local_; ShardExchange self_; ShardExchange* ex_;
    std::vector<std::pair<uint64_t, uint64_t>> ranges_;
    std::vector<sk_shard*> shards_;
    size_t pw_ = 0, cap_ = 0, win_ = 64;
    sk_tableau* full_ = nullptr; uint64_t* d_blk_ = nullptr; uint64_t* d_blks_ = nullptr; size_t blk_words_ = 0;
    int32_t* d_cand_ = nullptr; uint64_t* d_part_ = nullptr; uint64_t* d_all_ = nullptr; uint64_t* d_row_ = nullptr;
};

}  // namespace stabkit
