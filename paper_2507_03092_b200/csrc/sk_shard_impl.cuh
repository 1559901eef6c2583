// sk_shard_impl.cuh -- C ABI of a row shard (include/stabkit_b200.h, "row sharding"); included at the end of sk_api.cu.
// Host orchestration only: kernels in kernels_shard.cuh, gate layers and transposes are the single-GPU kernels.
#pragma once
#include "kernels_shard.cuh"

struct sk_shard {
    sk_ctx* ctx = nullptr;
    uint64_t n = 0, lo = 0, hi = 0;
    int nloc = 0, W = 0, Wp = 0, RW = 0, NS = 0, PW = 0;
    DMat m;
    bool r_valid = false;
    size_t cols_bytes = 0, rows_bytes = 0, sgn_bytes = 0;
    u64* d_mask = nullptr; u64* d_cnt = nullptr;          // d_cnt: [0] rowsums in the random branch, [1] in the deterministic branch
    u32* d_q = nullptr; size_t q_cap = 0; uint8_t* d_out = nullptr;
    std::vector<uint32_t> scratch;
    // Clifford runs already layered and resident on the device, keyed by a hash of the gate bytes: the rounds of a memory experiment
    // repeat the same run, so validation, layering, the upload and its synchronisation are paid once
    struct Run { uint64_t hash = 0; size_t ngates = 0; sk_gate* d_gates = nullptr; std::vector<uint32_t> sizes; uint64_t used = 0; };
    std::vector<Run> runs; uint64_t run_clock = 0;
};
static uint64_t gate_bytes_hash(const sk_gate* g, size_t n) {
    const unsigned char* p = reinterpret_cast<const unsigned char*>(g);
    const size_t bytes = n * sizeof(sk_gate), words = bytes / 8;
    uint64_t h = 0x9e3779b97f4a7c15ull ^ bytes;
    for (size_t i = 0; i < words; ++i) { uint64_t w; memcpy(&w, p + 8 * i, 8); h = (h ^ w) * 0xff51afd7ed558ccdull; h ^= h >> 32; }
    for (size_t i = words * 8; i < bytes; ++i) h = (h ^ p[i]) * 0x100000001b3ull;
    return h;
}

static int32_t shard_identity(sk_shard* s) {
    sk_ctx* c = s->ctx;
    SK_CUDA(c, cudaMemsetAsync(s->m.cols, 0, s->cols_bytes, c->stream));
    SK_CUDA(c, cudaMemsetAsync(s->m.rows, 0, s->rows_bytes, c->stream));
    SK_CUDA(c, cudaMemsetAsync(s->m.sgn, 0, s->sgn_bytes, c->stream));
    SK_CUDA(c, cudaMemsetAsync(s->d_cnt, 0, 16, c->stream));
    if (s->nloc) {
        k_shard_identity<<<(s->nloc + 255) / 256, 256, 0, c->stream>>>(s->m.cols, s->m.rows, int(s->lo), s->nloc, s->RW, s->Wp, s->NS);
        c->cnt.kernel_launches++;
    }
    SK_CUDA(c, cudaGetLastError());
    s->r_valid = true;
    return SK_OK;
}

extern "C" void sk_shard_destroy(sk_shard* s) {
    if (!s) return;
    sk_ctx* c = s->ctx;
    cudaSetDevice(c->device);
    for (void* p : {(void*)s->m.cols, (void*)s->m.rows, (void*)s->m.sgn, (void*)s->d_mask, (void*)s->d_cnt, (void*)s->d_q, (void*)s->d_out}) dfree(c, p);
    for (auto& r : s->runs) dfree(c, r.d_gates);
    delete s;
}

extern "C" int32_t sk_shard_create(sk_ctx* c, uint64_t n, uint64_t slot_lo, uint64_t slot_hi, sk_shard** out) {
    if (!c || !out) return SK_EARG;
    *out = nullptr;
    if (n == 0) SK_FAIL(c, SK_EDIM, "new_identity: n must be >= 1 (SPEC:129)");
    if (n > (1u << 20)) SK_FAIL(c, SK_EDIM, "n=%llu exceeds the supported 2^20 qubits", (unsigned long long)n);
    if (slot_lo > slot_hi || slot_hi > n) SK_FAIL(c, SK_EDIM, "shard slots [%llu, %llu) outside [0, %llu)", (unsigned long long)slot_lo, (unsigned long long)slot_hi, (unsigned long long)n);
    SK_CUDA(c, cudaSetDevice(c->device));
    sk_shard* s = new sk_shard();
    s->ctx = c; s->n = n; s->lo = slot_lo; s->hi = slot_hi; s->nloc = int(slot_hi - slot_lo);
    s->W = int((n + 63) / 64); s->Wp = (s->W + 1) & ~1;
    s->NS = std::max(64, (s->nloc + 63) & ~63); s->RW = 2 * s->NS / 64; s->PW = 2 * s->Wp + 2;
    s->m.n = n; s->m.W = s->W; s->m.Wp = s->Wp; s->m.RW = s->RW;
    s->cols_bytes = (size_t)n * 2 * s->RW * 8;
    s->rows_bytes = (size_t)64 * s->RW * 2 * s->Wp * 8;
    s->sgn_bytes = (size_t)s->RW * 8;
    cudaError_t e1 = dmalloc(c, &s->m.cols, s->cols_bytes), e2 = dmalloc(c, &s->m.rows, s->rows_bytes), e3 = dmalloc(c, &s->m.sgn, s->sgn_bytes);
    cudaError_t e4 = dmalloc(c, &s->d_mask, (size_t)s->RW * 8), e5 = dmalloc(c, &s->d_cnt, 16);
    if (e1 || e2 || e3 || e4 || e5) { sk_shard_destroy(s); SK_FAIL(c, SK_ECUDA, "cudaMalloc failed for a shard of %d slots x %llu qubits", int(slot_hi - slot_lo), (unsigned long long)n); }
    int32_t rc = shard_identity(s);
    if (rc) { sk_shard_destroy(s); return rc; }
    *out = s;
    return SK_OK;
}
extern "C" int32_t sk_shard_reset(sk_shard* s) { return s ? shard_identity(s) : SK_EARG; }
extern "C" uint64_t sk_shard_partial_words(const sk_shard* s) { return s ? uint64_t(s->PW) : 0; }

// Clifford gates: the ordinary fused-layer kernel on this shard's columns; no communication.
extern "C" int32_t sk_shard_apply_gates(sk_shard* s, const sk_gate* gates, size_t ngates) {
    if (!s || (!gates && ngates)) return SK_EARG;
    sk_ctx* c = s->ctx;
    if (ngates == 0) return SK_OK;
    const uint64_t hsh = gate_bytes_hash(gates, ngates);
    sk_shard::Run* run = nullptr;
    for (auto& r : s->runs) if (r.hash == hsh && r.ngates == ngates) { run = &r; break; }
    if (!run) {
        for (size_t i = 0; i < ngates; ++i) {
            int32_t rc = validate_gate(c, gates[i], s->n, i);
            if (rc) return rc;
            if (gates[i].kind >= SK_M) SK_FAIL(c, SK_EUNSUPPORTED, "gate %zu: M/T/TDG in a Clifford sequence (SPEC:191)", i);
        }
        std::vector<sk_gate> ordered; std::vector<uint32_t> sizes;
        sk_layer_run(gates, ngates, s->n, s->scratch, ordered, sizes);
        if (s->runs.size() >= 8) {             // evict the least recently used run
            size_t victim = 0;
            for (size_t i = 1; i < s->runs.size(); ++i) if (s->runs[i].used < s->runs[victim].used) victim = i;
            dfree(c, s->runs[victim].d_gates);
            s->runs.erase(s->runs.begin() + victim);
        }
        sk_shard::Run nr; nr.hash = hsh; nr.ngates = ngates; nr.sizes = sizes;
        SK_CUDA(c, dmalloc(c, &nr.d_gates, ngates * sizeof(sk_gate)));
        SK_CUDA(c, cudaMemcpyAsync(nr.d_gates, ordered.data(), ngates * sizeof(sk_gate), cudaMemcpyHostToDevice, c->stream));
        SK_CUDA(c, cudaStreamSynchronize(c->stream));     // `ordered` dies at the end of this block
        s->runs.push_back(std::move(nr));
        run = &s->runs.back();
    }
    run->used = ++s->run_clock;
    const int threads = std::min(256, std::max(32, (s->RW / 2 + 31) & ~31));
    const int target_ctas = layer_target_ctas(c, threads);
    size_t off = 0;
    for (uint32_t sz : run->sizes) {
        const int ng = int(sz), gpb = std::max(1, (ng + target_ctas - 1) / target_ctas);
        k_layer<<<(ng + gpb - 1) / gpb, threads, 0, c->stream>>>(s->m.cols, s->m.sgn, (const sk_gate*)run->d_gates + off, ng, s->RW, gpb, nullptr);
        c->cnt.kernel_launches++; c->cnt.layers++;
        off += sz;
    }
    s->r_valid = false;
    SK_CUDA(c, cudaGetLastError());
    return SK_OK;
}

static int32_t shard_rows(sk_shard* s) {               // C -> R, both halves
    if (s->r_valid) return SK_OK;
    sk_ctx* c = s->ctx;
    int32_t rc = launch_transpose(c, reinterpret_cast<const u32*>(s->m.cols), (size_t)4 * s->RW, int(s->n), 2 * s->RW,
                                  reinterpret_cast<u32*>(s->m.rows), (size_t)4 * s->Wp, 64 * s->RW, 2 * s->Wp,
                                  (size_t)2 * s->RW, (size_t)2 * s->Wp, nullptr);
    if (rc) return rc;
    c->cnt.transposes++;
    s->r_valid = true;
    return SK_OK;
}
static int32_t shard_qubits(sk_shard* s, const uint32_t* qubits, size_t m) {
    sk_ctx* c = s->ctx;
    for (size_t i = 0; i < m; ++i)
        if (qubits[i] >= s->n) SK_FAIL(c, SK_EDIM, "measure: qubit %u out of range for %llu qubits", qubits[i], (unsigned long long)s->n);
    if (m > s->q_cap) {
        dfree(c, s->d_q); dfree(c, s->d_out); s->d_q = nullptr; s->d_out = nullptr; s->q_cap = 0;
        const size_t cap = std::max<size_t>(2 * m, 1024);
        SK_CUDA(c, dmalloc(c, &s->d_q, cap * 4));
        SK_CUDA(c, dmalloc(c, &s->d_out, cap));
        s->q_cap = cap;
    }
    SK_CUDA(c, cudaMemcpyAsync(s->d_q, qubits, m * 4, cudaMemcpyHostToDevice, c->stream));
    return SK_OK;
}

extern "C" int32_t sk_shard_pivot_search(sk_shard* s, const uint32_t* qubits, size_t m, int32_t* d_cand) {
    if (!s || (!qubits && m) || !d_cand) return SK_EARG;
    sk_ctx* c = s->ctx;
    if (m == 0) return SK_OK;
    int32_t rc = shard_qubits(s, qubits, m);
    if (rc) return rc;
    k_shard_pivot<<<(unsigned)((m * 32 + 255) / 256), 256, 0, c->stream>>>(s->m.cols, s->d_q, int(m), s->RW, s->NS / 64, int(s->lo), d_cand);
    c->cnt.kernel_launches++;
    SK_CUDA(c, cudaGetLastError());
    return SK_OK;
}

extern "C" int32_t sk_shard_det_partial(sk_shard* s, const uint32_t* qubits, size_t m, uint64_t* d_part) {
    if (!s || (!qubits && m) || !d_part) return SK_EARG;
    sk_ctx* c = s->ctx;
    if (m == 0) return SK_OK;
    int32_t rc = shard_qubits(s, qubits, m);
    if (rc) return rc;
    if ((rc = shard_rows(s))) return rc;
    k_shard_det_partial<<<(unsigned)((m * 32 + 255) / 256), 256, 0, c->stream>>>(s->m, s->d_q, int(m), s->NS, (u64*)d_part, s->PW, s->d_cnt + 1);
    c->cnt.kernel_launches++;
    SK_CUDA(c, cudaGetLastError());
    return SK_OK;
}

extern "C" int32_t sk_shard_det_combine(sk_shard* s, const uint64_t* d_gathered, uint32_t nshards, size_t m, uint8_t* outcomes) {
    if (!s || !d_gathered || !outcomes || nshards == 0) return SK_EARG;
    sk_ctx* c = s->ctx;
    if (m == 0) return SK_OK;
    if (m > s->q_cap) SK_FAIL(c, SK_EARG, "det_combine: %zu measurements, but the preceding det_partial had at most %zu", m, s->q_cap);
    k_shard_det_combine<<<(unsigned)((m * 32 + 255) / 256), 256, 0, c->stream>>>((const u64*)d_gathered, int(nshards), int(m), s->W, s->Wp, s->PW, s->d_out, c->d_err);
    c->cnt.kernel_launches++;
    SK_CUDA(c, cudaGetLastError());
    SK_CUDA(c, cudaMemcpyAsync(outcomes, s->d_out, m, cudaMemcpyDeviceToHost, c->stream));
    return check_ws(c);
}

extern "C" int32_t sk_shard_pivot_row(sk_shard* s, uint64_t p, uint64_t* d_row) {
    if (!s || !d_row) return SK_EARG;
    sk_ctx* c = s->ctx;
    if (p < s->lo || p >= s->hi) SK_FAIL(c, SK_EDIM, "pivot_row: stabilizer %llu is not in this shard's slots [%llu, %llu)", (unsigned long long)p, (unsigned long long)s->lo, (unsigned long long)s->hi);
    int32_t rc = shard_rows(s);
    if (rc) return rc;
    k_shard_get_row<<<1, 128, 0, c->stream>>>(s->m, int(p - s->lo), (u64*)d_row);
    c->cnt.kernel_launches++;
    SK_CUDA(c, cudaGetLastError());
    return SK_OK;
}

extern "C" int32_t sk_shard_random_update(sk_shard* s, uint32_t q, uint64_t p, const uint64_t* d_row, uint8_t outcome) {
    if (!s || !d_row) return SK_EARG;
    sk_ctx* c = s->ctx;
    if (q >= s->n || p >= s->n) SK_FAIL(c, SK_EDIM, "random_update: qubit %u / pivot %llu out of range", q, (unsigned long long)p);
    int32_t rc = shard_rows(s);
    if (rc) return rc;
    const int pb = (p >= s->lo && p < s->hi) ? int(p - s->lo) : -1;
    k_shard_mask<<<(s->RW + 127) / 128, 128, 0, c->stream>>>(s->m.cols, q, s->RW, s->NS, pb, s->d_mask);
    k_shard_rowsum<<<(64 * s->RW * 32 + 255) / 256, 256, 0, c->stream>>>(s->m, s->d_mask, (const u64*)d_row, c->d_err, s->d_cnt);
    k_shard_colxor<<<(unsigned)((s->n * 32 + 255) / 256), 256, 0, c->stream>>>(s->m, s->d_mask, (const u64*)d_row);
    c->cnt.kernel_launches += 3;
    if (pb >= 0) { k_shard_fix<<<1, 256, 0, c->stream>>>(s->m, s->NS, pb, q, (const u64*)d_row, int(outcome & 1)); c->cnt.kernel_launches++; }
    SK_CUDA(c, cudaGetLastError());
    return SK_OK;
}

// rows of this shard, row-major: stabilizers lo..hi-1 then destabilizers lo..hi-1
extern "C" int32_t sk_shard_download(sk_shard* s, uint64_t* x, uint64_t* z, uint8_t* sign) {
    if (!s || !x || !z || !sign) return SK_EARG;
    sk_ctx* c = s->ctx;
    if (s->nloc == 0) return check_ws(c);
    int32_t rc = shard_rows(s);
    if (rc) return rc;
    const size_t nrows = 2 * (size_t)s->nloc, words = nrows * s->W;
    rc = sk_ctx_reserve_tmp(c, words * 16 + nrows + 64);
    if (rc) return rc;
    u64* dx = (u64*)c->d_tmp; u64* dz = dx + words; uint8_t* ds = (uint8_t*)(dz + words);
    k_unpack_rows<<<(unsigned)((words + 255) / 256), 256, 0, c->stream>>>(s->m.rows, dx, dz, int(nrows), s->W, s->Wp, s->nloc, s->NS);
    k_signs_to_bytes<<<(unsigned)((nrows + 255) / 256), 256, 0, c->stream>>>(s->m.sgn, ds, int(nrows), s->nloc, s->NS);
    c->cnt.kernel_launches += 2;
    SK_CUDA(c, cudaGetLastError());
    SK_CUDA(c, cudaMemcpyAsync(x, dx, words * 8, cudaMemcpyDeviceToHost, c->stream));
    SK_CUDA(c, cudaMemcpyAsync(z, dz, words * 8, cudaMemcpyDeviceToHost, c->stream));
    SK_CUDA(c, cudaMemcpyAsync(sign, ds, nrows, cudaMemcpyDeviceToHost, c->stream));
    return check_ws(c);
}

// ---- replicated elimination of a random measurement block ------------------------------------------
// A shard's rows travel as one contiguous block: stabilizer rows (nloc x 2*Wp words), destabilizer rows (same), then the sign words of
// the two halves (ceil(nloc/64) each; slot ranges are whole 64-row words, so they are word aligned in the full tableau as well).
// Every rank gathers all blocks into a full sk_tableau, runs the single-GPU measurement kernel on it -- the result is the same on
// every rank -- and takes its own rows back.  Communication: one allgather of the tableau per random block instead of an exchange per
// measurement; the elimination itself is replicated, not sharded (tableaux beyond one GPU's memory keep the per-measurement protocol).
static size_t shard_block_words(int nloc, int Wp) { return (size_t)2 * nloc * 2 * Wp + 2 * (size_t)((nloc + 63) / 64); }
extern "C" uint64_t sk_shard_export_words(const sk_shard* s) { return s ? uint64_t(shard_block_words(s->nloc, s->Wp)) : 0; }
extern "C" int32_t sk_shard_export_rows(sk_shard* s, uint64_t* d_buf) {
    if (!s || !d_buf) return SK_EARG;
    sk_ctx* c = s->ctx;
    if (s->nloc == 0) return SK_OK;
    int32_t rc = shard_rows(s);
    if (rc) return rc;
    const size_t half = (size_t)s->nloc * 2 * s->Wp, sw = (size_t)(s->nloc + 63) / 64;
    SK_CUDA(c, cudaMemcpyAsync(d_buf, s->m.rows, half * 8, cudaMemcpyDeviceToDevice, c->stream));
    SK_CUDA(c, cudaMemcpyAsync(d_buf + half, s->m.rows + (size_t)s->NS * 2 * s->Wp, half * 8, cudaMemcpyDeviceToDevice, c->stream));
    SK_CUDA(c, cudaMemcpyAsync(d_buf + 2 * half, s->m.sgn, sw * 8, cudaMemcpyDeviceToDevice, c->stream));
    SK_CUDA(c, cudaMemcpyAsync(d_buf + 2 * half + sw, s->m.sgn + s->NS / 64, sw * 8, cudaMemcpyDeviceToDevice, c->stream));
    return SK_OK;
}
extern "C" int32_t sk_shard_import_rows(sk_shard* s, const uint64_t* d_buf) {
    if (!s || !d_buf) return SK_EARG;
    sk_ctx* c = s->ctx;
    if (s->nloc == 0) return SK_OK;
    const size_t half = (size_t)s->nloc * 2 * s->Wp, sw = (size_t)(s->nloc + 63) / 64;
    SK_CUDA(c, cudaMemcpyAsync(s->m.rows, d_buf, half * 8, cudaMemcpyDeviceToDevice, c->stream));
    SK_CUDA(c, cudaMemcpyAsync(s->m.rows + (size_t)s->NS * 2 * s->Wp, d_buf + half, half * 8, cudaMemcpyDeviceToDevice, c->stream));
    SK_CUDA(c, cudaMemcpyAsync(s->m.sgn, d_buf + 2 * half, sw * 8, cudaMemcpyDeviceToDevice, c->stream));
    SK_CUDA(c, cudaMemcpyAsync(s->m.sgn + s->NS / 64, d_buf + 2 * half + sw, sw * 8, cudaMemcpyDeviceToDevice, c->stream));
    s->r_valid = true;
    // the gate form follows from the rows (R -> C, both halves)
    int32_t rc = launch_transpose(c, reinterpret_cast<const u32*>(s->m.rows), (size_t)4 * s->Wp, 64 * s->RW, 2 * s->Wp,
                                  reinterpret_cast<u32*>(s->m.cols), (size_t)4 * s->RW, int(s->n), 2 * s->RW,
                                  (size_t)2 * s->Wp, (size_t)2 * s->RW, nullptr);
    if (rc) return rc;
    c->cnt.transposes++;
    return SK_OK;
}
// the block of the slots [lo, hi) into / out of a full tableau (same block layout); commit derives the gate form after all imports
extern "C" int32_t sk_tableau_import_block(sk_tableau* t, uint64_t lo, uint64_t hi, const uint64_t* d_buf) {
    if (!t || !d_buf) return SK_EARG;
    sk_ctx* c = t->ctx;
    if (lo == hi) return SK_OK;                         // a shard without slots
    if (lo > hi || hi > t->n || (lo & 63)) SK_FAIL(c, SK_EDIM, "import_block: slots [%llu, %llu) of %llu qubits (lo must be a multiple of 64)", (unsigned long long)lo, (unsigned long long)hi, (unsigned long long)t->n);
    const int nloc = int(hi - lo);
    if (nloc == 0) return SK_OK;
    const size_t half = (size_t)nloc * 2 * t->Wp, sw = (size_t)(nloc + 63) / 64;
    SK_CUDA(c, cudaMemcpyAsync(t->m.rows + (size_t)lo * 2 * t->Wp, d_buf, half * 8, cudaMemcpyDeviceToDevice, c->stream));
    SK_CUDA(c, cudaMemcpyAsync(t->m.rows + ((size_t)t->NS + lo) * 2 * t->Wp, d_buf + half, half * 8, cudaMemcpyDeviceToDevice, c->stream));
    SK_CUDA(c, cudaMemcpyAsync(t->m.sgn + lo / 64, d_buf + 2 * half, sw * 8, cudaMemcpyDeviceToDevice, c->stream));
    SK_CUDA(c, cudaMemcpyAsync(t->m.sgn + ((size_t)t->NS + lo) / 64, d_buf + 2 * half + sw, sw * 8, cudaMemcpyDeviceToDevice, c->stream));
    return SK_OK;
}
extern "C" int32_t sk_tableau_commit_blocks(sk_tableau* t) {
    if (!t) return SK_EARG;
    t->r_valid = true; t->r_destab_stale = false;
    return cols_from_rows(t);
}
extern "C" int32_t sk_tableau_export_block(sk_tableau* t, uint64_t lo, uint64_t hi, uint64_t* d_buf) {
    if (!t || !d_buf) return SK_EARG;
    sk_ctx* c = t->ctx;
    if (lo == hi) return SK_OK;
    if (lo > hi || hi > t->n || (lo & 63)) SK_FAIL(c, SK_EDIM, "export_block: slots [%llu, %llu) of %llu qubits (lo must be a multiple of 64)", (unsigned long long)lo, (unsigned long long)hi, (unsigned long long)t->n);
    const int nloc = int(hi - lo);
    if (nloc == 0) return SK_OK;
    { int32_t rc = rows_full(t); if (rc) return rc; }
    const size_t half = (size_t)nloc * 2 * t->Wp, sw = (size_t)(nloc + 63) / 64;
    SK_CUDA(c, cudaMemcpyAsync(d_buf, t->m.rows + (size_t)lo * 2 * t->Wp, half * 8, cudaMemcpyDeviceToDevice, c->stream));
    SK_CUDA(c, cudaMemcpyAsync(d_buf + half, t->m.rows + ((size_t)t->NS + lo) * 2 * t->Wp, half * 8, cudaMemcpyDeviceToDevice, c->stream));
    SK_CUDA(c, cudaMemcpyAsync(d_buf + 2 * half, t->m.sgn + lo / 64, sw * 8, cudaMemcpyDeviceToDevice, c->stream));
    SK_CUDA(c, cudaMemcpyAsync(d_buf + 2 * half + sw, t->m.sgn + ((size_t)t->NS + lo) / 64, sw * 8, cudaMemcpyDeviceToDevice, c->stream));
    return SK_OK;
}

// rowsums performed by this shard: out2[0] random branch, out2[1] deterministic branch.  Synchronises.
extern "C" int32_t sk_shard_counters(sk_shard* s, uint64_t out2[2]) {
    if (!s || !out2) return SK_EARG;
    sk_ctx* c = s->ctx;
    SK_CUDA(c, cudaMemcpyAsync(out2, s->d_cnt, 16, cudaMemcpyDeviceToHost, c->stream));
    return check_ws(c);
}

// ---- plain device buffers for the exchange (so that a host binding needs no CUDA headers of its own) ----------------
extern "C" int32_t sk_dev_alloc(sk_ctx* c, size_t bytes, void** out) {
    if (!c || !out) return SK_EARG;
    *out = nullptr;
    SK_CUDA(c, cudaSetDevice(c->device));
    SK_CUDA(c, cudaMalloc(out, bytes ? bytes : 16));
    return SK_OK;
}
extern "C" void sk_dev_free(sk_ctx* c, void* p) { if (c && p) { cudaSetDevice(c->device); cudaStreamSynchronize(c->stream); cudaFree(p); } }
// kind: 0 host->device, 1 device->host (synchronises), 2 device->device; ordered on the context's stream
extern "C" int32_t sk_dev_copy(sk_ctx* c, void* dst, const void* src, size_t bytes, int kind) {
    if (!c || (!dst && bytes) || (!src && bytes) || kind < 0 || kind > 2) return SK_EARG;
    if (bytes == 0) return SK_OK;
    const cudaMemcpyKind k = kind == 0 ? cudaMemcpyHostToDevice : kind == 1 ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    SK_CUDA(c, cudaMemcpyAsync(dst, src, bytes, k, c->stream));
    if (kind != 2) SK_CUDA(c, cudaStreamSynchronize(c->stream));
    return SK_OK;
}
