// sk_rows_impl.cuh -- C ABI part 2 (included by sk_api.cu): device Pauli row sets, grouping
// and the Clifford+T -> PBC pass (Algorithms 2-4).
// Host orchestration only; kernels are in kernels_rows.cuh / kernels_layer.cuh / kernels_transpose.cuh.
#pragma once
#include <climits>
#include <memory>
#include <numeric>

#include "kernels_rows.cuh"

// ---- generic C/R store helpers (any row-bit count; no stabilizer/destabilizer split) -----------
static int32_t dm_transpose_c2r(sk_ctx* c, const DMat& m) {
    const u32* src = reinterpret_cast<const u32*>(m.cols);
    u32* dst = reinterpret_cast<u32*>(m.rows);
    int32_t rc = launch_transpose(c, src, (size_t)4 * m.RW, int(m.n), 2 * m.RW, dst, (size_t)4 * m.Wp, 64 * m.RW, 2 * m.Wp,
                                  (size_t)2 * m.RW, (size_t)2 * m.Wp, nullptr);
    if (rc) return rc;
    c->cnt.transposes++;
    return SK_OK;
}
static int32_t dm_transpose_r2c(sk_ctx* c, const DMat& m) {
    const u32* src = reinterpret_cast<const u32*>(m.rows);
    u32* dst = reinterpret_cast<u32*>(m.cols);
    int32_t rc = launch_transpose(c, src, (size_t)4 * m.Wp, 64 * m.RW, 2 * m.Wp, dst, (size_t)4 * m.RW, int(m.n), 2 * m.RW,
                                  (size_t)2 * m.Wp, (size_t)2 * m.RW, nullptr);
    if (rc) return rc;
    c->cnt.transposes++;
    return SK_OK;
}
static void dm_launch_layer(sk_ctx* c, const DMat& m, const sk_gate* d_gates, int ngates) {
    const int RW2 = m.RW / 2;
    int threads = std::min(256, std::max(32, (RW2 + 31) & ~31));
    int target_ctas = c->num_sms * std::max(1, 1536 / threads);
    int gpb = std::max(1, (ngates + target_ctas - 1) / target_ctas);
    int grid = (ngates + gpb - 1) / gpb;
    k_layer<<<grid, threads, 0, c->stream>>>(m.cols, m.sgn, d_gates, ngates, m.RW, gpb, nullptr);
    c->cnt.kernel_launches++; c->cnt.layers++;
}
template <class... A> static void launch_push(sk_ctx* c, int W, int nrows, A... args) {
    const int wpl = (W + 31) / 32;
    dim3 grid((unsigned)((nrows * 32 + 255) / 256));
    if (wpl <= 1) k_push_through<1><<<grid, 256, 0, c->stream>>>(args...);
    else if (wpl <= 2) k_push_through<2><<<grid, 256, 0, c->stream>>>(args...);
    else if (wpl <= 4) k_push_through<4><<<grid, 256, 0, c->stream>>>(args...);
    else if (wpl <= 8) k_push_through<8><<<grid, 256, 0, c->stream>>>(args...);
    else k_push_through<16><<<grid, 256, 0, c->stream>>>(args...);
    c->cnt.kernel_launches++;
}

// first-fit over rows [0, count) of an R-form array (K5 bitmap + resolver, block by block).
// d_group: device u32[count] (output).  Returns the number of groups.
static int32_t device_first_fit(sk_ctx* c, const u64* d_rows, int Wp, int W, int count, int mode, u32* d_group, uint64_t* ngroups) {
    *ngroups = 0;
    if (count == 0) return SK_OK;
    const int B = std::min(count, 1024);
    const int GW32 = count / 32 + 2;
    u32* d_bitmap = nullptr; u32* d_ng = nullptr; u32* d_ff = nullptr;
    u32* d_cnt = nullptr; u32* d_off = nullptr; u32* d_fillc = nullptr; u64* d_gterms = nullptr; u32* d_gmin = nullptr;
    SkDevScope scope; scope.own(&d_bitmap); scope.own(&d_ng); scope.own(&d_cnt); scope.own(&d_off); scope.own(&d_fillc); scope.own(&d_gterms);
    SK_CUDA(c, cudaMalloc(&d_bitmap, (size_t)B * GW32 * 4));
    SK_CUDA(c, cudaMalloc(&d_ng, 4 + (size_t)B * 4));
    d_ff = d_ng + 1;
    SK_CUDA(c, cudaMemsetAsync(d_ng, 0, 4, c->stream));
    const int Bt = std::max(1, std::min(B, (40 * 1024) / (2 * W * 8)));     // block terms staged per CTA (<= 40 KB smem)
    const size_t smem = (size_t)Bt * 2 * W * 8;
    if (smem > 48 * 1024) SK_FAIL(c, SK_EDIM, "rows too wide for the conflict kernel (W=%d)", W);
    // group-major path (W <= 2, i.e. up to 128 qubits -- BASELINE config 4): CSR of the placed terms, thread per group
    static const bool csr_off = getenv("SK_GROUP_CSR") && atoi(getenv("SK_GROUP_CSR")) == 0;
    const bool csr = W <= 2 && !csr_off && count > B;
    static const bool legacy_resolver = getenv("SK_GROUP_RESOLVER") && atoi(getenv("SK_GROUP_RESOLVER")) == 0;   // A/B switch: the sequential-scan resolver
    if (csr) {
        cudaError_t e1 = cudaMalloc(&d_cnt, ((size_t)count + 4) * 4), e2 = cudaMalloc(&d_off, ((size_t)count + 2) * 4);
        cudaError_t e3 = cudaMalloc(&d_fillc, ((size_t)count + 2) * 4), e4 = cudaMalloc(&d_gterms, (size_t)count * 32);
        if (e1 || e2 || e3 || e4) SK_FAIL(c, SK_ECUDA, "cudaMalloc failed for the grouped term store");
        SK_CUDA(c, cudaMemsetAsync(d_cnt, 0, ((size_t)count + 4) * 4, c->stream));
        d_gmin = d_cnt + count + 3;
    }
    // free-list resolver (k_first_fit_lists): rows of <= 128 qubits, plain first fit; SK_GROUP_RESOLVER=1 selects the candidate-tracking one
    static const bool lists_off = getenv("SK_GROUP_RESOLVER") != nullptr;
    // (the resolver asks for ALL the shared memory of its SM although it uses 128 KB: no CTA of the conflict kernel that runs beside it on
    //  the side stream may become co-resident and take issue slots from the one warp that is the critical path of the whole grouping)
    const size_t kListSmem = std::max<size_t>((size_t)32 * 1024 * 4, (size_t)c->max_smem_optin - 6 * 1024);
    const bool use_lists = W <= 2 && !(mode & kOrderedFit) && !lists_off && B == 1024;
    u32* d_fl = nullptr; u32* d_fcnt = nullptr; u32* d_cb = nullptr;
    scope.own(&d_fl); scope.own(&d_cb);
    if (use_lists) {
        SK_CUDA(c, cudaMalloc(&d_fl, (size_t)B * (kFreeList + 1) * 4));
        SK_CUDA(c, cudaMalloc(&d_cb, (size_t)B * 32 * 4));                      // in-block conflict matrix, a 1024-bit row per term
        d_fcnt = d_fl + (size_t)B * kFreeList;
        static bool attr_set = false;
        if (!attr_set) { SK_CUDA(c, cudaFuncSetAttribute(k_first_fit_lists, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kListSmem))); attr_set = true; }
    }
    const int Btg = std::min(B, 128);                                           // block terms per CTA: 8 CTAs per 256 groups keep the SMs busy while groups are few (GC)
    unsigned long long* npred = reinterpret_cast<unsigned long long*>(c->d_err) + 1;
    static const bool pipe_off = getenv("SK_GROUP_PIPELINE") && atoi(getenv("SK_GROUP_PIPELINE")) == 0;      // A/B switch
    const int nblocks = (count + B - 1) / B;
    if (use_lists && csr && !pipe_off && nblocks >= 3) {
        // Two streams.  The resolver occupies ONE SM for about 0.35 ms per block; the group-major conflict kernel of the NEXT block
        // (0.15 ms on the whole machine) does not have to wait for it if it works on the groups as they were one block earlier:
        //   side:  [resolver n-2 done] -> CSR of the terms of blocks <= n-2 -> conflicts of block n with those groups -> in-block matrix of block n
        //   main:  [side done] -> k_conflict_prev: block n against the terms block n-1 placed -> free lists -> resolver n
        // Same bitmap as the one-stream order by the time the free lists are made: identical groups.
        u32* d_bm2 = nullptr; u32* d_cb2 = nullptr; u32* d_ngh = nullptr;
        scope.own(&d_bm2); scope.own(&d_cb2); scope.own(&d_ngh);
        SK_CUDA(c, cudaMalloc(&d_bm2, (size_t)B * GW32 * 4));
        SK_CUDA(c, cudaMalloc(&d_cb2, (size_t)B * 32 * 4));
        SK_CUDA(c, cudaMalloc(&d_ngh, (size_t)nblocks * 4));
        // Stream priorities: the resolver's chain runs on a stream of the HIGHEST priority, the side stream on the lowest (the
        // default, which is also what the context's stream has): when the chain has a kernel to run (k_conflict_prev,
        // k_free_lists) its CTAs go first instead of queueing behind the ~30 000 CTAs of the next block's conflict kernel
        // (in situ those two kernels take 130 + 70 us against 37 + 10 alone -- they share the memory system with the conflict
        // kernel -- and 147 + 75 without the priorities; the resolver itself, alone on its SM, is not slowed).
        cudaStream_t S = nullptr, M = nullptr;
        { int lo = 0, hi = 0; cudaDeviceGetStreamPriorityRange(&lo, &hi);
          if (cudaStreamCreateWithPriority(&S, cudaStreamNonBlocking, lo) != cudaSuccess) { cudaGetLastError(); S = nullptr; }
          if (cudaStreamCreateWithPriority(&M, cudaStreamNonBlocking, hi) != cudaSuccess) { cudaGetLastError(); M = nullptr; } }
        struct StScope { cudaStream_t* s; ~StScope() { if (*s) { cudaStreamSynchronize(*s); cudaStreamDestroy(*s); } } } stscope{&S}, mtscope{&M};
        if (!S || !M) SK_FAIL(c, SK_ECUDA, "could not create the streams of the grouping pipeline");
        cudaEvent_t e_conf[2] = {nullptr, nullptr}, e_res[2] = {nullptr, nullptr};
        struct EvScope { cudaEvent_t* a; cudaEvent_t* b; ~EvScope() { for (int k = 0; k < 2; ++k) { if (a[k]) cudaEventDestroy(a[k]); if (b[k]) cudaEventDestroy(b[k]); } } } evscope{e_conf, e_res};
        for (int k = 0; k < 2; ++k) { SK_CUDA(c, cudaEventCreateWithFlags(&e_conf[k], cudaEventDisableTiming)); SK_CUDA(c, cudaEventCreateWithFlags(&e_res[k], cudaEventDisableTiming)); }
        SK_CUDA(c, cudaEventRecord(e_res[0], c->stream)); SK_CUDA(c, cudaStreamWaitEvent(S, e_res[0], 0)); SK_CUDA(c, cudaStreamWaitEvent(M, e_res[0], 0));     // both start behind the set-up above
        for (int n = 0; n < nblocks; ++n) {
            const int t0 = n * B, b = std::min(B, count - t0), par = n & 1;
            u32* bm = par ? d_bm2 : d_bitmap; u32* cbn = par ? d_cb2 : d_cb;
            // ---- side stream
            if (n >= 2) SK_CUDA(c, cudaStreamWaitEvent(S, e_res[par], 0));          // resolver n-2: its groups are final, its bitmap buffer is free
            SK_CUDA(c, cudaMemsetAsync(bm, 0, (size_t)b * GW32 * 4, S));
            if (n >= 2) {
                const int tl = t0 - B;                                               // terms [0, tl) are in the lagging CSR
                SK_CUDA(c, cudaMemsetAsync(d_gmin, 0xff, 4, S));
                k_csr_count<<<(B + 255) / 256, 256, 0, S>>>(d_group, tl - B, tl, d_cnt, d_gmin);
                k_csr_scan<<<1, 1024, 0, S>>>(d_cnt, d_ngh + (n - 2), d_off, d_gmin);
                SK_CUDA(c, cudaMemsetAsync(d_fillc, 0, ((size_t)tl + 1) * 4, S));
                k_csr_fill<<<(tl + 255) / 256, 256, 0, S>>>(d_rows, Wp, W, d_group, tl, d_off, d_fillc, d_gterms);
                dim3 grid((tl + 255) / 256, (b + Btg - 1) / Btg);
                // (28 KB of shared memory requested, 4 KB used: at most seven of these long-running CTAs per SM, so that a 256-thread
                //  slot stays free on every SM for the short kernels of the resolver's chain)
                k_conflict_groups<<<grid, 256, std::max<size_t>((size_t)Btg * 32, 28 * 1024), S>>>(d_rows, Wp, W, t0, b, Btg, d_ngh + (n - 2), d_off, d_gterms, mode, bm, GW32, npred);
                c->cnt.kernel_launches += 4;
            }
            k_conflict_block<<<(b * 32 + 255) / 256, 256, 0, S>>>(d_rows, Wp, W, t0, b, mode & 0xff, cbn);
            SK_CUDA(c, cudaEventRecord(e_conf[par], S));
            // ---- main stream
            SK_CUDA(c, cudaStreamWaitEvent(M, e_conf[par], 0));
            if (n >= 1) { k_conflict_prev<<<(b * 32 + 255) / 256, 256, 0, M>>>(d_rows, Wp, W, t0, b, t0 - B, B, mode & 0xff, d_group, bm, GW32, npred); c->cnt.kernel_launches++; }
            k_free_lists<<<b, 256, 0, M>>>(bm, GW32, d_ng, d_fl, d_fcnt);
            k_first_fit_lists<<<1, 1024, kListSmem, M>>>(t0, b, bm, GW32, d_group, d_ng, d_fl, d_fcnt, cbn);
            SK_CUDA(c, cudaMemcpyAsync(d_ngh + n, d_ng, 4, cudaMemcpyDeviceToDevice, M));
            SK_CUDA(c, cudaEventRecord(e_res[par], M));
            c->cnt.kernel_launches += 3;
        }
        SK_CUDA(c, cudaGetLastError());
        u32 ngp = 0;
        SK_CUDA(c, cudaMemcpyAsync(&ngp, d_ng, 4, cudaMemcpyDeviceToHost, M));
        SK_CUDA(c, cudaStreamSynchronize(M));
        SK_CUDA(c, cudaStreamSynchronize(S));
        SK_CUDA(c, cudaStreamSynchronize(c->stream));
        *ngroups = ngp;
        return SK_OK;
    }
    for (int t0 = 0; t0 < count; t0 += B) {
        const int b = std::min(B, count - t0);
        SK_CUDA(c, cudaMemsetAsync(d_bitmap, 0, (size_t)b * GW32 * 4, c->stream));
        if (t0 > 0 && csr) {
            SK_CUDA(c, cudaMemsetAsync(d_gmin, 0xff, 4, c->stream));
            k_csr_count<<<(B + 255) / 256, 256, 0, c->stream>>>(d_group, t0 - B, t0, d_cnt, d_gmin);      // the previous block's terms
            k_csr_scan<<<1, 1024, 0, c->stream>>>(d_cnt, d_ng, d_off, d_gmin);
            SK_CUDA(c, cudaMemsetAsync(d_fillc, 0, ((size_t)t0 + 1) * 4, c->stream));
            k_csr_fill<<<(t0 + 255) / 256, 256, 0, c->stream>>>(d_rows, Wp, W, d_group, t0, d_off, d_fillc, d_gterms);
            dim3 grid((t0 + 255) / 256, (b + Btg - 1) / Btg);
            k_conflict_groups<<<grid, 256, (size_t)Btg * 32, c->stream>>>(d_rows, Wp, W, t0, b, Btg, d_ng, d_off, d_gterms, mode, d_bitmap, GW32,
                                                                         reinterpret_cast<unsigned long long*>(c->d_err) + 1);
            c->cnt.kernel_launches += 4;
        } else if (t0 > 0) {
            dim3 grid((t0 + 255) / 256, (b + Bt - 1) / Bt);
            k_conflict_bitmap<<<grid, 256, smem, c->stream>>>(d_rows, Wp, W, t0, b, Bt, d_group, mode, d_bitmap, GW32);
            c->cnt.kernel_launches++;
        }
        if (use_lists) {
            k_free_lists<<<b, 256, 0, c->stream>>>(d_bitmap, GW32, d_ng, d_fl, d_fcnt);
            k_conflict_block<<<(b * 32 + 255) / 256, 256, 0, c->stream>>>(d_rows, Wp, W, t0, b, mode & 0xff, d_cb);
            k_first_fit_lists<<<1, 1024, kListSmem, c->stream>>>(t0, b, d_bitmap, GW32, d_group, d_ng, d_fl, d_fcnt, d_cb);
            c->cnt.kernel_launches++;
        } else {
            k_first_free<<<b, 256, 0, c->stream>>>(d_bitmap, GW32, d_ng, d_ff);
            if ((mode & kOrderedFit) || legacy_resolver) k_first_fit_block<<<1, 1024, 0, c->stream>>>(d_rows, Wp, W, t0, b, mode, d_bitmap, GW32, d_group, d_ng, d_ff);
            else k_first_fit_threads<<<1, 1024, 0, c->stream>>>(d_rows, Wp, W, t0, b, mode, d_bitmap, GW32, d_group, d_ng, d_ff);
        }
        c->cnt.kernel_launches += 2;
    }
    SK_CUDA(c, cudaGetLastError());
    u32 ng = 0;
    SK_CUDA(c, cudaMemcpyAsync(&ng, d_ng, 4, cudaMemcpyDeviceToHost, c->stream));
    SK_CUDA(c, cudaStreamSynchronize(c->stream));
    *ngroups = ng;                       // (scope frees the scratch buffers)
    return SK_OK;
}

// ------------------------------------------------------------------------------- sk_rows ------
struct sk_rows {
    sk_ctx* ctx = nullptr;
    uint64_t n = 0, cap = 0, count = 0;
    DMat m;                      // rows (R) always allocated; cols (C) on first conj_layer
    bool r_valid = true, c_valid = false;
    size_t rows_bytes = 0, cols_bytes = 0, sgn_bytes = 0;
};

extern "C" int32_t sk_rows_create(sk_ctx* c, uint64_t n, uint64_t capacity, sk_rows** out) {
    if (!c || !out) return SK_EARG;
    *out = nullptr;
    if (n == 0) SK_FAIL(c, SK_EDIM, "rows: n must be >= 1");
    if (capacity == 0) capacity = 1;
    if (capacity > (1ull << 26)) SK_FAIL(c, SK_EDIM, "rows: capacity %llu too large", (unsigned long long)capacity);
    sk_rows* r = new sk_rows();
    r->ctx = c; r->n = n; r->cap = capacity;
    r->m.n = n; r->m.W = uint32_t((n + 63) / 64); r->m.Wp = (r->m.W + 1) & ~1u;
    r->m.RW = uint32_t(((capacity + 63) / 64 + 1) & ~1ull);
    r->rows_bytes = (size_t)64 * r->m.RW * 2 * r->m.Wp * 8;
    r->cols_bytes = (size_t)n * 2 * r->m.RW * 8;
    r->sgn_bytes = (size_t)r->m.RW * 8;
    if (cudaMalloc(&r->m.rows, r->rows_bytes) || cudaMalloc(&r->m.sgn, r->sgn_bytes)) { sk_rows_destroy(r); SK_FAIL(c, SK_ECUDA, "cudaMalloc failed for %llu rows", (unsigned long long)capacity); }
    SK_CUDA(c, cudaMemsetAsync(r->m.rows, 0, r->rows_bytes, c->stream));
    SK_CUDA(c, cudaMemsetAsync(r->m.sgn, 0, r->sgn_bytes, c->stream));
    *out = r;
    return SK_OK;
}
extern "C" void sk_rows_destroy(sk_rows* r) {
    if (!r) return;
    cudaSetDevice(r->ctx->device);
    cudaStreamSynchronize(r->ctx->stream);
    cudaFree(r->m.rows); cudaFree(r->m.cols); cudaFree(r->m.sgn);
    delete r;
}
extern "C" uint64_t sk_rows_count(const sk_rows* r) { return r ? r->count : 0; }

static int32_t rows_need_r(sk_rows* r) {
    if (r->r_valid) return SK_OK;
    int32_t rc = dm_transpose_c2r(r->ctx, r->m);
    if (!rc) r->r_valid = true;
    return rc;
}
static int32_t rows_need_c(sk_rows* r) {
    sk_ctx* c = r->ctx;
    if (!r->m.cols) SK_CUDA(c, cudaMalloc(&r->m.cols, r->cols_bytes));
    if (r->c_valid) return SK_OK;
    int32_t rc = dm_transpose_r2c(c, r->m);
    if (!rc) r->c_valid = true;
    return rc;
}

extern "C" int32_t sk_rows_upload(sk_rows* r, const uint64_t* x, const uint64_t* z, const uint8_t* sign, uint64_t m) {
    if (!r || (m && (!x || !z || !sign))) return SK_EARG;
    sk_ctx* c = r->ctx;
    if (m > r->cap) SK_FAIL(c, SK_EDIM, "rows: %llu rows exceed the capacity %llu", (unsigned long long)m, (unsigned long long)r->cap);
    const int W = r->m.W; const size_t words = (size_t)m * W;
    SK_CUDA(c, cudaMemsetAsync(r->m.rows, 0, r->rows_bytes, c->stream));
    SK_CUDA(c, cudaMemsetAsync(r->m.sgn, 0, r->sgn_bytes, c->stream));
    if (m) {
        int32_t rc = sk_ctx_reserve_tmp(c, words * 16 + m + 64);
        if (rc) return rc;
        u64* dx = (u64*)c->d_tmp; u64* dz = dx + words; uint8_t* ds = (uint8_t*)(dz + words);
        SK_CUDA(c, cudaMemcpyAsync(dx, x, words * 8, cudaMemcpyHostToDevice, c->stream));
        SK_CUDA(c, cudaMemcpyAsync(dz, z, words * 8, cudaMemcpyHostToDevice, c->stream));
        SK_CUDA(c, cudaMemcpyAsync(ds, sign, m, cudaMemcpyHostToDevice, c->stream));
        k_pack_rows<<<(unsigned)((words + 255) / 256), 256, 0, c->stream>>>(dx, dz, r->m.rows, int(m), W, r->m.Wp, int(m), 0);
        k_bytes_to_signs<<<(unsigned)((m + 255) / 256), 256, 0, c->stream>>>(ds, r->m.sgn, int(m), int(m), 0);
        c->cnt.kernel_launches += 2;
        SK_CUDA(c, cudaGetLastError());
        SK_CUDA(c, cudaStreamSynchronize(c->stream));
    }
    r->count = m; r->r_valid = true; r->c_valid = false;
    return SK_OK;
}
extern "C" int32_t sk_rows_append(sk_rows* r, const uint64_t* x, const uint64_t* z, const uint8_t* sign, uint64_t m) {
    if (!r || (m && (!x || !z || !sign))) return SK_EARG;
    sk_ctx* c = r->ctx;
    if (m == 0) return SK_OK;
    if (r->count + m > r->cap) SK_FAIL(c, SK_EDIM, "rows: appending %llu rows to %llu exceeds the capacity %llu", (unsigned long long)m, (unsigned long long)r->count, (unsigned long long)r->cap);
    int32_t rc = rows_need_r(r);
    if (rc) return rc;
    const int W = r->m.W; const size_t words = (size_t)m * W;
    rc = sk_ctx_reserve_tmp(c, words * 16 + m + 64);
    if (rc) return rc;
    u64* dx = (u64*)c->d_tmp; u64* dz = dx + words; uint8_t* ds = (uint8_t*)(dz + words);
    SK_CUDA(c, cudaMemcpyAsync(dx, x, words * 8, cudaMemcpyHostToDevice, c->stream));
    SK_CUDA(c, cudaMemcpyAsync(dz, z, words * 8, cudaMemcpyHostToDevice, c->stream));
    SK_CUDA(c, cudaMemcpyAsync(ds, sign, m, cudaMemcpyHostToDevice, c->stream));
    // rows [count, count + m) of the R form (all-zero until now); sign bits likewise
    k_pack_rows<<<(unsigned)((words + 255) / 256), 256, 0, c->stream>>>(dx, dz, r->m.rows + (size_t)2 * r->count * r->m.Wp, int(m), W, r->m.Wp, int(m), 0);
    k_bytes_to_signs_at<<<(unsigned)((m + 255) / 256), 256, 0, c->stream>>>(ds, r->m.sgn, int(m), int(r->count));
    c->cnt.kernel_launches += 2;
    SK_CUDA(c, cudaGetLastError());
    SK_CUDA(c, cudaStreamSynchronize(c->stream));
    r->count += m; r->c_valid = false;
    return SK_OK;
}
extern "C" int32_t sk_commute_matrix_tile(sk_rows* r, int mode, uint64_t i0, uint64_t ni, uint64_t j0, uint64_t nj, uint64_t* out_bits) {
    if (!r || (!out_bits && ni && nj)) return SK_EARG;
    sk_ctx* c = r->ctx;
    if (mode != 0 && mode != 1) SK_FAIL(c, SK_EARG, "commute_matrix_tile: mode must be 0 (general) or 1 (qubit-wise)");
    if (i0 + ni > r->count || j0 + nj > r->count) SK_FAIL(c, SK_EDIM, "commute_matrix_tile: tile [%llu,+%llu) x [%llu,+%llu) outside the %llu rows", (unsigned long long)i0, (unsigned long long)ni, (unsigned long long)j0, (unsigned long long)nj, (unsigned long long)r->count);
    if (ni == 0 || nj == 0) return SK_OK;
    int32_t rc = rows_need_r(r);
    if (rc) return rc;
    const size_t words = (nj + 63) / 64, total = ni * words;
    rc = sk_ctx_reserve_tmp(c, total * 8 + 64);
    if (rc) return rc;
    u64* d_out = (u64*)c->d_tmp;
    const size_t threads = total * 32;
    k_commute_tile<<<(unsigned)((threads + 255) / 256), 256, 0, c->stream>>>(r->m.rows, r->m.Wp, r->m.W, mode, int(i0), int(ni), int(j0), int(nj), int(words), d_out);
    c->cnt.kernel_launches++;
    c->cnt.pred_evals += ni * nj;
    SK_CUDA(c, cudaGetLastError());
    SK_CUDA(c, cudaMemcpyAsync(out_bits, d_out, total * 8, cudaMemcpyDeviceToHost, c->stream));
    SK_CUDA(c, cudaStreamSynchronize(c->stream));
    return SK_OK;
}
extern "C" int32_t sk_rows_download(sk_rows* r, uint64_t* x, uint64_t* z, uint8_t* sign) {
    if (!r) return SK_EARG;
    sk_ctx* c = r->ctx;
    const uint64_t m = r->count;
    if (m == 0) return SK_OK;
    if (!x || !z || !sign) return SK_EARG;
    int32_t rc = rows_need_r(r);
    if (rc) return rc;
    const int W = r->m.W; const size_t words = (size_t)m * W;
    rc = sk_ctx_reserve_tmp(c, words * 16 + m + 64);
    if (rc) return rc;
    u64* dx = (u64*)c->d_tmp; u64* dz = dx + words; uint8_t* ds = (uint8_t*)(dz + words);
    k_unpack_rows<<<(unsigned)((words + 255) / 256), 256, 0, c->stream>>>(r->m.rows, dx, dz, int(m), W, r->m.Wp, int(m), 0);
    k_signs_to_bytes<<<(unsigned)((m + 255) / 256), 256, 0, c->stream>>>(r->m.sgn, ds, int(m), int(m), 0);
    c->cnt.kernel_launches += 2;
    SK_CUDA(c, cudaGetLastError());
    SK_CUDA(c, cudaMemcpyAsync(x, dx, words * 8, cudaMemcpyDeviceToHost, c->stream));
    SK_CUDA(c, cudaMemcpyAsync(z, dz, words * 8, cudaMemcpyDeviceToHost, c->stream));
    SK_CUDA(c, cudaMemcpyAsync(sign, ds, m, cudaMemcpyDeviceToHost, c->stream));
    return check_ws(c);
}

extern "C" int32_t sk_rows_conj_layer(sk_rows* r, const sk_gate* gates, size_t ngates) {
    if (!r || (!gates && ngates)) return SK_EARG;
    sk_ctx* c = r->ctx;
    if (ngates == 0 || r->count == 0) return SK_OK;
    for (size_t i = 0; i < ngates; ++i) {
        int32_t rc = validate_gate(c, gates[i], r->n, i);
        if (rc) return rc;
        if (gates[i].kind >= SK_M) SK_FAIL(c, SK_EUNSUPPORTED, "gate %zu: only Clifford gates conjugate a row set (SPEC:518)", i);
    }
    int32_t rc = rows_need_c(r);
    if (rc) return rc;
    std::vector<sk_gate> ordered; std::vector<uint32_t> sizes, scratch;
    sk_layer_run(gates, ngates, r->n, scratch, ordered, sizes);
    rc = sk_ctx_reserve_gates(c, ngates * sizeof(sk_gate));
    if (rc) return rc;
    SK_CUDA(c, cudaMemcpyAsync(c->d_gates, ordered.data(), ngates * sizeof(sk_gate), cudaMemcpyHostToDevice, c->stream));
    size_t off = 0;
    for (uint32_t s : sizes) { dm_launch_layer(c, r->m, (const sk_gate*)c->d_gates + off, int(s)); off += s; }
    SK_CUDA(c, cudaGetLastError());
    SK_CUDA(c, cudaStreamSynchronize(c->stream));
    r->r_valid = false;
    return SK_OK;
}

// uploads p as [x Wp | z Wp] into the tmp buffer at byte offset `at`
static int32_t upload_pauli(sk_ctx* c, const DMat& m, const uint64_t* px, const uint64_t* pz, u64* d_p) {
    std::vector<u64> h(2 * m.Wp, 0);
    for (uint32_t w = 0; w < m.W; ++w) { h[w] = px[w]; h[m.Wp + w] = pz[w]; }
    SK_CUDA(c, cudaMemcpyAsync(d_p, h.data(), h.size() * 8, cudaMemcpyHostToDevice, c->stream));
    SK_CUDA(c, cudaStreamSynchronize(c->stream));      // h dies at return
    return SK_OK;
}

extern "C" int32_t sk_commutation_vector(sk_rows* r, const uint64_t* px, const uint64_t* pz, uint64_t* out_bits) {
    if (!r || !px || !pz || !out_bits) return SK_EARG;
    sk_ctx* c = r->ctx;
    const int m = int(r->count);
    if (m == 0) return SK_OK;
    int32_t rc = rows_need_r(r);
    if (rc) return rc;
    const size_t ow = (size_t)(m + 63) / 64;
    rc = sk_ctx_reserve_tmp(c, (2 * r->m.Wp + ow + 8) * 8);
    if (rc) return rc;
    u64* d_p = (u64*)c->d_tmp; u64* d_out = d_p + 2 * r->m.Wp;
    rc = upload_pauli(c, r->m, px, pz, d_p);
    if (rc) return rc;
    SK_CUDA(c, cudaMemsetAsync(d_out, 0, ow * 8, c->stream));
    k_commutation_vector<<<(unsigned)((m * 32 + 255) / 256), 256, 0, c->stream>>>(r->m.rows, r->m.Wp, r->m.W, m, d_p, d_out);
    c->cnt.kernel_launches++;
    SK_CUDA(c, cudaGetLastError());
    SK_CUDA(c, cudaMemcpyAsync(out_bits, d_out, ow * 8, cudaMemcpyDeviceToHost, c->stream));
    SK_CUDA(c, cudaStreamSynchronize(c->stream));
    return SK_OK;
}

extern "C" int32_t sk_rowsum_plus_i_where_anticommuting(sk_rows* r, const uint64_t* px, const uint64_t* pz,
                                                        uint8_t psign, uint64_t* n_updated) {
    if (!r || !px || !pz) return SK_EARG;
    sk_ctx* c = r->ctx;
    if (n_updated) *n_updated = 0;
    const int m = int(r->count);
    if (m == 0) return SK_OK;
    int32_t rc = rows_need_r(r);
    if (rc) return rc;
    rc = sk_ctx_reserve_tmp(c, (2 * r->m.Wp + 8) * 8);
    if (rc) return rc;
    u64* d_p = (u64*)c->d_tmp; unsigned long long* d_n = (unsigned long long*)(d_p + 2 * r->m.Wp); uint8_t* d_s = (uint8_t*)(d_n + 1);
    rc = upload_pauli(c, r->m, px, pz, d_p);
    if (rc) return rc;
    SK_CUDA(c, cudaMemsetAsync(d_n, 0, 8, c->stream));
    SK_CUDA(c, cudaMemcpyAsync(d_s, &psign, 1, cudaMemcpyHostToDevice, c->stream));
    launch_push(c, r->m.W, m, r->m.rows, r->m.sgn, int(r->m.Wp), int(r->m.W), 0, m, (const int*)nullptr, (const u64*)d_p,
                (const uint8_t*)d_s, (const int*)nullptr, 1, c->d_err, d_n);
    SK_CUDA(c, cudaGetLastError());
    unsigned long long hn = 0;
    SK_CUDA(c, cudaMemcpyAsync(&hn, d_n, 8, cudaMemcpyDeviceToHost, c->stream));
    r->c_valid = false;
    rc = check_ws(c);
    if (n_updated) *n_updated = hn;
    return rc;
}

static int32_t dup_pairs(sk_ctx* c, const u64* d_rows, int Wp, int W, int m, const int* d_lvl, int* d_pair /* [m] */, u64* d_hash /* [m] */) {
    k_row_hash<<<(unsigned)((m * 32 + 255) / 256), 256, 0, c->stream>>>(d_rows, Wp, W, m, d_hash);
    k_dup_rank<<<(unsigned)((m + 255) / 256), 256, 0, c->stream>>>(d_rows, Wp, W, m, d_hash, d_lvl, d_pair);
    c->cnt.kernel_launches += 2;
    SK_CUDA(c, cudaGetLastError());
    return SK_OK;
}

extern "C" int32_t sk_find_first_duplicate(sk_rows* r, int* found, uint64_t* i, uint64_t* j) {
    if (!r || !found || !i || !j) return SK_EARG;
    sk_ctx* c = r->ctx;
    *found = 0;
    const int m = int(r->count);
    if (m < 2) return SK_OK;
    int32_t rc = rows_need_r(r);
    if (rc) return rc;
    rc = sk_ctx_reserve_tmp(c, (size_t)m * 12 + 64);
    if (rc) return rc;
    u64* d_hash = (u64*)c->d_tmp; int* d_pair = (int*)(d_hash + m); unsigned long long* d_min = (unsigned long long*)(d_hash + m + (m + 1) / 2 + 1);
    rc = dup_pairs(c, r->m.rows, r->m.Wp, r->m.W, m, nullptr, d_pair, d_hash);
    if (rc) return rc;
    SK_CUDA(c, cudaMemsetAsync(d_min, 0xFF, 8, c->stream));
    k_min_pair<<<(unsigned)((m + 255) / 256), 256, 0, c->stream>>>(d_pair, m, d_min);
    c->cnt.kernel_launches++;
    unsigned long long key = ~0ull;
    SK_CUDA(c, cudaMemcpyAsync(&key, d_min, 8, cudaMemcpyDeviceToHost, c->stream));
    SK_CUDA(c, cudaStreamSynchronize(c->stream));
    if (key != ~0ull) { *found = 1; *i = key >> 32; *j = key & 0xffffffffu; }
    return SK_OK;
}

extern "C" int32_t sk_weight_sum(sk_rows* r, uint64_t* out) {
    if (!r || !out) return SK_EARG;
    sk_ctx* c = r->ctx;
    *out = 0;
    const int m = int(r->count);
    if (m == 0) return SK_OK;
    int32_t rc = rows_need_r(r);
    if (rc) return rc;
    rc = sk_ctx_reserve_tmp(c, 64);
    if (rc) return rc;
    unsigned long long* d_o = (unsigned long long*)c->d_tmp;
    SK_CUDA(c, cudaMemsetAsync(d_o, 0, 8, c->stream));
    k_weight_sum<<<std::min(1024, (m * int(r->m.W) + 255) / 256), 256, 0, c->stream>>>(r->m.rows, r->m.Wp, r->m.W, m, nullptr, d_o);
    c->cnt.kernel_launches++;
    SK_CUDA(c, cudaGetLastError());
    unsigned long long h = 0;
    SK_CUDA(c, cudaMemcpyAsync(&h, d_o, 8, cudaMemcpyDeviceToHost, c->stream));
    SK_CUDA(c, cudaStreamSynchronize(c->stream));
    *out = h;
    return SK_OK;
}

extern "C" int32_t sk_group_first_fit(sk_rows* r, int mode, uint32_t* group_of, uint64_t* ngroups) {
    if (!r || !group_of || !ngroups || (mode != 0 && mode != 1)) return SK_EARG;
    sk_ctx* c = r->ctx;
    *ngroups = 0;
    const int m = int(r->count);
    if (m == 0) SK_FAIL(c, SK_EARG, "group_greedy: empty input (SPEC:448)");
    int32_t rc = rows_need_r(r);
    if (rc) return rc;
    u32* d_group = nullptr;
    SK_CUDA(c, cudaMalloc(&d_group, (size_t)m * 4));
    rc = device_first_fit(c, r->m.rows, r->m.Wp, r->m.W, m, mode, d_group, ngroups);
    if (!rc) {
        cudaError_t e = cudaMemcpyAsync(group_of, d_group, (size_t)m * 4, cudaMemcpyDeviceToHost, c->stream);
        if (!e) e = cudaStreamSynchronize(c->stream);
        if (e) { cudaFree(d_group); SK_FAIL(c, SK_ECUDA, "group download: %s", cudaGetErrorString(e)); }
    }
    cudaFree(d_group);
    return rc;
}

// ---- first fit with the pair matrix sharded by row blocks (north_star "Commutation grouping shards the pair matrix
// by row blocks").  Every shard holds the replicated input and the replicated group assignment; the conflict bitmap of a block
// of 1024 terms against the placed groups -- where the predicate evaluations are -- is split: shard s of S evaluates the groups
// of the bitmap words w with w % S == s.  The driver (paper_2507_03092_b200/group_sharded.py: torch.distributed / NCCL, or several
// shards in one process) ORs the shards' bitmaps -- an allreduce-SUM, the words are disjoint -- and every shard then resolves the
// block itself (the resolver is sequential in the term index and deterministic: identical assignments everywhere).
struct sk_group_shard {
    sk_ctx* ctx = nullptr; sk_rows* rows = nullptr;
    int mode = 0, shard = 0, nshards = 1, count = 0, B = 0, GW32 = 0;
    u32 *d_group = nullptr, *d_ng = nullptr, *d_ff = nullptr, *d_cnt = nullptr, *d_off = nullptr, *d_fillc = nullptr, *d_gmin = nullptr;
    u64* d_gterms = nullptr;
    uint64_t next_block = 0;
};
extern "C" void sk_group_shard_destroy(sk_group_shard* g) {
    if (!g) return;
    cudaSetDevice(g->ctx->device);
    for (void* p : {(void*)g->d_group, (void*)g->d_ng, (void*)g->d_cnt, (void*)g->d_off, (void*)g->d_fillc, (void*)g->d_gterms}) if (p) cudaFree(p);
    delete g;
}
extern "C" int32_t sk_group_shard_create(sk_rows* r, int mode, uint32_t shard, uint32_t nshards, sk_group_shard** out) {
    if (!r || !out || (mode != 0 && mode != 1)) return SK_EARG;
    *out = nullptr;
    sk_ctx* c = r->ctx;
    if (nshards == 0 || shard >= nshards) SK_FAIL(c, SK_EARG, "group shard %u of %u", shard, nshards);
    if (r->count == 0) SK_FAIL(c, SK_EARG, "group_greedy: empty input (SPEC:448)");
    if (r->m.W > 2) SK_FAIL(c, SK_EUNSUPPORTED, "sharded grouping uses the group-major conflict kernel: rows of at most 128 qubits (BASELINE config 4), got %llu", (unsigned long long)r->n);
    int32_t rc = rows_need_r(r);
    if (rc) return rc;
    sk_group_shard* g = new sk_group_shard();
    g->ctx = c; g->rows = r; g->mode = mode; g->shard = int(shard); g->nshards = int(nshards);
    g->count = int(r->count); g->B = std::min(g->count, 1024); g->GW32 = g->count / 32 + 2;
    const size_t n = size_t(g->count);
    cudaError_t e = cudaMalloc(&g->d_group, n * 4);
    if (!e) e = cudaMalloc(&g->d_ng, 4 + (size_t)g->B * 4);
    if (!e) e = cudaMalloc(&g->d_cnt, (n + 4) * 4);
    if (!e) e = cudaMalloc(&g->d_off, (n + 2) * 4);
    if (!e) e = cudaMalloc(&g->d_fillc, (n + 2) * 4);
    if (!e) e = cudaMalloc(&g->d_gterms, n * 32);
    if (e) { sk_group_shard_destroy(g); SK_FAIL(c, SK_ECUDA, "cudaMalloc failed for a grouping shard: %s", cudaGetErrorString(e)); }
    g->d_ff = g->d_ng + 1; g->d_gmin = g->d_cnt + n + 3;
    cudaMemsetAsync(g->d_ng, 0, 4, c->stream); cudaMemsetAsync(g->d_cnt, 0, (n + 4) * 4, c->stream);
    *out = g;
    return SK_OK;
}
extern "C" uint64_t sk_group_shard_blocks(const sk_group_shard* g) { return g ? uint64_t((g->count + g->B - 1) / g->B) : 0; }
/* u32 words of one block's conflict bitmap: rows of GW32 words, one row per block term */
extern "C" uint64_t sk_group_shard_bitmap_words(const sk_group_shard* g) { return g ? uint64_t(g->B) * uint64_t(g->GW32) : 0; }
/* Conflicts of block k's terms with the groups this shard owns, into d_bitmap (device, bitmap_words u32, zeroed here). */
extern "C" int32_t sk_group_shard_conflicts(sk_group_shard* g, uint64_t block, uint32_t* d_bitmap) {
    if (!g || !d_bitmap) return SK_EARG;
    sk_ctx* c = g->ctx;
    if (block != g->next_block) SK_FAIL(c, SK_EARG, "grouping shard: block %llu out of order (next is %llu)", (unsigned long long)block, (unsigned long long)g->next_block);
    const int t0 = int(block) * g->B;
    if (t0 >= g->count) SK_FAIL(c, SK_EARG, "grouping shard: block %llu beyond the input", (unsigned long long)block);
    const int b = std::min(g->B, g->count - t0);
    const DMat& m = g->rows->m;
    SK_CUDA(c, cudaMemsetAsync(d_bitmap, 0, (size_t)g->B * g->GW32 * 4, c->stream));
    if (t0 > 0) {
        const int Btg = std::min(g->B, 128);
        SK_CUDA(c, cudaMemsetAsync(g->d_gmin, 0xff, 4, c->stream));
        k_csr_count<<<(g->B + 255) / 256, 256, 0, c->stream>>>(g->d_group, t0 - g->B, t0, g->d_cnt, g->d_gmin);
        k_csr_scan<<<1, 1024, 0, c->stream>>>(g->d_cnt, g->d_ng, g->d_off, g->d_gmin);
        SK_CUDA(c, cudaMemsetAsync(g->d_fillc, 0, ((size_t)t0 + 1) * 4, c->stream));
        k_csr_fill<<<(t0 + 255) / 256, 256, 0, c->stream>>>(m.rows, m.Wp, m.W, g->d_group, t0, g->d_off, g->d_fillc, g->d_gterms);
        dim3 grid(((t0 + g->nshards - 1) / g->nshards + 255) / 256 + 1, (b + Btg - 1) / Btg);
        k_conflict_groups<<<grid, 256, (size_t)Btg * 32, c->stream>>>(m.rows, m.Wp, m.W, t0, b, Btg, g->d_ng, g->d_off, g->d_gterms, g->mode, d_bitmap, g->GW32,
                                                                     reinterpret_cast<unsigned long long*>(c->d_err) + 1, g->shard, g->nshards);
        c->cnt.kernel_launches += 4;
    }
    SK_CUDA(c, cudaGetLastError());
    return SK_OK;
}
/* First fit of block k given the COMBINED bitmap (all shards' words OR-ed together); every shard runs it and gets the same groups. */
extern "C" int32_t sk_group_shard_resolve(sk_group_shard* g, uint64_t block, uint32_t* d_bitmap) {
    if (!g || !d_bitmap) return SK_EARG;
    sk_ctx* c = g->ctx;
    if (block != g->next_block) SK_FAIL(c, SK_EARG, "grouping shard: block %llu out of order (next is %llu)", (unsigned long long)block, (unsigned long long)g->next_block);
    const int t0 = int(block) * g->B, b = std::min(g->B, g->count - t0);
    const DMat& m = g->rows->m;
    k_first_free<<<b, 256, 0, c->stream>>>(d_bitmap, g->GW32, g->d_ng, g->d_ff);
    k_first_fit_threads<<<1, 1024, 0, c->stream>>>(m.rows, m.Wp, m.W, t0, b, g->mode, d_bitmap, g->GW32, g->d_group, g->d_ng, g->d_ff);
    c->cnt.kernel_launches += 2;
    SK_CUDA(c, cudaGetLastError());
    g->next_block++;
    return SK_OK;
}
extern "C" int32_t sk_group_shard_result(sk_group_shard* g, uint32_t* group_of, uint64_t* ngroups) {
    if (!g || !group_of || !ngroups) return SK_EARG;
    sk_ctx* c = g->ctx;
    if (g->next_block != sk_group_shard_blocks(g)) SK_FAIL(c, SK_EARG, "grouping shard: %llu of %llu blocks resolved", (unsigned long long)g->next_block, (unsigned long long)sk_group_shard_blocks(g));
    u32 ng = 0;
    SK_CUDA(c, cudaMemcpyAsync(&ng, g->d_ng, 4, cudaMemcpyDeviceToHost, c->stream));
    SK_CUDA(c, cudaMemcpyAsync(group_of, g->d_group, (size_t)g->count * 4, cudaMemcpyDeviceToHost, c->stream));
    SK_CUDA(c, cudaStreamSynchronize(c->stream));
    *ngroups = ng;
    return SK_OK;
}

extern "C" int32_t sk_verify_grouping(sk_rows* r, int mode, const uint32_t* group_of, uint64_t* nviolations) {
    if (!r || !group_of || !nviolations || (mode != 0 && mode != 1)) return SK_EARG;
    sk_ctx* c = r->ctx;
    *nviolations = 0;
    const int m = int(r->count);
    if (m == 0) return SK_OK;
    int32_t rc = rows_need_r(r);
    if (rc) return rc;
    rc = sk_ctx_reserve_tmp(c, (size_t)m * 4 + 64);
    if (rc) return rc;
    unsigned long long* d_n = (unsigned long long*)c->d_tmp; u32* d_g = (u32*)(d_n + 1);
    SK_CUDA(c, cudaMemsetAsync(d_n, 0, 8, c->stream));
    SK_CUDA(c, cudaMemcpyAsync(d_g, group_of, (size_t)m * 4, cudaMemcpyHostToDevice, c->stream));
    k_verify_grouping<<<(unsigned)((m + 255) / 256), 256, 0, c->stream>>>(r->m.rows, r->m.Wp, r->m.W, m, d_g, mode, d_n);
    c->cnt.kernel_launches++;
    SK_CUDA(c, cudaGetLastError());
    unsigned long long h = 0;
    SK_CUDA(c, cudaMemcpyAsync(&h, d_n, 8, cudaMemcpyDeviceToHost, c->stream));
    SK_CUDA(c, cudaStreamSynchronize(c->stream));
    *nviolations = h;
    return SK_OK;
}

// ------------------------------------------------------------------------------- transpile ----
struct sk_pbc {
    sk_ctx* ctx = nullptr;
    uint64_t n = 0; int W = 0;
    uint64_t stats[5] = {0, 0, 0, 0, 0};
    std::vector<std::vector<uint32_t>> layers;        // T-row ids per layer, forward time order
    std::vector<u64> tx, tz; std::vector<uint8_t> ts; // all T rows (row-major, W words), host cache
    std::vector<u64> mx, mz; std::vector<uint8_t> ms; // final M_tab, 2n rows
};
extern "C" void sk_pbc_destroy(sk_pbc* p) { delete p; }
extern "C" int32_t sk_pbc_stats(sk_pbc* p, uint64_t out5[5]) { if (!p || !out5) return SK_EARG; for (int k = 0; k < 5; ++k) out5[k] = p->stats[k]; return SK_OK; }
extern "C" uint64_t sk_pbc_layer_rows(sk_pbc* p, uint64_t layer) { return (p && layer < p->layers.size()) ? p->layers[layer].size() : 0; }
extern "C" int32_t sk_pbc_layer_download(sk_pbc* p, uint64_t layer, uint64_t* x, uint64_t* z, uint8_t* sign) {
    if (!p || layer >= p->layers.size() || !x || !z || !sign) return SK_EARG;
    const auto& L = p->layers[layer];
    for (size_t k = 0; k < L.size(); ++k) {
        std::copy(&p->tx[(size_t)L[k] * p->W], &p->tx[(size_t)L[k] * p->W] + p->W, x + k * p->W);
        std::copy(&p->tz[(size_t)L[k] * p->W], &p->tz[(size_t)L[k] * p->W] + p->W, z + k * p->W);
        sign[k] = p->ts[L[k]];
    }
    return SK_OK;
}
extern "C" int32_t sk_pbc_mtab_download(sk_pbc* p, uint64_t* x, uint64_t* z, uint8_t* sign) {
    if (!p || !x || !z || !sign) return SK_EARG;
    std::copy(p->mx.begin(), p->mx.end(), x); std::copy(p->mz.begin(), p->mz.end(), z); std::copy(p->ms.begin(), p->ms.end(), sign);
    return SK_OK;
}

extern "C" int32_t sk_transpile_ex(sk_ctx* c, uint64_t n, const sk_gate* gates, size_t ngates, uint32_t flags, sk_pbc** out);
extern "C" int32_t sk_transpile(sk_ctx* c, uint64_t n, const sk_gate* gates, size_t ngates, sk_pbc** out) {
    return sk_transpile_ex(c, n, gates, ngates, 0u, out);
}
// Default (flags 0 or SK_TRANSPILE_EXACT): unitary-exact form -- the backward walk of Algorithm 2 conjugates by the inverse
// gate (S <-> S^dagger) and Algorithm 3 / the safety pass place a row right after the last layer holding an anticommuting
// member.  SK_TRANSPILE_PUBLISHED: Algorithms 2-3 verbatim (see include/stabkit_b200.h and DESIGN.md section 8).
extern "C" int32_t sk_transpile_ex(sk_ctx* c, uint64_t n, const sk_gate* gates, size_t ngates, uint32_t flags, sk_pbc** out) {
    if (!c || !out || (!gates && ngates)) return SK_EARG;
    const bool exact = (flags & SK_TRANSPILE_PUBLISHED) == 0;
    const int fit_mode = exact ? kOrderedFit : 0;
    *out = nullptr;
    if (n == 0) SK_FAIL(c, SK_EDIM, "transpile: circuit has zero qubits");
    size_t end = ngates;
    while (end > 0 && gates[end - 1].kind == SK_M) --end;                    // terminal measurements are stripped
    size_t nT = 0;
    for (size_t i = 0; i < end; ++i) {
        int32_t rc = validate_gate(c, gates[i], n, i);
        if (rc) return rc;
        if (gates[i].kind == SK_M) SK_FAIL(c, SK_EUNSUPPORTED, "gate %zu: mid-circuit measurement is not supported by the transpiler (SPEC:519)", i);
        nT += (gates[i].kind == SK_T || gates[i].kind == SK_TDG);
    }
    // ---- Algorithm 2 on one C-form matrix: M_tab rows (stab [0,n), destab [NS,NS+n)) and the T rows
    //      at row-bits 2*NS + k, k = index of the T gate in forward time.  Unappended rows are all-zero,
    //      i.e. identity, and every Clifford rule maps identity to identity with sign 0, so "apply G to
    //      the rows appended so far" is simply "apply G to all rows".
    DMat m; m.n = n; m.W = uint32_t((n + 63) / 64); m.Wp = (m.W + 1) & ~1u;
    const int W = m.W, NS = 64 * W, T0 = 2 * NS;
    m.RW = uint32_t((2 * W + (nT + 63) / 64 + 1) & ~1ull);
    const size_t cols_bytes = (size_t)n * 2 * m.RW * 8, rows_bytes = (size_t)64 * m.RW * 2 * m.Wp * 8, sgn_bytes = (size_t)m.RW * 8;
    struct Guard { DMat* m; std::vector<void*> extra; ~Guard() { cudaFree(m->cols); cudaFree(m->rows); cudaFree(m->sgn); for (void* p : extra) cudaFree(p); } } guard{&m, {}};
    SK_CUDA(c, cudaMalloc(&m.cols, cols_bytes));
    SK_CUDA(c, cudaMalloc(&m.rows, rows_bytes));
    SK_CUDA(c, cudaMalloc(&m.sgn, sgn_bytes));
    SK_CUDA(c, cudaMemsetAsync(m.cols, 0, cols_bytes, c->stream));
    SK_CUDA(c, cudaMemsetAsync(m.rows, 0, rows_bytes, c->stream));
    SK_CUDA(c, cudaMemsetAsync(m.sgn, 0, sgn_bytes, c->stream));
    k_identity<<<(unsigned)((n + 255) / 256), 256, 0, c->stream>>>(m.cols, m.rows, int(n), m.RW, m.Wp, NS);
    c->cnt.kernel_launches++;
    {
        std::vector<sk_gate> rev; rev.reserve(end);
        size_t tk = nT;
        for (size_t k = end; k-- > 0;) {
            sk_gate g = gates[k];
            if (g.kind == SK_T || g.kind == SK_TDG) { --tk; g.kind = (g.kind == SK_T) ? SK_APPEND_T : SK_APPEND_TDG; g.q1 = uint32_t(T0 + tk); }
            else if (exact && g.kind == SK_S) g.kind = SK_SDG;
            else if (exact && g.kind == SK_SDG) g.kind = SK_S;
            rev.push_back(g);
        }
        std::vector<sk_gate> ordered; std::vector<uint32_t> sizes, scratch;
        sk_layer_run(rev.data(), rev.size(), n, scratch, ordered, sizes);   // append ops are single-qubit ops on q0
        if (!ordered.empty()) {
            int32_t rc = sk_ctx_reserve_gates(c, ordered.size() * sizeof(sk_gate));
            if (rc) return rc;
            SK_CUDA(c, cudaMemcpyAsync(c->d_gates, ordered.data(), ordered.size() * sizeof(sk_gate), cudaMemcpyHostToDevice, c->stream));
            size_t off = 0;
            for (uint32_t s : sizes) { dm_launch_layer(c, m, (const sk_gate*)c->d_gates + off, int(s)); off += s; }
            SK_CUDA(c, cudaGetLastError());
            SK_CUDA(c, cudaStreamSynchronize(c->stream));
        }
    }
    int32_t rc = dm_transpose_c2r(c, m);
    if (rc) return rc;
    u64* rowsT = m.rows + (size_t)2 * T0 * m.Wp;                             // R-form view of the T rows
    std::unique_ptr<sk_pbc> p_owner(new sk_pbc());       // released into *out on success only: every early return frees it
    sk_pbc* p = p_owner.get();
    p->ctx = c; p->n = n; p->W = W; p->stats[0] = nT;
    std::vector<int> lvl(nT, 0);
    uint64_t passes = 0;
    if (nT > 0) {
        // ---- Algorithm 3: first fit (GC) in forward time order == T-row id order
        u32* d_group = nullptr; int* d_lvl = nullptr; int* d_pair = nullptr; u64* d_hash = nullptr;
        SK_CUDA(c, cudaMalloc(&d_group, nT * 4)); guard.extra.push_back(d_group);
        SK_CUDA(c, cudaMalloc(&d_lvl, nT * 4)); guard.extra.push_back(d_lvl);
        SK_CUDA(c, cudaMalloc(&d_pair, nT * 4)); guard.extra.push_back(d_pair);
        SK_CUDA(c, cudaMalloc(&d_hash, nT * 8)); guard.extra.push_back(d_hash);
        uint64_t nl = 0;
        rc = device_first_fit(c, rowsT, m.Wp, W, int(nT), fit_mode, d_group, &nl);
        if (rc) return rc;
        SK_CUDA(c, cudaMemcpyAsync(lvl.data(), d_group, nT * 4, cudaMemcpyDeviceToHost, c->stream));
        SK_CUDA(c, cudaStreamSynchronize(c->stream));
        // ---- Algorithm 4, one pass = pairs from the pass-start state + ordered push-through
        std::vector<int> pair(nT); std::vector<u64> sg(m.RW);
        for (;;) {
            ++passes;
            SK_CUDA(c, cudaMemcpyAsync(d_lvl, lvl.data(), nT * 4, cudaMemcpyHostToDevice, c->stream));
            rc = dup_pairs(c, rowsT, m.Wp, W, int(nT), d_lvl, d_pair, d_hash);
            if (rc) return rc;
            SK_CUDA(c, cudaMemcpyAsync(pair.data(), d_pair, nT * 4, cudaMemcpyDeviceToHost, c->stream));
            SK_CUDA(c, cudaMemcpyAsync(sg.data(), m.sgn, sgn_bytes, cudaMemcpyDeviceToHost, c->stream));
            SK_CUDA(c, cudaStreamSynchronize(c->stream));
            auto sign_of = [&](int k) { const int rb = T0 + k; return int((sg[rb >> 6] >> (rb & 63)) & 1ull); };
            struct Push { int level, first, sign; };
            std::vector<Push> pushes; bool any = false;
            for (size_t j = 0; j < nT; ++j) {
                if (pair[j] < 0) continue;
                any = true;
                const int i = pair[j];
                if (sign_of(i) == sign_of(int(j))) pushes.push_back({lvl[i], i, sign_of(i)});   // equal signs: quarter rotation
                // opposite signs cancel; either way both rows leave the layer
            }
            if (!any) break;
            std::sort(pushes.begin(), pushes.end(), [](const Push& a, const Push& b) { return a.level != b.level ? a.level > b.level : a.first < b.first; });
            const int np = int(pushes.size());
            if (np > 0) {
                std::vector<int> idx(np), plevel(np); std::vector<uint8_t> psign(np);
                for (int k = 0; k < np; ++k) { idx[k] = pushes[k].first; plevel[k] = pushes[k].level; psign[k] = uint8_t(pushes[k].sign); }
                const size_t need = (size_t)np * 2 * m.Wp * 8 + (size_t)np * 9 + 256;
                rc = sk_ctx_reserve_tmp(c, need);
                if (rc) return rc;
                u64* d_push = (u64*)c->d_tmp; int* d_idx = (int*)(d_push + (size_t)np * 2 * m.Wp); int* d_plevel = d_idx + np; uint8_t* d_psign = (uint8_t*)(d_plevel + np);
                SK_CUDA(c, cudaMemcpyAsync(d_idx, idx.data(), np * 4, cudaMemcpyHostToDevice, c->stream));
                SK_CUDA(c, cudaMemcpyAsync(d_plevel, plevel.data(), np * 4, cudaMemcpyHostToDevice, c->stream));
                SK_CUDA(c, cudaMemcpyAsync(d_psign, psign.data(), np, cudaMemcpyHostToDevice, c->stream));
                k_gather_rows<<<(unsigned)(((size_t)np * 2 * m.Wp + 255) / 256), 256, 0, c->stream>>>(rowsT, m.Wp, d_idx, np, d_push);
                c->cnt.kernel_launches++;
                for (size_t j = 0; j < nT; ++j) if (pair[j] >= 0) { lvl[j] = -1; lvl[pair[j]] = -1; }
                SK_CUDA(c, cudaMemcpyAsync(d_lvl, lvl.data(), nT * 4, cudaMemcpyHostToDevice, c->stream));
                // T rows of later layers, then both halves of M_tab (every push reaches the measurement end)
                launch_push(c, W, int(nT), m.rows, m.sgn, int(m.Wp), W, T0, int(nT), (const int*)d_lvl, (const u64*)d_push,
                            (const uint8_t*)d_psign, (const int*)d_plevel, np, c->d_err, (unsigned long long*)nullptr);
                launch_push(c, W, int(n), m.rows, m.sgn, int(m.Wp), W, 0, int(n), (const int*)nullptr, (const u64*)d_push,
                            (const uint8_t*)d_psign, (const int*)nullptr, np, c->d_err, (unsigned long long*)nullptr);
                launch_push(c, W, int(n), m.rows, m.sgn, int(m.Wp), W, NS, int(n), (const int*)nullptr, (const u64*)d_push,
                            (const uint8_t*)d_psign, (const int*)nullptr, np, c->d_err, (unsigned long long*)nullptr);
                SK_CUDA(c, cudaGetLastError());
                SK_CUDA(c, cudaStreamSynchronize(c->stream));       // host vectors die at scope end
            } else {
                for (size_t j = 0; j < nT; ++j) if (pair[j] >= 0) { lvl[j] = -1; lvl[pair[j]] = -1; }
            }
        }
    }
    rc = check_ws(c);
    if (rc) return rc;
    // ---- read back: T rows (host cache), M_tab
    {
        const size_t words = nT * (size_t)W;
        p->tx.assign(words, 0); p->tz.assign(words, 0); p->ts.assign(nT, 0);
        p->mx.assign(2 * n * W, 0); p->mz.assign(2 * n * W, 0); p->ms.assign(2 * n, 0);
        const size_t total_rows = 2 * n + nT, tw = total_rows * W;
        rc = sk_ctx_reserve_tmp(c, tw * 16 + total_rows + 64);
        if (rc) return rc;
        u64* dx = (u64*)c->d_tmp; u64* dz = dx + tw; uint8_t* ds = (uint8_t*)(dz + tw);
        // M_tab with the tableau split mapping, then the T rows with a flat mapping shifted by T0
        k_unpack_rows<<<(unsigned)((2 * n * W + 255) / 256), 256, 0, c->stream>>>(m.rows, dx, dz, int(2 * n), W, m.Wp, int(n), NS);
        k_signs_to_bytes<<<(unsigned)((2 * n + 255) / 256), 256, 0, c->stream>>>(m.sgn, ds, int(2 * n), int(n), NS);
        if (nT) {
            k_unpack_rows<<<(unsigned)((words + 255) / 256), 256, 0, c->stream>>>(rowsT, dx + 2 * n * W, dz + 2 * n * W, int(nT), W, m.Wp, int(nT), 0);
            k_signs_to_bytes<<<(unsigned)((nT + 255) / 256), 256, 0, c->stream>>>(m.sgn, ds + 2 * n, int(nT), 0, T0);
        }
        c->cnt.kernel_launches += 4;
        SK_CUDA(c, cudaGetLastError());
        SK_CUDA(c, cudaMemcpyAsync(p->mx.data(), dx, 2 * n * W * 8, cudaMemcpyDeviceToHost, c->stream));
        SK_CUDA(c, cudaMemcpyAsync(p->mz.data(), dz, 2 * n * W * 8, cudaMemcpyDeviceToHost, c->stream));
        SK_CUDA(c, cudaMemcpyAsync(p->ms.data(), ds, 2 * n, cudaMemcpyDeviceToHost, c->stream));
        if (nT) {
            SK_CUDA(c, cudaMemcpyAsync(p->tx.data(), dx + 2 * n * W, words * 8, cudaMemcpyDeviceToHost, c->stream));
            SK_CUDA(c, cudaMemcpyAsync(p->tz.data(), dz + 2 * n * W, words * 8, cudaMemcpyDeviceToHost, c->stream));
            SK_CUDA(c, cudaMemcpyAsync(p->ts.data(), ds + 2 * n, nT, cudaMemcpyDeviceToHost, c->stream));
        }
        SK_CUDA(c, cudaStreamSynchronize(c->stream));
    }
    // ---- layers in forward order; empty layers dropped; safety re-separation
    int maxl = -1;
    for (size_t k = 0; k < nT; ++k) maxl = std::max(maxl, lvl[k]);
    std::vector<std::vector<uint32_t>> layers(maxl + 1);
    for (size_t k = 0; k < nT; ++k) if (lvl[k] >= 0) layers[lvl[k]].push_back(uint32_t(k));
    for (auto& L : layers) {
        if (L.empty()) continue;
        // intra-layer commutation check on the device: group ids = 0 for members, unique for the rest
        std::vector<uint32_t> gid(nT);
        for (size_t k = 0; k < nT; ++k) gid[k] = 0x40000000u + uint32_t(k);
        for (uint32_t k : L) gid[k] = 0;
        rc = sk_ctx_reserve_tmp(c, nT * 4 + 64);
        if (rc) return rc;
        unsigned long long* d_n = (unsigned long long*)c->d_tmp; u32* d_g = (u32*)(d_n + 1);
        SK_CUDA(c, cudaMemsetAsync(d_n, 0, 8, c->stream));
        SK_CUDA(c, cudaMemcpyAsync(d_g, gid.data(), nT * 4, cudaMemcpyHostToDevice, c->stream));
        k_verify_grouping<<<(unsigned)((nT + 255) / 256), 256, 0, c->stream>>>(rowsT, m.Wp, W, int(nT), d_g, 0, d_n);
        c->cnt.kernel_launches++;
        unsigned long long bad = 0;
        SK_CUDA(c, cudaMemcpyAsync(&bad, d_n, 8, cudaMemcpyDeviceToHost, c->stream));
        SK_CUDA(c, cudaStreamSynchronize(c->stream));
        if (bad == 0) { p->layers.push_back(L); continue; }
        // re-separate this layer's rows (in order) with the same first-fit kernels
        sk_rows* sub = nullptr;
        rc = sk_rows_create(c, n, L.size(), &sub);
        if (rc) return rc;
        std::vector<u64> sx(L.size() * W), sz(L.size() * W); std::vector<uint8_t> ss(L.size());
        for (size_t k = 0; k < L.size(); ++k) {
            std::copy(&p->tx[(size_t)L[k] * W], &p->tx[(size_t)L[k] * W] + W, &sx[k * W]);
            std::copy(&p->tz[(size_t)L[k] * W], &p->tz[(size_t)L[k] * W] + W, &sz[k * W]);
            ss[k] = p->ts[L[k]];
        }
        std::vector<uint32_t> sub_of(L.size()); uint64_t nsub = 0;
        rc = sk_rows_upload(sub, reinterpret_cast<const uint64_t*>(sx.data()), reinterpret_cast<const uint64_t*>(sz.data()), ss.data(), L.size());
        if (!rc) rc = rows_need_r(sub);
        if (!rc) {
            u32* d_sub = nullptr;
            if (cudaMalloc(&d_sub, L.size() * 4) != cudaSuccess) { c->err = "cudaMalloc failed in the safety re-separation"; rc = SK_ECUDA; }
            else {
                rc = device_first_fit(c, sub->m.rows, sub->m.Wp, sub->m.W, int(L.size()), fit_mode, d_sub, &nsub);
                if (!rc && cudaMemcpy(sub_of.data(), d_sub, L.size() * 4, cudaMemcpyDeviceToHost) != cudaSuccess) { c->err = "copy failed in the safety re-separation"; rc = SK_ECUDA; }
                cudaFree(d_sub);
            }
        }
        sk_rows_destroy(sub);
        if (rc) return rc;
        std::vector<std::vector<uint32_t>> parts(nsub);
        for (size_t k = 0; k < L.size(); ++k) parts[sub_of[k]].push_back(L[k]);
        for (auto& q : parts) p->layers.push_back(q);
    }
    uint64_t rows_left = 0, weight = 0;
    for (auto& L : p->layers) for (uint32_t k : L) {
        ++rows_left;
        for (int w = 0; w < W; ++w) weight += __builtin_popcountll(p->tx[(size_t)k * W + w] | p->tz[(size_t)k * W + w]);
    }
    p->stats[1] = rows_left; p->stats[2] = weight; p->stats[3] = p->layers.size(); p->stats[4] = nT ? passes : 1;
    *out = p_owner.release();
    return SK_OK;
}
