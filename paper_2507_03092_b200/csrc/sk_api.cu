// sk_api.cu -- C ABI (include/stabkit_b200.h): context, tableau, engine.
// Host orchestration only; all arithmetic is in the kernels_*.cuh files.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <thread>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <new>

#include "kernels_layer.cuh"
#include "kernels_measure.cuh"
#include "kernels_rows.cuh"
#include "kernels_transpose.cuh"
#include "sk_internal.hpp"

using namespace skd;

// ------------------------------------------------------------------ context --
extern "C" const char* sk_version(void) { return "stabkit-b200 0.1 (sm_100a)"; }

extern "C" int32_t sk_ctx_create(int device, void* stream, sk_ctx** out) {
    if (!out) return SK_EARG;
    *out = nullptr;
    static thread_local std::string s_err;
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count <= 0 || device < 0 || device >= count) {
        fprintf(stderr, "stabkit_b200: no usable CUDA device %d (%s); there is no CPU fallback\n", device,
                e != cudaSuccess ? cudaGetErrorString(e) : "device ordinal out of range");
        return SK_ECUDA;
    }
    sk_ctx* c = new (std::nothrow) sk_ctx();
    if (!c) return SK_ECUDA;
    c->device = device;
    if (cudaSetDevice(device) != cudaSuccess) { delete c; return SK_ECUDA; }
    cudaDeviceProp prop{};
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) { delete c; return SK_ECUDA; }
    c->num_sms = prop.multiProcessorCount;
    if (getenv("SK_DEBUG_PROF")) c->prof = 1;
    if (const char* e = getenv("SK_NO_GRAPH")) c->no_graph = atoi(e);
    if (const char* e = getenv("SK_NO_FOLD")) c->no_fold = atoi(e);
    if (const char* e = getenv("SK_ROW_CAP")) c->row_cap = atoi(e);
    if (const char* e = getenv("SK_PANEL_COLUMNS")) c->force_columns = atoi(e);
    if (const char* e = getenv("SK_PANEL_SEQ")) c->seq_rows = atoi(e);
    if (const char* e = getenv("SK_PDL")) c->pdl = atoi(e);
    if (const char* e = getenv("SK_WAVE_KERNEL")) c->no_wave_kernel = atoi(e) == 0;
    if (const char* e = getenv("SK_PIPELINE")) c->no_pipe = atoi(e) == 0;
    if (const char* e = getenv("SK_FUSE_H")) c->no_fuse_h = atoi(e) == 0;
    if (const char* e = getenv("SK_TRANSPOSE_REGS")) c->no_tr_regs = atoi(e) == 0;
    if (const char* e = getenv("SK_PANEL_REPL")) c->no_repl = atoi(e) == 0;
    if (const char* e = getenv("SK_MEAS_GRID")) c->meas_grid_override = atoi(e);
    c->max_smem_optin = int(prop.sharedMemPerBlockOptin);
    if (stream) { c->stream = (cudaStream_t)stream; c->own_stream = false; }
    else {
        if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) { delete c; return SK_ECUDA; }
        c->own_stream = true;
    }
    if (cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) != cudaSuccess) c->no_pipe = 1;
    if (cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking) != cudaSuccess) c->copy = nullptr;
    for (cudaEvent_t* e : {&c->ev_fork, &c->ev_cols, &c->ev_rows, &c->ev_side})
        if (cudaEventCreateWithFlags(e, cudaEventDisableTiming) != cudaSuccess) c->no_pipe = 1;
    cudaGetLastError();
    {
        cudaMemPool_t pool = nullptr;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) { uint64_t keep = ~0ull; cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep); }
    }
    if (cudaMalloc(&c->d_err, 256) != cudaSuccess) { delete c; return SK_ECUDA; }
    cudaMemsetAsync(c->d_err, 0, 256, c->stream);
    if (cudaMalloc(&c->d_ws, sizeof(MeasWs)) != cudaSuccess) { cudaFree(c->d_err); delete c; return SK_ECUDA; }
    cudaMemsetAsync(c->d_ws, 0, sizeof(MeasWs), c->stream);
    *out = c;
    return SK_OK;
}

extern "C" void sk_ctx_destroy(sk_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    if (c->side) { cudaStreamSynchronize(c->side); cudaStreamDestroy(c->side); }
    if (c->copy) { cudaStreamSynchronize(c->copy); cudaStreamDestroy(c->copy); }
    for (cudaEvent_t e : {c->ev_fork, c->ev_cols, c->ev_rows, c->ev_side}) if (e) cudaEventDestroy(e);
    cudaFree(c->d_gates); cudaFree(c->d_tmp); cudaFree(c->d_err); cudaFree(c->d_ws);
    if (c->h_pin) cudaFreeHost(c->h_pin);
    if (c->own_stream) cudaStreamDestroy(c->stream);
    delete c;
}
extern "C" const char* sk_last_error(const sk_ctx* c) { return c ? c->err.c_str() : "null context"; }
extern "C" void* sk_ctx_stream(const sk_ctx* c) { return c ? (void*)c->stream : nullptr; }
extern "C" int32_t sk_ctx_sync(sk_ctx* c) {
    if (!c) return SK_EARG;
    SK_CUDA(c, cudaStreamSynchronize(c->stream));
    return SK_OK;
}

int32_t sk_ctx_reserve_gates(sk_ctx* c, size_t bytes) {
    if (bytes <= c->d_gates_cap) return SK_OK;
    SK_CUDA(c, cudaStreamSynchronize(c->stream));
    cudaFree(c->d_gates); c->d_gates = nullptr; c->d_gates_cap = 0;
    size_t cap = std::max<size_t>(bytes * 2, 1 << 16);
    SK_CUDA(c, cudaMalloc(&c->d_gates, cap));
    c->d_gates_cap = cap;
    return SK_OK;
}
int32_t sk_ctx_reserve_tmp(sk_ctx* c, size_t bytes) {
    if (bytes <= c->d_tmp_cap) return SK_OK;
    SK_CUDA(c, cudaStreamSynchronize(c->stream));
    cudaFree(c->d_tmp); c->d_tmp = nullptr; c->d_tmp_cap = 0;
    size_t cap = std::max<size_t>(bytes * 2, 1 << 16);
    SK_CUDA(c, cudaMalloc(&c->d_tmp, cap));
    c->d_tmp_cap = cap;
    return SK_OK;
}

// Stream-ordered allocations from the device's default memory pool (kept resident: release threshold = max), so that
// creating / destroying tableaux and programs inside sk_sim costs microseconds after the first call.
template <class T> static cudaError_t dmalloc(sk_ctx* c, T** p, size_t bytes) { return cudaMallocAsync((void**)p, bytes ? bytes : 16, c->stream); }
static void dfree(sk_ctx* c, void* p) { if (p) cudaFreeAsync(p, c->stream); }

// ------------------------------------------------------------------ tableau --
struct sk_tableau {
    sk_ctx* ctx = nullptr;
    uint64_t n = 0;
    int W = 0, Wp = 0, RW = 0, NS = 0;
    DMat m;
    bool r_valid = false;           // C form is always valid; R form on demand
    bool r_destab_stale = false;    // R holds the stabilizer rows only (C -> R was restricted to that half)
    size_t cols_bytes = 0, rows_bytes = 0, sgn_bytes = 0;
    u32* d_q = nullptr; uint8_t* d_out = nullptr; uint8_t* d_det = nullptr; size_t rec_cap = 0;
    int meas_grid = 0; size_t meas_smem = 0; bool lv_ok = false;
    u32* d_wpiv = nullptr; u32* d_wl = nullptr; u64* d_wsgn = nullptr;
    // panel-mode scratch (kernels_measure.cuh)
    uint64_t uid = 0;               // distinguishes tableaux that reuse a host address (graph cache key)
    int B = 0; u64* d_pan = nullptr; u64* d_pivbuf = nullptr; u64* d_detacc = nullptr; PanelInfo* d_info = nullptr;
    u32* d_tlist = nullptr; u64* d_tM = nullptr; u64* d_rowM = nullptr; u64* d_tbits = nullptr; u32 tcap = 0; u32* d_alist_h = nullptr; u64* d_alist_b = nullptr; u32* d_dpart = nullptr;
};

// the main stream waits for what is still running on the side stream (k_wave_rows of the last measurement block): called
// before anything that writes the row form or reuses the wave buffers, and before control goes back to the caller
static void join_side(sk_ctx* c) {
    if (!c->side_pending) return;
    cudaStreamWaitEvent(c->stream, c->ev_side, 0);
    c->side_pending = false;
}
// x and z halves in one launch (grid.z = 2); `flag` != nullptr makes the launch conditional on *flag
static int32_t launch_transpose(sk_ctx* c, const u32* src, size_t sstride, int srows, int swords,
                                u32* dst, size_t dstride, int drows, int dwords,
                                size_t src_zoff, size_t dst_zoff, const u32* flag, bool pdl = true) {
    // register-block kernel when every row start and width is 16-byte aligned (true for tableaux with an even word count)
    // and the matrix is large enough for its 512 x 512-bit tiles to fill the machine
    const bool regs = !c->no_tr_regs && (size_t)((srows + kTrRows - 1) / kTrRows) * ((swords + kTrWords - 1) / kTrWords) * 2 >= (size_t)c->num_sms && ((sstride | dstride | src_zoff | dst_zoff | (size_t)swords | (size_t)dwords) & 3) == 0 &&
                      ((reinterpret_cast<size_t>(src) | reinterpret_cast<size_t>(dst)) & 15) == 0;
    dim3 grid = regs ? dim3((srows + kTrRows - 1) / kTrRows, (swords + kTrWords - 1) / kTrWords, 2) : dim3((srows + 255) / 256, (swords + 7) / 8, 2);
    auto* kern = regs ? k_transpose_regs : k_transpose_bits;
    if (c->pdl && pdl) {
        cudaLaunchConfig_t cfg = {}; cfg.gridDim = grid; cfg.blockDim = dim3(256); cfg.stream = c->stream;
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        SK_CUDA(c, cudaLaunchKernelEx(&cfg, kern, src, sstride, srows, swords, dst, dstride, drows, dwords, src_zoff, dst_zoff, flag));
    } else
    kern<<<grid, 256, 0, c->stream>>>(src, sstride, srows, swords, dst, dstride, drows, dwords, src_zoff, dst_zoff, flag);
    c->cnt.kernel_launches++;
    SK_CUDA(c, cudaGetLastError());
    return SK_OK;
}
// C -> R ; stab_only: just the stabilizer rows (all an all-deterministic measurement block reads; the measurement kernel
// derives the destabilizer rows itself if it has to enter panel mode)
static int32_t rows_from_cols(sk_tableau* t, bool stab_only = false, bool pdl = true) {
    sk_ctx* c = t->ctx;
    int32_t rc = launch_transpose(c, reinterpret_cast<const u32*>(t->m.cols), (size_t)4 * t->RW, int(t->n), stab_only ? t->RW : 2 * t->RW,
                                  reinterpret_cast<u32*>(t->m.rows), (size_t)4 * t->Wp, stab_only ? t->NS : 64 * t->RW, 2 * t->Wp,
                                  (size_t)2 * t->RW, (size_t)2 * t->Wp, nullptr, pdl);
    if (rc) return rc;
    c->cnt.transposes++;
    t->r_valid = true; t->r_destab_stale = stab_only;
    return SK_OK;
}
static int32_t rows_full(sk_tableau* t) { return (!t->r_valid || t->r_destab_stale) ? rows_from_cols(t, false) : SK_OK; }
// R -> C ; with `flag` only if the device-side stale flag is raised
static int32_t cols_from_rows(sk_tableau* t, const u32* flag = nullptr) {
    sk_ctx* c = t->ctx;
    int32_t rc = launch_transpose(c, reinterpret_cast<const u32*>(t->m.rows), (size_t)4 * t->Wp, 64 * t->RW, 2 * t->Wp,
                                  reinterpret_cast<u32*>(t->m.cols), (size_t)4 * t->RW, int(t->n), 2 * t->RW,
                                  (size_t)2 * t->Wp, (size_t)2 * t->RW, flag);
    if (rc) return rc;
    if (!flag) c->cnt.transposes++;
    return SK_OK;
}

static int32_t tableau_identity(sk_tableau* t) {
    sk_ctx* c = t->ctx;
    SK_CUDA(c, cudaMemsetAsync(t->m.cols, 0, t->cols_bytes, c->stream));
    SK_CUDA(c, cudaMemsetAsync(t->m.rows, 0, t->rows_bytes, c->stream));
    SK_CUDA(c, cudaMemsetAsync(t->m.sgn, 0, t->sgn_bytes, c->stream));
    SK_CUDA(c, cudaMemsetAsync(t->d_rowM, 0, (size_t)2 * 64 * t->RW * 8, c->stream));
    SK_CUDA(c, cudaMemsetAsync(t->d_tbits, 0, (size_t)t->RW * 8, c->stream));
    k_identity<<<(unsigned)((t->n + 255) / 256), 256, 0, c->stream>>>(t->m.cols, t->m.rows, int(t->n), t->RW, t->Wp, t->NS);
    c->cnt.kernel_launches++;
    SK_CUDA(c, cudaGetLastError());
    t->r_valid = true; t->r_destab_stale = false;
    return SK_OK;
}

extern "C" int32_t sk_tableau_create(sk_ctx* c, uint64_t n, sk_tableau** out) {
    if (!c || !out) return SK_EARG;
    *out = nullptr;
    if (n == 0) SK_FAIL(c, SK_EDIM, "new_identity: n must be >= 1 (SPEC:129)");
    if (n > (1u << 20)) SK_FAIL(c, SK_EDIM, "n=%llu exceeds the supported 2^20 qubits", (unsigned long long)n);
    SK_CUDA(c, cudaSetDevice(c->device));
    sk_tableau* t = new sk_tableau();
    t->ctx = c; t->n = n; t->uid = ++c->tableau_uid;
    t->W = int((n + 63) / 64); t->Wp = (t->W + 1) & ~1; t->RW = 2 * t->W; t->NS = 64 * t->W;
    t->m.n = n; t->m.W = t->W; t->m.Wp = t->Wp; t->m.RW = t->RW;
    t->cols_bytes = (size_t)n * 2 * t->RW * 8;
    t->rows_bytes = (size_t)64 * t->RW * 2 * t->Wp * 8;
    t->sgn_bytes = (size_t)t->RW * 8;
    {
        // dynamic shared memory of k_measure_block: per-warp accumulators + pivot-value scratch, or the panel
        cudaFuncAttributes fa{};
        SK_CUDA(c, cudaFuncGetAttributes(&fa, k_measure_block));
        const size_t avail = (size_t)c->max_smem_optin - fa.sharedSizeBytes - 1024;
        // the attribute belongs to the function (per device), not to a context: always opt in to the device maximum
        SK_CUDA(c, cudaFuncSetAttribute(k_measure_block, cudaFuncAttributeMaxDynamicSharedMemorySize, int(c->max_smem_optin - fa.sharedSizeBytes)));
        const size_t acc_words = (size_t)kMeasWarps * 2 * t->Wp;
        const size_t col_words = (size_t)t->RW + 2;             // + virtual-row word + pad
        const size_t aux_words = 2 * ((size_t)t->RW + 1);       // nzm | retired
        if ((acc_words + 2) * 8 > avail || (col_words + aux_words) * 8 > avail) {
            delete t;
            SK_FAIL(c, SK_EDIM, "n=%llu needs more shared memory per CTA than the %zu B available", (unsigned long long)n, avail);
        }
        int B = int(std::min<size_t>(kPanelMax, (avail / 8 - aux_words) / col_words));
        if (const char* e = getenv("SK_PANEL")) B = std::max(1, std::min(B, atoi(e)));
        t->meas_grid = c->meas_grid_override > 0 ? std::min(c->meas_grid_override, c->num_sms) : c->num_sms;
        const int ncons = std::max(1, t->meas_grid - 1);         // consumer CTAs of the pivot-value phase
        const int wpc = (t->W + ncons - 1) / ncons;
        while (B > 1 && (acc_words + (size_t)B * 2 * wpc) * 8 > avail) --B;
        t->B = B;
        t->meas_smem = std::max<size_t>(std::max(acc_words + (size_t)B * 2 * wpc, (size_t)B * col_words + aux_words) * 8, std::max<size_t>(2 * 512 * 9 * 4, level_smem_bytes(t->NS)));   // >= the in-kernel transpose tiles
        const size_t lvb = lv_smem_bytes(t->NS, t->W, t->Wp, t->meas_grid, B);
        t->lv_ok = lv_supported(t->W) && lvb <= avail;
        if (t->lv_ok) t->meas_smem = std::max(t->meas_smem, lvb);
    }
    cudaError_t e1 = dmalloc(c, &t->m.cols, t->cols_bytes);
    cudaError_t e2 = dmalloc(c, &t->m.rows, t->rows_bytes);
    cudaError_t e3 = dmalloc(c, &t->m.sgn, t->sgn_bytes);
    const size_t window = (size_t)c->num_sms * kMeasWarps * kSlotsPerWarp;
    cudaError_t e4 = dmalloc(c, &t->d_wpiv, 2 * window * 4);
    if (!e4) e4 = dmalloc(c, &t->d_wl, 2 * window * kWarpList * 4);
    if (!e4) e4 = dmalloc(c, &t->d_wsgn, (size_t)t->W * 8);
    cudaError_t e5 = dmalloc(c, &t->d_pan, (size_t)t->B * t->RW * 8);
    cudaError_t e6 = dmalloc(c, &t->d_pivbuf, (size_t)t->B * 2 * t->Wp * 8);
    cudaError_t e7 = dmalloc(c, &t->d_detacc, (size_t)4 * t->B * 2 * t->Wp * 8);       // x4: a deterministic step's partner product may come in four parts (kernels_panel.cuh D1)
    cudaError_t e8 = dmalloc(c, &t->d_info, sizeof(PanelInfo));
    t->tcap = u32(64 * t->RW + 2 * kPanelMax);
    cudaError_t e9 = dmalloc(c, &t->d_tlist, (size_t)2 * t->tcap * 4);
    cudaError_t e10 = dmalloc(c, &t->d_tM, (size_t)2 * t->tcap * 8);
    cudaError_t e11 = dmalloc(c, &t->d_rowM, (size_t)2 * 64 * t->RW * 8);
    if (!e11) e11 = dmalloc(c, &t->d_tbits, (size_t)t->RW * 8);
    cudaError_t e12 = dmalloc(c, &t->d_alist_h, (size_t)64 * t->RW * 4);
    cudaError_t e13 = dmalloc(c, &t->d_alist_b, (size_t)2 * 64 * t->RW * 8);      // two pair-list buffers (kernels_panel.cuh)
    cudaError_t e14 = dmalloc(c, &t->d_dpart, (size_t)kPanelMax * kRowSlots * 4);
    if (!e8) e8 = cudaMemsetAsync(t->d_info, 0, sizeof(PanelInfo), c->stream);
    if (e1 || e2 || e3 || e4 || e5 || e6 || e7 || e8 || e9 || e10 || e11 || e12 || e13 || e14) { sk_tableau_destroy(t); SK_FAIL(c, SK_ECUDA, "cudaMalloc failed for a %llu-qubit tableau", (unsigned long long)n); }

    int per_sm = 0;
    SK_CUDA(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_measure_block, kMeasThreads, t->meas_smem));
    if (per_sm < 1) { sk_tableau_destroy(t); SK_FAIL(c, SK_ECUDA, "measurement kernel does not fit on an SM"); }
    int32_t rc = tableau_identity(t);
    if (rc) { sk_tableau_destroy(t); return rc; }
    *out = t;
    return SK_OK;
}

extern "C" void sk_tableau_destroy(sk_tableau* t) {
    if (!t) return;
    sk_ctx* c = t->ctx;
    cudaSetDevice(c->device);
    for (void* p : {(void*)t->m.cols, (void*)t->m.rows, (void*)t->m.sgn, (void*)t->d_wpiv, (void*)t->d_wl, (void*)t->d_wsgn, (void*)t->d_pan, (void*)t->d_pivbuf, (void*)t->d_detacc,
                    (void*)t->d_info, (void*)t->d_tlist, (void*)t->d_tM, (void*)t->d_rowM, (void*)t->d_tbits, (void*)t->d_alist_h, (void*)t->d_alist_b, (void*)t->d_dpart,
                    (void*)t->d_q, (void*)t->d_out, (void*)t->d_det})
        dfree(c, p);          // stream-ordered: queued behind the work that still uses the buffers
    delete t;
}
extern "C" int32_t sk_tableau_reset(sk_tableau* t) { return t ? tableau_identity(t) : SK_EARG; }
extern "C" uint64_t sk_tableau_qubits(const sk_tableau* t) { return t ? t->n : 0; }

extern "C" int32_t sk_tableau_upload(sk_tableau* t, const uint64_t* x, const uint64_t* z, const uint8_t* sign) {
    if (!t || !x || !z || !sign) return SK_EARG;
    sk_ctx* c = t->ctx;
    const size_t nrows = 2 * t->n, words = nrows * t->W;
    int32_t rc = sk_ctx_reserve_tmp(c, words * 16 + nrows + 64);
    if (rc) return rc;
    u64* dx = (u64*)c->d_tmp; u64* dz = dx + words; uint8_t* ds = (uint8_t*)(dz + words);
    SK_CUDA(c, cudaMemcpyAsync(dx, x, words * 8, cudaMemcpyHostToDevice, c->stream));
    SK_CUDA(c, cudaMemcpyAsync(dz, z, words * 8, cudaMemcpyHostToDevice, c->stream));
    SK_CUDA(c, cudaMemcpyAsync(ds, sign, nrows, cudaMemcpyHostToDevice, c->stream));
    SK_CUDA(c, cudaMemsetAsync(t->m.rows, 0, t->rows_bytes, c->stream));
    SK_CUDA(c, cudaMemsetAsync(t->m.sgn, 0, t->sgn_bytes, c->stream));
    k_pack_rows<<<(unsigned)((words + 255) / 256), 256, 0, c->stream>>>(dx, dz, t->m.rows, int(nrows), t->W, t->Wp, int(t->n), t->NS);
    k_bytes_to_signs<<<(unsigned)((nrows + 255) / 256), 256, 0, c->stream>>>(ds, t->m.sgn, int(nrows), int(t->n), t->NS);
    c->cnt.kernel_launches += 2;
    SK_CUDA(c, cudaGetLastError());
    t->r_valid = true; t->r_destab_stale = false;
    rc = cols_from_rows(t);
    if (rc) return rc;
    SK_CUDA(c, cudaStreamSynchronize(c->stream));
    return SK_OK;
}

extern "C" int32_t sk_tableau_audit(sk_tableau* t, uint64_t* violations) {
    if (!t || !violations) return SK_EARG;
    sk_ctx* c = t->ctx;
    { int32_t rc0 = rows_full(t); if (rc0) return rc0; }
    unsigned long long* d_v = reinterpret_cast<unsigned long long*>(c->d_err) + 2;
    SK_CUDA(c, cudaMemsetAsync(d_v, 0, 8, c->stream));
    const int rowbits = 2 * t->NS, words = (rowbits + 63) / 64;
    const int step = 4096;                       // row-bits per launch: keeps the grid below 2^31 threads
    for (int a0 = 0; a0 < rowbits; a0 += step) {
        const int na = std::min(step, rowbits - a0);
        const size_t threads = (size_t)na * words * 32;
        k_audit_tile<<<(unsigned)((threads + 255) / 256), 256, 0, c->stream>>>(t->m.rows, t->Wp, t->W, t->NS, int(t->n), a0, na, d_v);
        c->cnt.kernel_launches++;
    }
    SK_CUDA(c, cudaGetLastError());
    unsigned long long v = 0;
    SK_CUDA(c, cudaMemcpyAsync(&v, d_v, 8, cudaMemcpyDeviceToHost, c->stream));
    SK_CUDA(c, cudaStreamSynchronize(c->stream));
    *violations = v;
    return SK_OK;
}

static int32_t check_ws(sk_ctx* c) {
    MeasWs* ws = (MeasWs*)c->d_ws;
    MeasWs h;
    SK_CUDA(c, cudaMemcpyAsync(&h, ws, sizeof h, cudaMemcpyDeviceToHost, c->stream));
    u32 e2 = 0;
    SK_CUDA(c, cudaMemcpyAsync(&e2, c->d_err, 4, cudaMemcpyDeviceToHost, c->stream));
    SK_CUDA(c, cudaStreamSynchronize(c->stream));
    if ((h.err & 0xC0000000u)) {
        cudaMemsetAsync(ws, 0, 32, c->stream); cudaMemsetAsync(&ws->err, 0, 4, c->stream);      // an aborted launch leaves its words behind
        SK_FAIL(c, SK_ECUDA, "measurement kernel timed out (err=0x%x)", h.err);
    }
    if ((h.err & 1u) || (e2 & 1u)) {
        cudaMemsetAsync(&ws->err, 0, 4, c->stream); cudaMemsetAsync(c->d_err, 0, 4, c->stream);
        SK_FAIL(c, SK_EINVARIANT, "rowsum produced an odd mod-4 phase (SPEC:169)");
    }
    return SK_OK;
}

extern "C" int32_t sk_tableau_download(sk_tableau* t, uint64_t* x, uint64_t* z, uint8_t* sign) {
    if (!t || !x || !z || !sign) return SK_EARG;
    sk_ctx* c = t->ctx;
    { int32_t rc0 = rows_full(t); if (rc0) return rc0; }
    const size_t nrows = 2 * t->n, words = nrows * t->W;
    int32_t rc = sk_ctx_reserve_tmp(c, words * 16 + nrows + 64);
    if (rc) return rc;
    u64* dx = (u64*)c->d_tmp; u64* dz = dx + words; uint8_t* ds = (uint8_t*)(dz + words);
    k_unpack_rows<<<(unsigned)((words + 255) / 256), 256, 0, c->stream>>>(t->m.rows, dx, dz, int(nrows), t->W, t->Wp, int(t->n), t->NS);
    k_signs_to_bytes<<<(unsigned)((nrows + 255) / 256), 256, 0, c->stream>>>(t->m.sgn, ds, int(nrows), int(t->n), t->NS);
    c->cnt.kernel_launches += 2;
    SK_CUDA(c, cudaGetLastError());
    SK_CUDA(c, cudaMemcpyAsync(x, dx, words * 8, cudaMemcpyDeviceToHost, c->stream));
    SK_CUDA(c, cudaMemcpyAsync(z, dz, words * 8, cudaMemcpyDeviceToHost, c->stream));
    SK_CUDA(c, cudaMemcpyAsync(sign, ds, nrows, cudaMemcpyDeviceToHost, c->stream));
    return check_ws(c);
}

// ------------------------------------------------------------- gate layers --
static int32_t validate_gate(sk_ctx* c, const sk_gate& g, uint64_t n, size_t idx) {
    if (g.kind > SK_TDG) SK_FAIL(c, SK_EARG, "gate %zu: unknown kind %u", idx, g.kind);
    if (g.q0 >= n) SK_FAIL(c, SK_EDIM, "gate %zu: qubit %u out of range for %llu qubits", idx, g.q0, (unsigned long long)n);
    if (sk_is_two_qubit(g.kind)) {
        if (g.q1 >= n) SK_FAIL(c, SK_EDIM, "gate %zu: qubit %u out of range for %llu qubits", idx, g.q1, (unsigned long long)n);
        if (g.q0 == g.q1) SK_FAIL(c, SK_EARG, "gate %zu: two-qubit gate on identical qubits %u (SPEC:159)", idx, g.q0);
    }
    return SK_OK;
}

static int layer_threads(const sk_tableau* t) { return std::min(256, std::max(32, (t->RW / 2 + 31) & ~31)); }
static int layer_target_ctas(const sk_ctx* c, int threads) { return c->num_sms * std::max(1, 1536 / threads); }
// one launch = one layer, or several merged layers with host-made chunk boundaries (d_boff[0..nblocks], relative to d_gates)
static void launch_layer(sk_tableau* t, const sk_gate* d_gates, int ngates, const u32* d_boff = nullptr, int nblocks = 0, int nlayers = 1) {
    sk_ctx* c = t->ctx;
    const int threads = layer_threads(t);
    int grid = nblocks, gpb = 0;
    if (!d_boff) {
        const int target_ctas = layer_target_ctas(c, threads);
        gpb = std::max(1, (ngates + target_ctas - 1) / target_ctas);
        grid = (ngates + gpb - 1) / gpb;
    }
    if (c->pdl) {       // the launch may be scheduled while the previous layer still runs (griddepcontrol.wait inside the kernel)
        cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(grid); cfg.blockDim = dim3(threads); cfg.stream = c->stream;
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        if (cudaLaunchKernelEx(&cfg, k_layer, t->m.cols, t->m.sgn, d_gates, ngates, t->RW, gpb, d_boff) != cudaSuccess) { c->err = "k_layer launch failed"; }
    } else
    k_layer<<<grid, threads, 0, c->stream>>>(t->m.cols, t->m.sgn, d_gates, ngates, t->RW, gpb, d_boff);
    c->cnt.kernel_launches++; c->cnt.layers += (uint64_t)nlayers;
    c->last_n = t->n;
    t->r_valid = false;
}

extern "C" int32_t sk_apply_layer(sk_tableau* t, const sk_gate* gates, size_t ngates) {
    if (!t || (!gates && ngates)) return SK_EARG;
    sk_ctx* c = t->ctx;
    if (ngates == 0) return SK_OK;
    if (c->q_epoch.size() < t->n) c->q_epoch.assign(t->n, 0);
    if (++c->epoch == 0) { std::fill(c->q_epoch.begin(), c->q_epoch.end(), 0); c->epoch = 1; }
    for (size_t i = 0; i < ngates; ++i) {
        int32_t rc = validate_gate(c, gates[i], t->n, i);
        if (rc) return rc;
        if (gates[i].kind >= SK_M) SK_FAIL(c, SK_EUNSUPPORTED, "gate %zu: M/T/TDG cannot be part of a Clifford layer (SPEC:191)", i);
        uint32_t qs[2] = {gates[i].q0, gates[i].q1};
        for (int k = 0; k < (sk_is_two_qubit(gates[i].kind) ? 2 : 1); ++k) {
            if (c->q_epoch[qs[k]] == c->epoch) SK_FAIL(c, SK_EARG, "gate %zu: qubit %u used twice in one layer (SPEC:263)", i, qs[k]);
            c->q_epoch[qs[k]] = c->epoch;
        }
        c->cnt.gate_hist[gates[i].kind]++;
    }
    int32_t rc = sk_ctx_reserve_gates(c, ngates * sizeof(sk_gate));
    if (rc) return rc;
    SK_CUDA(c, cudaMemcpyAsync(c->d_gates, gates, ngates * sizeof(sk_gate), cudaMemcpyHostToDevice, c->stream));
    launch_layer(t, (const sk_gate*)c->d_gates, int(ngates));
    SK_CUDA(c, cudaGetLastError());
    // the staging buffer is reused by the next call
    SK_CUDA(c, cudaStreamSynchronize(c->stream));
    return SK_OK;
}

void sk_layer_run(const sk_gate* g, size_t ng, uint64_t n, std::vector<uint32_t>& level,
                  std::vector<sk_gate>& out, std::vector<uint32_t>& layer_sizes) {
    if (level.size() < n) level.assign(n, 0);
    std::vector<uint32_t> lay(ng);
    uint32_t depth = 0;
    for (size_t i = 0; i < ng; ++i) {
        uint32_t l = level[g[i].q0];
        if (sk_is_two_qubit(g[i].kind)) l = std::max(l, level[g[i].q1]);
        lay[i] = l;
        level[g[i].q0] = l + 1;
        if (sk_is_two_qubit(g[i].kind)) level[g[i].q1] = l + 1;
        depth = std::max(depth, l + 1);
    }
    for (size_t i = 0; i < ng; ++i) { level[g[i].q0] = 0; if (sk_is_two_qubit(g[i].kind)) level[g[i].q1] = 0; }
    std::vector<uint32_t> start(depth + 1, 0);
    for (size_t i = 0; i < ng; ++i) start[lay[i] + 1]++;
    for (uint32_t d = 0; d < depth; ++d) { layer_sizes.push_back(start[d + 1]); start[d + 1] += start[d]; }
    size_t base = out.size();
    out.resize(base + ng);
    for (size_t i = 0; i < ng; ++i) out[base + start[lay[i]]++] = g[i];
}

extern "C" int32_t sk_apply_gates(sk_tableau* t, const sk_gate* gates, size_t ngates) {
    if (!t || (!gates && ngates)) return SK_EARG;
    sk_ctx* c = t->ctx;
    if (ngates == 0) return SK_OK;
    for (size_t i = 0; i < ngates; ++i) {
        int32_t rc = validate_gate(c, gates[i], t->n, i);
        if (rc) return rc;
        if (gates[i].kind >= SK_M) SK_FAIL(c, SK_EUNSUPPORTED, "gate %zu: M/T/TDG in a Clifford sequence (SPEC:191)", i);
        c->cnt.gate_hist[gates[i].kind]++;
    }
    std::vector<sk_gate> ordered; std::vector<uint32_t> sizes, scratch;
    sk_layer_run(gates, ngates, t->n, scratch, ordered, sizes);
    int32_t rc = sk_ctx_reserve_gates(c, ngates * sizeof(sk_gate));
    if (rc) return rc;
    SK_CUDA(c, cudaMemcpyAsync(c->d_gates, ordered.data(), ngates * sizeof(sk_gate), cudaMemcpyHostToDevice, c->stream));
    size_t off = 0;
    for (uint32_t s : sizes) { launch_layer(t, (const sk_gate*)c->d_gates + off, int(s)); off += s; }
    SK_CUDA(c, cudaGetLastError());
    SK_CUDA(c, cudaStreamSynchronize(c->stream));
    return SK_OK;
}

// ------------------------------------------------------------ measurement --
static int32_t launch_measure(sk_tableau* t, const u32* d_qubits, int count, uint64_t seed, uint64_t ordinal0,
                              uint8_t* d_out, uint8_t* d_det) {
    sk_ctx* c = t->ctx;
    if (count <= 0) return SK_OK;
    c->last_n = t->n;
    const bool joined = c->side_pending;
    join_side(c);          // the previous block's k_wave_rows is done with the row form, the lists and the sign copy
    // the launch-scoped words (barrier counter, progress counter, wave slots) are zero: the previous launch's last CTA
    // re-zeroed them on its way out (check_ws does it after an error)
    MeasWs* ws = (MeasWs*)c->d_ws;
    MeasArgs a;
    a.m = t->m; a.n = int(t->n); a.NS = t->NS; a.qubits = d_qubits; a.count = count;
    a.seed = seed; a.ordinal0 = ordinal0; a.outcomes = d_out; a.dets = d_det; a.ws = ws; a.wpiv = t->d_wpiv; a.wl = t->d_wl; a.wsgn = t->d_wsgn;
    a.B = t->B; a.pan = t->d_pan; a.pivbuf = t->d_pivbuf; a.detacc = t->d_detacc; a.info = t->d_info; a.tlist = t->d_tlist; a.tM = t->d_tM; a.rowM = t->d_rowM; a.tbits = t->d_tbits; a.tcap = t->tcap; a.fold = c->no_fold ? 0 : 1; a.row_cap = c->row_cap > 0 ? std::min(c->row_cap, kRowCap) : kRowCap; a.alist_h = t->d_alist_h; a.alist_b = t->d_alist_b; a.dpart = t->d_dpart;
    a.prof = c->prof; a.force_columns = c->force_columns; a.seq_rows = c->seq_rows; a.lv_enable = (t->lv_ok && !c->no_repl && !c->force_columns && !c->seq_rows) ? 1 : 0;
    a.from_wave = 0;
    const size_t window = (size_t)c->num_sms * kMeasWarps * kSlotsPerWarp;
    const bool wave = !c->no_wave_kernel && count >= 2048;
    // long blocks: the deterministic measurements (all of them in rounds 2..d of a memory experiment) by two ordinary
    // one-warp-per-measurement grids; the cooperative kernel starts at ws->wpos.  When the whole block fits the wave buffers the
    // two run on the side stream: k_wave_cols next to the transposition (both only read the gate form), k_wave_rows after the
    // cooperative kernel was enqueued -- it reads nothing the NEXT gate layers write, so those need not wait for it.
    const int wend = int(std::min<size_t>((size_t)count, 2 * window));
    const bool pipe = wave && !c->no_pipe && count <= wend;
    static int wave_per_sm = 0;
    if (wave && wave_per_sm == 0 && (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&wave_per_sm, k_wave_rows, kWaveThreads, 0) != cudaSuccess || wave_per_sm < 1)) wave_per_sm = 2;
    const int wgrid = std::max(1, std::min((wend + kWaveThreads / 32 - 1) / (kWaveThreads / 32), c->num_sms * std::max(1, wave_per_sm)));
    static const bool no_fuse = getenv("SK_FUSE_COLS") && atoi(getenv("SK_FUSE_COLS")) == 0;      // A/B aid
    if (wave && !t->r_valid && !c->no_tr_regs && (t->W & 1) == 0 && !no_fuse) {
        // transposition of the stabilizer half (register-block tiles: 16-byte aligned rows) + k_wave_cols in one launch
        dim3 grid((unsigned)((t->n + kTrRows - 1) / kTrRows), (unsigned)((t->RW + kTrWords - 1) / kTrWords), 3);
        const u32* src = reinterpret_cast<const u32*>(t->m.cols); u32* dst = reinterpret_cast<u32*>(t->m.rows);
        const size_t ss = (size_t)4 * t->RW, ds = (size_t)4 * t->Wp, sz = (size_t)2 * t->RW, dz = (size_t)2 * t->Wp;
        const int srows = int(t->n), swords = t->RW, drows = t->NS, dwords = 2 * t->Wp, pp = pipe ? 1 : 0;
        if (c->pdl && !joined) {         // (no programmatic launch behind a cross-stream wait)
            cudaLaunchConfig_t cfg = {}; cfg.gridDim = grid; cfg.blockDim = dim3(256); cfg.stream = c->stream;
            cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at; cfg.numAttrs = 1;
            SK_CUDA(c, cudaLaunchKernelEx(&cfg, k_transpose_wave, src, ss, srows, swords, dst, ds, drows, dwords, sz, dz, a, wend, pp));
        } else
        k_transpose_wave<<<grid, 256, 0, c->stream>>>(src, ss, srows, swords, dst, ds, drows, dwords, sz, dz, a, wend, pp);
        c->cnt.kernel_launches++; c->cnt.transposes++;
        t->r_valid = true; t->r_destab_stale = true;
    } else {
        if (wave) { k_wave_cols<<<wgrid, kWaveThreads, 0, c->stream>>>(a, wend, pipe ? 1 : 0); c->cnt.kernel_launches++; }
        if (!t->r_valid) { int32_t rc = rows_from_cols(t, true, !joined); if (rc) return rc; }
    }
    a.destab_stale = t->r_destab_stale ? 1 : 0;
    if (wave) {
        a.from_wave = 1;
        if (pipe) SK_CUDA(c, cudaEventRecord(c->ev_rows, c->stream));
        else { k_wave_rows<<<wgrid, kWaveThreads, 0, c->stream>>>(a, wend); c->cnt.kernel_launches++; }
    }
    // (Measured, round 2: inside a captured graph the cooperative kernel as the body of an IF node whose condition k_wave_cols
    // sets -- so that the deterministic blocks skip the empty 148-CTA launch, 6 us each -- works, bit-exact, and is SLOWER: d=71
    // 8.88 ms against 8.41 ms, graph launch 0.19 ms against 0.02 ms and sk_sim end to end 28 ms against 19 ms for the
    // instantiation.  A conditional node costs more than the launch it saves.  Removed.)
    if (c->prof_mark && wave) (*c->prof_mark)(3);          // profiled run: the wave kernels are a class of their own
    void* args[] = {&a};
    SK_CUDA(c, cudaLaunchCooperativeKernel((void*)k_measure_block, dim3(t->meas_grid), dim3(kMeasThreads), args, t->meas_smem, c->stream));
    c->cnt.kernel_launches++;
    if (pipe) {
        SK_CUDA(c, cudaStreamWaitEvent(c->side, c->ev_rows, 0));
        k_wave_rows<<<wgrid, kWaveThreads, 0, c->side>>>(a, wend);
        c->cnt.kernel_launches++;
        SK_CUDA(c, cudaEventRecord(c->ev_side, c->side));
        c->side_pending = true;
    }
    return SK_OK;          // (a block that entered panel mode re-derives the C form itself before it exits)
}

static int32_t reserve_record(sk_tableau* t, size_t m) {
    sk_ctx* c = t->ctx;
    if (m <= t->rec_cap) return SK_OK;
    dfree(c, t->d_q); dfree(c, t->d_out); dfree(c, t->d_det);
    t->d_q = nullptr; t->d_out = nullptr; t->d_det = nullptr; t->rec_cap = 0;
    size_t cap = std::max<size_t>(m * 2, 1024);
    SK_CUDA(c, dmalloc(c, &t->d_q, cap * 4));
    SK_CUDA(c, dmalloc(c, &t->d_out, cap));
    SK_CUDA(c, dmalloc(c, &t->d_det, cap));
    t->rec_cap = cap;
    return SK_OK;
}

extern "C" int32_t sk_measure_batch(sk_tableau* t, const uint32_t* qubits, size_t m, uint64_t seed,
                                    uint64_t ordinal0, uint8_t* outcomes, uint8_t* deterministic) {
    if (!t || (!qubits && m) || !outcomes || !deterministic) return SK_EARG;
    sk_ctx* c = t->ctx;
    if (m == 0) return SK_OK;
    for (size_t i = 0; i < m; ++i)
        if (qubits[i] >= t->n) SK_FAIL(c, SK_EDIM, "measure: qubit %u out of range for %llu qubits", qubits[i], (unsigned long long)t->n);
    int32_t rc = reserve_record(t, m);
    if (rc) return rc;
    SK_CUDA(c, cudaMemcpyAsync(t->d_q, qubits, m * 4, cudaMemcpyHostToDevice, c->stream));
    rc = launch_measure(t, t->d_q, int(m), seed, ordinal0, t->d_out, t->d_det);
    join_side(c);
    if (rc) return rc;
    c->cnt.gate_hist[SK_M] += m;
    SK_CUDA(c, cudaMemcpyAsync(outcomes, t->d_out, m, cudaMemcpyDeviceToHost, c->stream));
    SK_CUDA(c, cudaMemcpyAsync(deterministic, t->d_det, m, cudaMemcpyDeviceToHost, c->stream));
    return check_ws(c);
}

extern "C" int32_t sk_measure_z(sk_tableau* t, uint32_t q, uint64_t seed, uint64_t ordinal,
                                uint8_t* outcome, uint8_t* deterministic) {
    return sk_measure_batch(t, &q, 1, seed, ordinal, outcome, deterministic);
}

extern "C" int32_t sk_tableau_rowsum(sk_tableau* t, uint64_t h, uint64_t i) {
    if (!t) return SK_EARG;
    sk_ctx* c = t->ctx;
    if (h >= 2 * t->n || i >= 2 * t->n || h == i) SK_FAIL(c, SK_EDIM, "rowsum(%llu,%llu): rows must differ and be < 2n (SPEC:167)", (unsigned long long)h, (unsigned long long)i);
    { int32_t rc = rows_full(t); if (rc) return rc; }
    int hb = h < t->n ? int(h) : t->NS + int(h - t->n);
    int ib = i < t->n ? int(i) : t->NS + int(i - t->n);
    k_rowsum_single<<<1, 256, 0, c->stream>>>(t->m, hb, ib, c->d_err);
    c->cnt.kernel_launches++;
    SK_CUDA(c, cudaGetLastError());
    return check_ws(c);
}

// ---------------------------------------------------------------- counters --
extern "C" int32_t sk_reset_counters(sk_ctx* c) {
    if (!c) return SK_EARG;
    c->cnt = sk_counters{};
    MeasWs* ws = (MeasWs*)c->d_ws;
    SK_CUDA(c, cudaMemsetAsync(&ws->n_rand, 0, (38 + 640 + 192) * 8, c->stream));
    SK_CUDA(c, cudaMemsetAsync(reinterpret_cast<unsigned long long*>(c->d_err) + 1, 0, 8, c->stream));
    return SK_OK;
}
extern "C" int32_t sk_get_counters(sk_ctx* c, sk_counters* out) {
    if (!c || !out) return SK_EARG;
    MeasWs h;
    SK_CUDA(c, cudaMemcpyAsync(&h, c->d_ws, sizeof h, cudaMemcpyDeviceToHost, c->stream));
    SK_CUDA(c, cudaStreamSynchronize(c->stream));
    unsigned long long npred = 0;
    SK_CUDA(c, cudaMemcpyAsync(&npred, reinterpret_cast<unsigned long long*>(c->d_err) + 1, 8, cudaMemcpyDeviceToHost, c->stream));
    SK_CUDA(c, cudaStreamSynchronize(c->stream));
    *out = c->cnt;
    out->n_rand = h.n_rand; out->n_det = h.n_det; out->k_rand = h.k_rand; out->k_det = h.k_det; out->waves = h.waves;
    out->pred_evals = c->cnt.pred_evals + npred;
    {   // columns read or written per gate kind x R/8 bytes, + 2 R/8 per fused layer for the sign column, + the measurement terms
        const double R = 2.0 * double(c->last_n), col = R / 8.0, W = double((c->last_n + 63) / 64);
        static const double kCols[12] = {4, 3, 3, 1, 2, 1, 6, 6, 8, 0, 0, 0};      // H S SDG X Y Z CX CZ SWAP M T TDG
        double b = 0;
        for (int k = 0; k < 12; ++k) b += kCols[k] * double(c->cnt.gate_hist[k]) * col;
        b += 2.0 * col * double(c->cnt.layers);
        b += double(h.n_rand) * (col + 48.0 * W) + double(h.k_rand) * 32.0 * W + double(h.n_det) * col + double(h.k_det) * 16.0 * W;
        out->algorithmic_bytes = b;
    }
    for (int k = 0; k < 4; ++k) out->class_ms[k] = c->class_ms[k];
    for (int k = 0; k < 8; ++k) out->meas_phase_ns[k] = h.prof[k];
    if (getenv("SK_DEBUG_PROF")) fprintf(stderr, "measure kernel CTA0 us: P1 %.0f P2 %.0f | gather %.0f factorise %.0f values+detA %.0f apply+detB %.0f | barriers wave %.0f panel %.0f | panels %llu\n",
                                         h.prof[0] / 1e3, h.prof[1] / 1e3, h.prof[2] / 1e3, h.prof[3] / 1e3, h.prof[4] / 1e3, h.prof[5] / 1e3, h.prof[6] / 1e3, h.prof[7] / 1e3, (unsigned long long)h.panels);
    if (getenv("SK_DEBUG_PROF")) {
        const char* nm[4] = {"G", "F", "V+D1", "A+D2"};
        for (int ph = 0; ph < 4; ++ph) {
            double mx = 0, sum = 0; int arg = 0, cnt = 0;
            for (int b = 0; b < 160; ++b) { double v = h.ctaphase[b * 4 + ph] / 1e3; if (v > 0) { sum += v; ++cnt; } if (v > mx) { mx = v; arg = b; } }
            fprintf(stderr, "panel phase %-5s own time per CTA (us): avg %.0f max %.0f (CTA %d) cta0 %.0f\n", nm[ph], cnt ? sum / cnt : 0.0, mx, arg, h.ctaphase[ph] / 1e3);
            if (getenv("SK_DEBUG_CTAS")) { fprintf(stderr, "   per CTA:"); for (int b = 0; b < 148; ++b) fprintf(stderr, " %.0f", h.ctaphase[b * 4 + ph] / 1e3); fprintf(stderr, "\n"); }
        }
    }
    if (getenv("SK_DEBUG_WAVE")) {
        for (int wsel = 0; wsel < 2; ++wsel) for (int r = 0; r < 3; ++r) {
            const u64* t = h.trace + wsel * 96 + r * 8;
            fprintf(stderr, "wave trace warp %s slot %d: start %.2f us after the first, column %.2f, product %.2f, signs+sum %.2f\n", wsel ? "mid" : "0", r,
                    (double)(long long)(t[0] - h.trace[0]) / 1e3, (double)(long long)(t[1] - t[0]) / 1e3, (double)(long long)(t[2] - t[1]) / 1e3, (double)(long long)(t[3] - t[2]) / 1e3);
        }
    } else
    if (getenv("SK_DEBUG_PROF") && h.trace[0]) {
        fprintf(stderr, "timeline (us from panel 20 start on CTA 0; replicated path: start, F, V+D1, barrier 1 left, A (thread 0), barrier 2 left, last arrival at barrier 2, at barrier 1; CTAs 0, G/2, G-1)\n");
        const u64 t0 = h.trace[0];
        for (int pnl = 0; pnl < 8; ++pnl) for (int cs = 0; cs < 3; ++cs) {
            fprintf(stderr, "  panel %d cta %s:", 20 + pnl, cs == 0 ? "0   " : cs == 1 ? "1   " : "last");
            for (int ev = 0; ev < 8; ++ev) { const u64 v = h.trace[(pnl * 3 + cs) * 8 + ev]; if (cs == 1 && ev == 6 && v) fprintf(stderr, " (last at barrier 2: CTA %llu)", (unsigned long long)(v & 0xff)); else if (v) fprintf(stderr, " %7.2f", (double)(long long)(v - t0) / 1e3); else fprintf(stderr, "       -"); }
            fprintf(stderr, "\n");
        }
    }
    if (getenv("SK_DEBUG_PROF") && h.cprof[8]) fprintf(stderr, "last panel-mode launch, CTA 0 us: destabilizer C->R %.1f, level-form panel loop %.1f, general panel loop %.1f, tail + R->C %.1f\n",
        (double)(long long)(h.cprof[9] - h.cprof[8]) / 1e3, (double)(long long)(h.cprof[10] - h.cprof[9]) / 1e3, (double)(long long)(h.cprof[11] - h.cprof[10]) / 1e3, (double)(long long)(h.cprof[12] - h.cprof[11]) / 1e3);
    if (getenv("SK_DEBUG_PANELS")) {
        fprintf(stderr, "per panel us: phase 1 (to the last arrival), barrier 1, phase 2, barrier 2\n");
        for (int pnl = 0; pnl < 160 && h.ptl[pnl * 6]; ++pnl)
            fprintf(stderr, "  panel %3d: %6.2f %5.2f %6.2f %5.2f  pairs %llu\n", pnl, (double)(long long)(h.ptl[pnl * 6 + 1] - h.ptl[pnl * 6]) / 1e3, (double)(long long)(h.ptl[pnl * 6 + 2] - h.ptl[pnl * 6 + 1]) / 1e3,
                    (double)(long long)(h.ptl[pnl * 6 + 3] - h.ptl[pnl * 6 + 2]) / 1e3, (double)(long long)(h.ptl[pnl * 6 + 4] - h.ptl[pnl * 6 + 3]) / 1e3, (unsigned long long)h.ptl[pnl * 6 + 5]);
    }
    if (getenv("SK_DEBUG_PROF") && h.cprof[15]) fprintf(stderr, "longest pair of the apply phase: %.2f us, %llu + %llu steps (stabilizer + destabilizer), flags %llu\n", (double)(h.cprof[15] >> 24) / 1e3, (unsigned long long)((h.cprof[15] >> 16) & 0xff), (unsigned long long)((h.cprof[15] >> 8) & 0xff), (unsigned long long)(h.cprof[15] & 0xff));
    if (getenv("SK_DEBUG_PROF")) { fprintf(stderr, "cprof cycles:"); for (int k = 0; k < 16; ++k) fprintf(stderr, " %llu", (unsigned long long)h.cprof[k]); fprintf(stderr, "\n"); }
    if (getenv("SK_DEBUG_PROF")) fprintf(stderr, "factorise us: load %.0f random steps %.0f (n=%llu) deterministic steps %.0f (n=%llu) tail %.0f\n",
                                         h.fprof[0] / 1e3, h.fprof[1] / 1e3, (unsigned long long)h.fprof[4], h.fprof[2] / 1e3, (unsigned long long)h.fprof[5], h.fprof[3] / 1e3);
    return SK_OK;
}

// ------------------------------------------------------------------ engine --
struct ProgOp { uint8_t type; uint32_t off, count; uint32_t boff = 0, nblocks = 0, nlayers = 1; };   // 0 = one k_layer launch (a layer, or merged layers with a chunk table d_boff[boff .. boff+nblocks]), 1 = measurement block
struct sk_program {
    sk_ctx* ctx = nullptr;
    uint64_t n = 0;
    std::vector<ProgOp> ops;
    sk_gate* d_gates = nullptr; size_t ngates = 0;
    u32* d_boff = nullptr;          // chunk tables of the merged-layer launches
    u32* d_mq = nullptr; uint8_t* d_out = nullptr; uint8_t* d_det = nullptr; size_t nmeas = 0;
    uint64_t hist[12] = {0};
    sk_tableau* last_t = nullptr;
    // the whole launch sequence of a run as a CUDA graph, replayed while (tableau, seed, entry state) stay the same
    cudaGraphExec_t gexec = nullptr; uint64_t g_tab_uid = 0, g_seed = 0; bool g_r_in = false, g_r_out = false, g_d_in = false, g_d_out = false, g_disabled = false;
    uint64_t g_launches = 0, g_layers = 0, g_transposes = 0;
};

extern "C" void sk_program_destroy(sk_program* p) {
    if (!p) return;
    cudaSetDevice(p->ctx->device);
    if (p->gexec) { cudaStreamSynchronize(p->ctx->stream); cudaGraphExecDestroy(p->gexec); }
    dfree(p->ctx, p->d_gates); dfree(p->ctx, p->d_boff); dfree(p->ctx, p->d_mq); dfree(p->ctx, p->d_out); dfree(p->ctx, p->d_det);
    delete p;
}
extern "C" uint64_t sk_program_measurements(const sk_program* p) { return p ? p->nmeas : 0; }


// ---- host-side compilation of a circuit with sim semantics -------------------------------
// Maximal runs of M gates are measurement blocks; the Clifford runs between them are layered independently
// (gates on disjoint qubits share a layer, per-qubit order preserved => same tableau as gate by gate).
struct Seg {
    size_t lo = 0, hi = 0; bool meas = false; size_t out = 0;   // gates [lo, hi) ; offset into the ordered gates / the qubit list
    std::vector<uint32_t> sizes;                               // Clifford run: gates per launch group (one layer, or merged layers)
    std::vector<uint32_t> glayers;                             //   logical layers in each group
    std::vector<uint32_t> gblocks;                             //   chunks in each group (0 = uniform chunks, no table)
    std::vector<uint32_t> boff;                                //   chunk tables of the merged groups, concatenated (nblocks+1 entries each, relative to the group)
    size_t bslot = 0;                                          //   first entry of this run's block in the chunk-table staging
    std::atomic<int> done{0};
};
static int target_ctas_for(const sk_ctx* c, uint64_t n) {
    const int W = int((n + 63) / 64);
    const int threads = std::min(256, std::max(32, (W + 31) & ~31));
    return layer_target_ctas(c, threads);
}
static unsigned host_threads(size_t ngates) {
    return ngates > (1u << 16) ? std::max(1u, std::min(16u, std::thread::hardware_concurrency())) : 1u;
}
template <class F> static void parallel_for(unsigned nthreads, size_t count, F&& fn) {          // fn(begin, end, thread)
    if (nthreads <= 1 || count < nthreads) { fn(size_t(0), count, 0u); return; }
    std::vector<std::thread> th;
    for (unsigned k = 0; k < nthreads; ++k) th.emplace_back([&, k] { fn(count * k / nthreads, count * (k + 1) / nthreads, k); });
    for (auto& t : th) t.join();
}
// threads look for any offending gate; the (rare) error path re-runs in order to report the first one
// pure scan (touches no context state, so it may run on a thread of its own): does any gate fail validation?
static bool circuit_has_bad_gate(uint64_t n, const sk_gate* gates, size_t ngates, unsigned nthreads) {
    std::atomic<bool> bad{false};
    parallel_for(nthreads, ngates, [&](size_t lo, size_t hi, unsigned) {
        bool b = false;
        for (size_t i = lo; i < hi; ++i) {
            const sk_gate& g = gates[i];
            b |= g.kind >= SK_T || g.q0 >= n || (sk_is_two_qubit(g.kind) && (g.q1 >= n || g.q0 == g.q1));
        }
        if (b) bad = true;
    });
    return bad;
}
// the slow path after a positive scan: the first offending gate, with its message in c->err
static int32_t report_bad_gate(sk_ctx* c, uint64_t n, const sk_gate* gates, size_t ngates) {
        for (size_t i = 0; i < ngates; ++i) {
            int32_t rc = validate_gate(c, gates[i], n, i);
            if (rc) return rc;
            if (gates[i].kind == SK_T || gates[i].kind == SK_TDG)
                SK_FAIL(c, SK_EUNSUPPORTED, "gate %zu: T/TDG is not a Clifford gate; use the transpiler path (SPEC:191)", i);
        }
    return SK_OK;
}
static int32_t validate_circuit(sk_ctx* c, uint64_t n, const sk_gate* gates, size_t ngates, unsigned nthreads) {
    return circuit_has_bad_gate(n, gates, ngates, nthreads) ? report_bad_gate(c, n, gates, ngates) : int32_t(SK_OK);
}
static std::vector<Seg> scan_segments(const sk_gate* gates, size_t ngates, size_t& ng, size_t& nm, unsigned nthreads = 1) {
    // boundaries = positions where "is a measurement" changes; found chunk-parallel, concatenated in order
    std::vector<std::vector<size_t>> cuts(std::max(1u, nthreads));
    parallel_for(nthreads, ngates, [&](size_t lo, size_t hi, unsigned k) {
        std::vector<size_t>& c = cuts[k];
        for (size_t i = std::max<size_t>(lo, 1); i < hi; ++i) if ((gates[i].kind == SK_M) != (gates[i - 1].kind == SK_M)) c.push_back(i);
    });
    std::vector<std::pair<size_t, size_t>> b;
    size_t start = 0;
    for (const auto& c : cuts) for (size_t i : c) { b.emplace_back(start, i); start = i; }
    if (ngates) b.emplace_back(start, ngates);
    std::vector<Seg> segs(b.size());
    ng = nm = 0;
    size_t nruns = 0;
    for (size_t k = 0; k < b.size(); ++k) {
        Seg& sg = segs[k];
        sg.lo = b[k].first; sg.hi = b[k].second; sg.meas = gates[sg.lo].kind == SK_M;
        if (sg.meas) { sg.out = nm; nm += sg.hi - sg.lo; } else { sg.out = ng; sg.bslot = 2 * ng + 2 * nruns; ++nruns; ng += sg.hi - sg.lo; }
    }
    return segs;
}
struct SegScratch { std::vector<uint32_t> level, lay, start, parent, csize, cid, corder, cstart, hopen, whead, wnext; std::vector<sk_gate> tmp, fused; };
static inline bool two_q(uint8_t k) { return sk_is_two_qubit(k) || k == SK_XCX; }
constexpr uint32_t kMaxCluster = 4;      // gates that share qubits across merged layers (e.g. H a ; CX a d) -- kept small so chunks stay balanced
// Layering of one Clifford run + merging of consecutive layers into launch groups.  Layers l and l+1 may share a launch
// when the gates that share qubits form small clusters: each cluster is then placed whole, in program order, inside one
// chunk of the launch (k_layer applies a chunk's gates in order per row-vector).  Surface-code rounds: H | CX | CX | CX | CX | H
// becomes {H,CX} {CX} {CX} {CX,H} -- 4 launches instead of 6.
// H-window pass over one Clifford run:  H a ; ... ; H a  with nothing but CX a->d on qubit a in between is the same Clifford as
// the window without its two H and every CX a->d replaced by XCX a,d = H_a CX H_a (H_a H_a = 1 between consecutive ones; gates
// on other qubits commute with H_a).  The X-type checks of a surface-code round lose both of their H layers this way: same
// tableau, bit for bit, two sub-layers less to stream.  Returns the (possibly shorter) run in sc.fused.
static size_t fuse_h_windows(const sk_gate* g, size_t cnt, uint64_t n, SegScratch& sc) {
    constexpr uint32_t NONE = 0xffffffffu; constexpr uint8_t DEL = 0xff;
    if (sc.hopen.size() < n) { sc.hopen.assign(n, 0); sc.whead.assign(n, NONE); }
    sc.fused.assign(g, g + cnt); sc.wnext.resize(cnt);
    std::vector<sk_gate>& f = sc.fused;
    size_t removed = 0;
    for (size_t i = 0; i < cnt; ++i) {
        const sk_gate G = f[i];
        if (G.kind == SK_H) {
            const uint32_t q = G.q0;
            if (sc.hopen[q]) {
                f[sc.hopen[q] - 1].kind = DEL; f[i].kind = DEL; removed += 2;
                for (uint32_t j = sc.whead[q]; j != NONE; j = sc.wnext[j]) f[j].kind = SK_XCX;
                sc.hopen[q] = 0;
            } else { sc.hopen[q] = uint32_t(i) + 1; sc.whead[q] = NONE; }
        } else if (G.kind == SK_CX) {
            sc.hopen[G.q1] = 0;                                   // a window does not survive being a target
            if (sc.hopen[G.q0]) { sc.wnext[i] = sc.whead[G.q0]; sc.whead[G.q0] = uint32_t(i); }
        } else { sc.hopen[G.q0] = 0; if (sk_is_two_qubit(G.kind)) sc.hopen[G.q1] = 0; }
    }
    for (size_t i = 0; i < cnt; ++i) { sc.hopen[g[i].q0] = 0; if (sk_is_two_qubit(g[i].kind)) sc.hopen[g[i].q1] = 0; }
    if (removed) { size_t o = 0; for (size_t i = 0; i < cnt; ++i) if (f[i].kind != DEL) f[o++] = f[i]; f.resize(o); }
    return f.size();
}
static void compile_segment(const sk_gate* gates, uint64_t n, Seg& sg, sk_gate* ordered, uint32_t* mq, SegScratch& sc, int target_ctas, bool fuse_h) {
    const sk_gate* g = gates + sg.lo; size_t cnt = sg.hi - sg.lo;
    if (sg.meas) { for (size_t i = 0; i < cnt; ++i) mq[sg.out + i] = g[i].q0; }
    else {
        if (fuse_h) { cnt = fuse_h_windows(g, cnt, n, sc); g = sc.fused.data(); }      // (the launch sizes below then add up to less than the run's length)
        if (sc.level.size() < n) { sc.level.assign(n, 0); sc.parent.assign(n, 0xffffffffu); sc.csize.assign(n, 0); }
        sc.lay.resize(cnt);
        uint32_t depth = 0;
        for (size_t i = 0; i < cnt; ++i) {
            uint32_t l = sc.level[g[i].q0];
            const bool two = two_q(g[i].kind);
            if (two) l = std::max(l, sc.level[g[i].q1]);
            sc.lay[i] = l; sc.level[g[i].q0] = l + 1; if (two) sc.level[g[i].q1] = l + 1;
            depth = std::max(depth, l + 1);
        }
        for (size_t i = 0; i < cnt; ++i) { sc.level[g[i].q0] = 0; if (two_q(g[i].kind)) sc.level[g[i].q1] = 0; }
        sc.start.assign(depth + 1, 0);
        for (size_t i = 0; i < cnt; ++i) sc.start[sc.lay[i] + 1]++;
        std::vector<uint32_t> lsize(depth);
        for (uint32_t d = 0; d < depth; ++d) { lsize[d] = sc.start[d + 1]; sc.start[d + 1] += sc.start[d]; }
        sk_gate* og = ordered + sg.out;
        for (size_t i = 0; i < cnt; ++i) og[sc.start[sc.lay[i]]++] = g[i];        // level-sorted, order within a level preserved
        // ---- merge consecutive levels into launch groups
        auto find = [&](uint32_t q) { while (sc.parent[q] != q) { sc.parent[q] = sc.parent[sc.parent[q]]; q = sc.parent[q]; } return q; };
        auto touch = [&](uint32_t q) { if (sc.parent[q] == 0xffffffffu) { sc.parent[q] = q; sc.csize[q] = 0; } };
        auto reset = [&](size_t lo, size_t hi) { for (size_t i = lo; i < hi; ++i) { sc.parent[og[i].q0] = 0xffffffffu; if (two_q(og[i].kind)) sc.parent[og[i].q1] = 0xffffffffu; } };
        auto add_gate = [&](const sk_gate& G) -> uint32_t {       // returns the gate count of the cluster the gate joins
            touch(G.q0);
            uint32_t r = find(G.q0);
            if (two_q(G.kind)) {
                touch(G.q1);
                uint32_t r1 = find(G.q1);
                if (r1 != r) { sc.parent[r1] = r; sc.csize[r] += sc.csize[r1]; }
            }
            return ++sc.csize[r];
        };
        sg.sizes.clear(); sg.glayers.clear(); sg.gblocks.clear(); sg.boff.clear();
        size_t lo = 0;                      // group = og[lo, hi)
        uint32_t d = 0;
        while (d < depth) {
            size_t hi = lo + lsize[d];
            uint32_t nl = 1, maxc = 0;
            for (size_t i = lo; i < hi; ++i) maxc = std::max(maxc, add_gate(og[i]));
            while (d + nl < depth) {        // try to take the next level in
                const size_t nhi = hi + lsize[d + nl];
                uint32_t m2 = maxc;
                for (size_t i = hi; i < nhi && m2 <= kMaxCluster; ++i) m2 = std::max(m2, add_gate(og[i]));
                if (m2 > kMaxCluster) {     // no: rebuild the union-find of the group without that level
                    reset(lo, nhi);
                    for (size_t i = lo; i < hi; ++i) add_gate(og[i]);
                    break;
                }
                maxc = m2; hi = nhi; ++nl;
            }
            const uint32_t gcount = uint32_t(hi - lo);
            uint32_t nblocks = 0;
            if (nl > 1) {
                // order the group's gates cluster by cluster (first appearance), keeping program order inside a cluster
                sc.cid.resize(gcount); sc.corder.clear();
                for (size_t i = lo; i < hi; ++i) {
                    const uint32_t r = find(og[i].q0);
                    if (!(sc.csize[r] & 0x80000000u)) { sc.csize[r] = 0x80000000u | uint32_t(sc.corder.size()); sc.corder.push_back(0); }
                    const uint32_t c = sc.csize[r] & 0x7fffffffu;
                    sc.cid[i - lo] = c; sc.corder[c]++;
                }
                sc.cstart.assign(sc.corder.size() + 1, 0);
                for (size_t c = 0; c < sc.corder.size(); ++c) sc.cstart[c + 1] = sc.cstart[c] + sc.corder[c];
                sc.tmp.resize(gcount);
                { std::vector<uint32_t>& pos = sc.corder; for (size_t c = 0; c < pos.size(); ++c) pos[c] = sc.cstart[c];
                  for (size_t i = 0; i < gcount; ++i) sc.tmp[pos[sc.cid[i]]++] = og[lo + i]; }
                for (size_t i = 0; i < gcount; ++i) og[lo + i] = sc.tmp[i];
                // chunks of about gcount / target_ctas gates, closed at cluster boundaries
                const uint32_t gpb = std::max<uint32_t>(1, (gcount + target_ctas - 1) / target_ctas);
                sg.boff.push_back(0);
                uint32_t open = 0;
                for (size_t c = 0; c + 1 < sc.cstart.size(); ++c) {
                    if (sc.cstart[c + 1] - open >= gpb) { sg.boff.push_back(sc.cstart[c + 1]); open = sc.cstart[c + 1]; ++nblocks; }
                }
                if (open != gcount) { sg.boff.push_back(gcount); ++nblocks; }
            }
            reset(lo, hi);
            sg.sizes.push_back(gcount); sg.glayers.push_back(nl); sg.gblocks.push_back(nblocks);
            lo = hi; d += nl;
        }
    }
    sg.done.store(1, std::memory_order_release);
}
// pinned host staging owned by the context (grown on demand): ordered gates then the measured-qubit list
static int32_t reserve_pinned(sk_ctx* c, size_t bytes) {
    if (bytes <= c->h_pin_cap) return SK_OK;
    SK_CUDA(c, cudaStreamSynchronize(c->stream));
    if (c->h_pin) cudaFreeHost(c->h_pin);
    c->h_pin = nullptr; c->h_pin_cap = 0;
    const size_t cap = std::max<size_t>(bytes + bytes / 4, 1 << 20);
    SK_CUDA(c, cudaHostAlloc(&c->h_pin, cap, cudaHostAllocDefault));
    c->h_pin_cap = cap;
    return SK_OK;
}

extern "C" int32_t sk_program_create(sk_ctx* c, uint64_t n, const sk_gate* gates, size_t ngates,
                                     const uint32_t* marks, size_t nmarks, int mode,
                                     sk_program** out, uint32_t* warnings) {
    if (!c || !out || (!gates && ngates) || (!marks && nmarks)) return SK_EARG;
    *out = nullptr;
    if (warnings) *warnings = 0;
    if (n == 0) SK_FAIL(c, SK_EDIM, "circuit has zero qubits");
    const unsigned nthreads = host_threads(ngates);
    { int32_t rc = validate_circuit(c, n, gates, ngates, nthreads); if (rc) return rc; }
    for (size_t k = 0; k < nmarks; ++k)
        if (marks[k] >= ngates || (k && marks[k] <= marks[k - 1])) SK_FAIL(c, SK_EARG, "chunk_marks must be strictly increasing and < gate count (SPEC:238)");

    sk_program* p = new sk_program();
    p->ctx = c; p->n = n;
    std::vector<sk_gate> ordered; ordered.reserve(ngates);
    std::vector<uint32_t> mq; std::vector<uint32_t> scratch, sizes, h_boff;
    uint32_t warn = 0;

    auto emit_sequential = [&](size_t lo, size_t hi) {      // sim semantics on gates [lo, hi)
        size_t i = lo;
        while (i < hi) {
            if (gates[i].kind == SK_M) {
                size_t j = i;
                while (j < hi && gates[j].kind == SK_M) { mq.push_back(gates[j].q0); ++j; }
                if (!p->ops.empty() && p->ops.back().type == 1) p->ops.back().count += uint32_t(j - i);
                else p->ops.push_back({1, uint32_t(mq.size() - (j - i)), uint32_t(j - i)});
                i = j; continue;
            }
            size_t j = i;
            while (j < hi && gates[j].kind != SK_M) ++j;
            sizes.clear();
            size_t base = ordered.size();
            sk_layer_run(gates + i, j - i, n, scratch, ordered, sizes);
            for (uint32_t s : sizes) { p->ops.push_back({0, uint32_t(base), s}); base += s; }
            i = j;
        }
    };
    if (mode == 0 || nmarks == 0) {
        size_t ng = 0, nm = 0;
        std::vector<Seg> segs = scan_segments(gates, ngates, ng, nm, nthreads);
        ordered.resize(ng); mq.resize(nm);
        std::atomic<size_t> next{0};
        const int tctas = target_ctas_for(c, n);
        parallel_for(nthreads, nthreads, [&](size_t, size_t, unsigned) {
            SegScratch sc;
            for (size_t si = next++; si < segs.size(); si = next++) compile_segment(gates, n, segs[si], ordered.data(), mq.data(), sc, tctas, !c->no_fuse_h);
        });
        for (const Seg& sg : segs) {
            if (sg.meas) { p->ops.push_back({1, uint32_t(sg.out), uint32_t(sg.hi - sg.lo)}); continue; }
            size_t base = sg.out, bo = 0;
            for (size_t k = 0; k < sg.sizes.size(); ++k) {
                ProgOp op{0, uint32_t(base), sg.sizes[k]};
                op.nlayers = sg.glayers[k]; op.nblocks = sg.gblocks[k];
                if (op.nblocks) { op.boff = uint32_t(h_boff.size()); h_boff.insert(h_boff.end(), sg.boff.begin() + bo, sg.boff.begin() + bo + op.nblocks + 1); bo += op.nblocks + 1; }
                p->ops.push_back(op);
                base += sg.sizes[k];
            }
        }
    } else {
        if (c->q_epoch.size() < n) c->q_epoch.assign(n, 0);
        size_t lo = 0;
        for (size_t k = 0; k <= nmarks; ++k) {
            size_t hi = (k < nmarks) ? marks[k] : ngates;
            if (hi == lo) continue;
            if (++c->epoch == 0) { std::fill(c->q_epoch.begin(), c->q_epoch.end(), 0); c->epoch = 1; }
            bool ok = true;
            for (size_t i = lo; i < hi && ok; ++i) {
                if (gates[i].kind == SK_M) { ok = false; break; }
                uint32_t qs[2] = {gates[i].q0, gates[i].q1};
                for (int e = 0; e < (sk_is_two_qubit(gates[i].kind) ? 2 : 1); ++e) {
                    if (c->q_epoch[qs[e]] == c->epoch) ok = false;
                    c->q_epoch[qs[e]] = c->epoch;
                }
            }
            if (ok) {                                     // validated chunk == one fused layer
                p->ops.push_back({0, uint32_t(ordered.size()), uint32_t(hi - lo)});
                ordered.insert(ordered.end(), gates + lo, gates + hi);
            } else {                                      // SPEC:324 fall back to sequential
                bool only_m = true;
                for (size_t i = lo; i < hi; ++i) only_m = only_m && gates[i].kind == SK_M;
                if (!only_m) warn |= 1u;
                emit_sequential(lo, hi);
            }
            lo = hi;
        }
    }
    for (size_t i = 0; i < ngates; ++i) p->hist[gates[i].kind]++;
    p->ngates = ordered.size(); p->nmeas = mq.size();
    cudaError_t e = cudaSuccess;
    if (p->ngates) { e = dmalloc(c, &p->d_gates, p->ngates * sizeof(sk_gate)); }
    if (!e && !h_boff.empty()) e = dmalloc(c, &p->d_boff, h_boff.size() * 4);
    if (!e && p->nmeas) { e = dmalloc(c, &p->d_mq, p->nmeas * 4); if (!e) e = dmalloc(c, &p->d_out, p->nmeas); if (!e) e = dmalloc(c, &p->d_det, p->nmeas); }
    if (e) { sk_program_destroy(p); SK_FAIL(c, SK_ECUDA, "cudaMalloc failed for the program: %s", cudaGetErrorString(e)); }
    if (p->ngates) e = cudaMemcpyAsync(p->d_gates, ordered.data(), p->ngates * sizeof(sk_gate), cudaMemcpyHostToDevice, c->stream);
    if (!e && !h_boff.empty()) e = cudaMemcpyAsync(p->d_boff, h_boff.data(), h_boff.size() * 4, cudaMemcpyHostToDevice, c->stream);
    if (!e && p->nmeas) e = cudaMemcpyAsync(p->d_mq, mq.data(), p->nmeas * 4, cudaMemcpyHostToDevice, c->stream);
    if (!e) e = cudaStreamSynchronize(c->stream);     // host vectors die at return
    if (e) { sk_program_destroy(p); SK_FAIL(c, SK_ECUDA, "program upload failed: %s", cudaGetErrorString(e)); }
    if (warnings) *warnings = warn;
    *out = p;
    return SK_OK;
}

static int32_t program_run_impl(sk_program* p, sk_tableau* t, uint64_t seed, float* class_ms) {
    if (!p || !t) return SK_EARG;
    sk_ctx* c = p->ctx;
    if (t->ctx != c) SK_FAIL(c, SK_EARG, "program and tableau belong to different contexts");
    if (t->n != p->n) SK_FAIL(c, SK_EDIM, "program is for %llu qubits, tableau has %llu", (unsigned long long)p->n, (unsigned long long)t->n);
    // profiled mode: CUDA events around every op on the launching stream; ms per kernel class
    // (0 fused layers, 1 transposes, 2 measurement blocks)
    std::vector<cudaEvent_t> ev; std::vector<int> cls;
    auto mark = [&](int k) {
        if (!class_ms) return;
        cudaEvent_t e; cudaEventCreate(&e); cudaEventRecord(e, c->stream); ev.push_back(e); cls.push_back(k);
    };
    auto enqueue_all = [&]() -> int32_t {
        mark(-1);
        for (const ProgOp& op : p->ops) {
            if (op.type == 0) {
                launch_layer(t, p->d_gates + op.off, int(op.count), op.nblocks ? p->d_boff + op.boff : nullptr, int(op.nblocks), int(op.nlayers));
                mark(0);
            } else {
                if (class_ms && !t->r_valid) { int32_t rc = rows_from_cols(t, true); if (rc) return rc; mark(1); }    // (otherwise launch_measure transposes, next to k_wave_cols)
                int32_t rc = launch_measure(t, p->d_mq + op.off, int(op.count), seed, op.off, p->d_out + op.off, p->d_det + op.off);
                if (rc) return rc;
                mark(2);
            }
        }
        join_side(c);
        return SK_OK;
    };
    const int no_pipe_in = c->no_pipe;
    if (class_ms) c->no_pipe = 1;            // class times: every kernel on the one stream, in order
    std::function<void(int)> mark_fn = mark;
    c->prof_mark = class_ms ? &mark_fn : nullptr;
    struct Restore { sk_ctx* c; int v; ~Restore() { c->no_pipe = v; c->prof_mark = nullptr; } } restore{c, no_pipe_in};
    const bool want_graph = !class_ms && !p->g_disabled && !c->no_graph && p->ops.size() >= 8;
    if (want_graph && p->gexec && p->g_tab_uid == t->uid && p->g_seed == seed && p->g_r_in == t->r_valid && p->g_d_in == t->r_destab_stale) {
        SK_CUDA(c, cudaGraphLaunch(p->gexec, c->stream));                     // replay
        t->r_valid = p->g_r_out; t->r_destab_stale = p->g_d_out;
        c->cnt.kernel_launches += p->g_launches; c->cnt.layers += p->g_layers; c->cnt.transposes += p->g_transposes;
    } else if (want_graph) {
        if (p->gexec) { cudaStreamSynchronize(c->stream); cudaGraphExecDestroy(p->gexec); p->gexec = nullptr; }
        const bool r_in = t->r_valid, d_in = t->r_destab_stale;
        const sk_counters before = c->cnt;
        cudaGraph_t graph = nullptr;
        int32_t rc = SK_OK;
        join_side(c);
        if (cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
            rc = enqueue_all();
            cudaError_t e = cudaStreamEndCapture(c->stream, &graph);
            if (!rc && e == cudaSuccess && graph && cudaGraphInstantiate(&p->gexec, graph, 0) == cudaSuccess) {
                p->g_tab_uid = t->uid; p->g_seed = seed; p->g_r_in = r_in; p->g_r_out = t->r_valid; p->g_d_in = d_in; p->g_d_out = t->r_destab_stale;
                p->g_launches = c->cnt.kernel_launches - before.kernel_launches; p->g_layers = c->cnt.layers - before.layers;
                p->g_transposes = c->cnt.transposes - before.transposes;
            } else { p->gexec = nullptr; p->g_disabled = true; c->side_pending = false; }
            if (graph) cudaGraphDestroy(graph);
            cudaGetLastError();
        } else { p->g_disabled = true; cudaGetLastError(); }
        if (rc) return rc;
        if (p->gexec) SK_CUDA(c, cudaGraphLaunch(p->gexec, c->stream));
        else {                              // capture is not possible here: plain stream launches
            t->r_valid = r_in; t->r_destab_stale = d_in; c->cnt = before;
            rc = enqueue_all();
            if (rc) return rc;
        }
    } else {
        int32_t rc = enqueue_all();
        if (rc) return rc;
    }
    SK_CUDA(c, cudaGetLastError());
    for (int k = 0; k < 12; ++k) c->cnt.gate_hist[k] += p->hist[k];
    p->last_t = t;
    if (class_ms) {
        SK_CUDA(c, cudaStreamSynchronize(c->stream));
        class_ms[0] = class_ms[1] = class_ms[2] = class_ms[3] = 0.f;
        for (size_t i = 1; i < ev.size(); ++i) { float ms = 0; cudaEventElapsedTime(&ms, ev[i - 1], ev[i]); class_ms[cls[i]] += ms; }
        for (int k = 0; k < 4; ++k) c->class_ms[k] = class_ms[k];
        for (cudaEvent_t e : ev) cudaEventDestroy(e);
    }
    return SK_OK;
}
extern "C" int32_t sk_program_run(sk_program* p, sk_tableau* t, uint64_t seed) { return program_run_impl(p, t, seed, nullptr); }
extern "C" int32_t sk_program_run_profiled(sk_program* p, sk_tableau* t, uint64_t seed, float class_ms[4]) {
    if (!class_ms) return SK_EARG;
    return program_run_impl(p, t, seed, class_ms);
}

// SPEC:330-338 run_shots: per-site counts of outcome 1 over `shots` runs with seeds seed ^ shot (device-side accumulation;
// nothing is synchronised between shots).
__global__ void k_accumulate_ones(const uint8_t* __restrict__ out, u32* __restrict__ counts, size_t nm) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nm && out[i]) counts[i] += 1u;
}
extern "C" int32_t sk_program_run_shots(sk_program* p, sk_tableau* t, uint64_t shots, uint64_t seed, uint32_t* ones, uint8_t* records) {
    if (!p || !t || !ones) return SK_EARG;
    sk_ctx* c = p->ctx;
    if (shots == 0) SK_FAIL(c, SK_EARG, "run_shots: shots must be >= 1 (SPEC:332)");
    const size_t nm = p->nmeas;
    u32* d_counts = nullptr;
    if (nm) { SK_CUDA(c, dmalloc(c, &d_counts, nm * 4)); SK_CUDA(c, cudaMemsetAsync(d_counts, 0, nm * 4, c->stream)); }
    const int keep = c->no_graph;
    c->no_graph = 1;                       // the seed changes every shot: plain launches instead of re-capturing a graph per shot
    int32_t rc = SK_OK;
    for (uint64_t s = 0; s < shots && !rc; ++s) {
        rc = tableau_identity(t);
        if (!rc) rc = program_run_impl(p, t, seed ^ s, nullptr);
        if (!rc && nm) {
            k_accumulate_ones<<<(unsigned)((nm + 255) / 256), 256, 0, c->stream>>>(p->d_out, d_counts, nm);
            c->cnt.kernel_launches++;
            if (records && cudaMemcpyAsync(records + s * nm, p->d_out, nm, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess) { c->err = "run_shots: record copy failed"; rc = SK_ECUDA; }
        }
    }
    c->no_graph = keep;
    if (!rc && nm && cudaMemcpyAsync(ones, d_counts, nm * 4, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess) { c->err = "run_shots: count copy failed"; rc = SK_ECUDA; }
    const int32_t rc2 = check_ws(c);       // synchronises
    dfree(c, d_counts);
    return rc ? rc : rc2;
}

extern "C" int32_t sk_program_read_record(sk_program* p, uint8_t* outcomes, uint8_t* deterministic) {
    if (!p) return SK_EARG;
    sk_ctx* c = p->ctx;
    if (p->nmeas) {
        if (!outcomes || !deterministic) return SK_EARG;
        SK_CUDA(c, cudaMemcpyAsync(outcomes, p->d_out, p->nmeas, cudaMemcpyDeviceToHost, c->stream));
        SK_CUDA(c, cudaMemcpyAsync(deterministic, p->d_det, p->nmeas, cudaMemcpyDeviceToHost, c->stream));
    }
    if (p->last_t) return check_ws(c);
    SK_CUDA(c, cudaStreamSynchronize(c->stream));
    return SK_OK;
}

// sim with host buffers, mode 0: compilation, upload and execution are pipelined.  Worker threads compile the
// segments in order into pinned staging; the calling thread uploads each finished segment (async copy) and enqueues
// its launches, so the device runs round r while the host still compiles round r+1.
static int32_t sim_pipelined(sk_ctx* c, uint64_t n, const sk_gate* gates, size_t ngates, uint64_t seed,
                             sk_tableau** out_t, uint8_t* outcomes, uint8_t* deterministic) {
    const unsigned nthreads = host_threads(ngates);
    static const bool dbg = getenv("SK_DEBUG_E2E") != nullptr;           // host-side stage times on stderr
    const auto tp0 = std::chrono::steady_clock::now();
    auto since = [&] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tp0).count(); };
    double ts_val = 0, ts_scan = 0, ts_alloc = 0, ts_first = 0, ts_enq = 0, ts_join = 0;
    // validation runs beside the segment scan and the allocations (neither looks at qubit indices); nothing is compiled or
    // launched before it has passed
    // (the thread only scans: c->err is written by the calling thread alone, after the join)
    bool vbad = false;
    std::thread vthread([&] { vbad = circuit_has_bad_gate(n, gates, ngates, std::max(1u, nthreads / 2)); ts_val = since(); });
    struct Joiner { std::thread& t; ~Joiner() { if (t.joinable()) t.join(); } } vjoin{vthread};
    int32_t rc = SK_OK;
    size_t ng = 0, nm = 0;
    std::vector<Seg> segs = scan_segments(gates, ngates, ng, nm, std::max(1u, nthreads / 2));
    ts_scan = since();
    const size_t nboff = 2 * ng + 2 * segs.size() + 2;       // chunk tables: a run of k gates needs at most 2k + 2 entries
    rc = reserve_pinned(c, ng * sizeof(sk_gate) + nm * 4 + nboff * 4 + 64);
    if (rc) return rc;
    sk_gate* h_gates = (sk_gate*)c->h_pin;
    uint32_t* h_mq = (uint32_t*)((char*)c->h_pin + ((ng * sizeof(sk_gate) + 15) & ~size_t(15)));
    uint32_t* h_boff = h_mq + ((nm + 3) & ~size_t(3));
    const int tctas = target_ctas_for(c, n);
    sk_program* p = new sk_program();
    p->ctx = c; p->n = n; p->ngates = ng; p->nmeas = nm;
    cudaError_t e = cudaSuccess;
    if (ng) { e = dmalloc(c, &p->d_gates, ng * sizeof(sk_gate)); if (!e) e = dmalloc(c, &p->d_boff, nboff * 4); }
    if (!e && nm) { e = dmalloc(c, &p->d_mq, nm * 4); if (!e) e = dmalloc(c, &p->d_out, nm); if (!e) e = dmalloc(c, &p->d_det, nm); }
    if (e) { sk_program_destroy(p); SK_FAIL(c, SK_ECUDA, "cudaMalloc failed for the program: %s", cudaGetErrorString(e)); }
    vthread.join();
    if (vbad) { sk_program_destroy(p); const int32_t vrc = report_bad_gate(c, n, gates, ngates); return vrc ? vrc : int32_t(SK_EARG); }
    sk_tableau* t = nullptr;
    rc = sk_tableau_create(c, n, &t);
    if (rc) { sk_program_destroy(p); return rc; }
    ts_alloc = since();
    std::atomic<size_t> next{0};
    std::vector<std::thread> workers;
    auto work = [&] { SegScratch sc; for (size_t si = next++; si < segs.size(); si = next++) compile_segment(gates, n, segs[si], h_gates, h_mq, sc, tctas, !c->no_fuse_h); };
    for (unsigned k = 1; k < nthreads; ++k) workers.emplace_back(work);
    SegScratch mine;
    size_t uploaded = 0, nbatches = 0;          // segments [0, uploaded) are on the device
    auto wait_done = [&](size_t si) {           // helps compiling while it waits
        while (!segs[si].done.load(std::memory_order_acquire)) {
            if (nthreads == 1 || next.load() <= si) { size_t k = next++; if (k < segs.size()) compile_segment(gates, n, segs[k], h_gates, h_mq, mine, tctas, !c->no_fuse_h); }
            else std::this_thread::yield();
        }
    };
    // uploads of large programs go through a stream of their own, ordered behind the allocations above and in front of the
    // launches that use them (small ones stay on the main stream: the events would cost more than the overlap gives)
    cudaStream_t copy_stream = nullptr; std::vector<cudaEvent_t> copy_events;
    struct CopyScope { cudaStream_t& s; std::vector<cudaEvent_t>& ev; ~CopyScope() { if (s) cudaStreamSynchronize(s); for (cudaEvent_t x : ev) cudaEventDestroy(x); } } copy_scope{copy_stream, copy_events};
    if (c->copy && !getenv("SK_NO_COPY_STREAM") && ng * sizeof(sk_gate) + nm * 4 >= (size_t)1 << 20) {
        cudaEvent_t ev = nullptr;
        if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess) { copy_events.push_back(ev); cudaEventRecord(ev, c->stream); cudaStreamWaitEvent(c->copy, ev, 0); copy_stream = c->copy; }
        else cudaGetLastError();
    }
    // one copy per array for every segment the workers have finished by now (they run ahead while the device is busy
    // with a measurement block): the ordered gates and the measured qubits are contiguous across segments
    auto upload_from = [&](size_t si) -> int32_t {
        size_t e_seg = si + 1;
        while (e_seg < segs.size() && segs[e_seg].done.load(std::memory_order_acquire)) ++e_seg;
        size_t g_lo = ~size_t(0), g_hi = 0, m_lo = ~size_t(0), m_hi = 0, b_lo = ~size_t(0), b_hi = 0;
        for (size_t k = si; k < e_seg; ++k) {
            const Seg& q = segs[k]; const size_t qc = q.hi - q.lo;
            if (q.meas) { m_lo = std::min(m_lo, q.out); m_hi = std::max(m_hi, q.out + qc); }
            else {
                g_lo = std::min(g_lo, q.out); g_hi = std::max(g_hi, q.out + qc);
                if (!q.boff.empty()) {
                    std::memcpy(h_boff + q.bslot, q.boff.data(), q.boff.size() * 4);
                    b_lo = std::min(b_lo, q.bslot); b_hi = std::max(b_hi, q.bslot + q.boff.size());
                }
            }
        }
        // on the copy stream: the kernels of earlier segments keep running on the main stream while the next batch comes up
        cudaStream_t cs = copy_stream ? copy_stream : c->stream;
        if (!e && m_hi > m_lo) e = cudaMemcpyAsync(p->d_mq + m_lo, h_mq + m_lo, (m_hi - m_lo) * 4, cudaMemcpyHostToDevice, cs);
        if (!e && g_hi > g_lo) e = cudaMemcpyAsync(p->d_gates + g_lo, h_gates + g_lo, (g_hi - g_lo) * sizeof(sk_gate), cudaMemcpyHostToDevice, cs);
        if (!e && b_hi > b_lo) e = cudaMemcpyAsync(p->d_boff + b_lo, h_boff + b_lo, (b_hi - b_lo) * 4, cudaMemcpyHostToDevice, cs);
        if (!e && copy_stream) {
            cudaEvent_t ev = nullptr;
            e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
            if (!e) { copy_events.push_back(ev); e = cudaEventRecord(ev, copy_stream); }
            if (!e) e = cudaStreamWaitEvent(c->stream, ev, 0);
        }
        if (e) { c->err = cudaGetErrorString(e); return SK_ECUDA; }
        uploaded = e_seg; ++nbatches;
        return SK_OK;
    };
    auto launch_seg = [&](size_t si) -> int32_t {
        const Seg& sg = segs[si];
        if (sg.meas) return launch_measure(t, p->d_mq + sg.out, int(sg.hi - sg.lo), seed, sg.out, p->d_out + sg.out, p->d_det + sg.out);
        size_t base = sg.out, bo = 0;
        for (size_t k = 0; k < sg.sizes.size(); ++k) {
            const uint32_t nb = sg.gblocks[k];
            launch_layer(t, p->d_gates + base, int(sg.sizes[k]), nb ? p->d_boff + sg.bslot + bo : nullptr, int(nb), int(sg.glayers[k]));
            if (nb) bo += nb + 1;
            base += sg.sizes[k];
        }
        return SK_OK;
    };
    // Plain stream launches, segment by segment as the worker threads finish compiling them.  (Round 1 launched everything behind
    // the first measurement block as one captured CUDA graph; measured again in round 2 with the shorter kernels: capture +
    // instantiation of the ~500 nodes is 3.8 ms of host time -- 7.7 ms with the two-stream measurement pipeline in the graph --
    // during which the device idles once the first block is done, against 1.8 ms of launch gaps this way: d=71 end to end 11.7 ms
    // here, 12.0 ms with the graph and no pipeline, 15.7 ms with both.  Graph replay stays where it pays: sk_program_run.)
    for (size_t si = 0; si < segs.size() && !rc; ++si) {
        wait_done(si);
        if (si == 0) ts_first = since();
        if (si >= uploaded) rc = upload_from(si);
        if (!rc) rc = launch_seg(si);
    }
    join_side(c);
    ts_enq = since();
    next = segs.size();
    for (auto& w : workers) w.join();
    ts_join = since();
    if (!rc) {
        uint64_t hist[12] = {0};
        for (size_t i = 0; i < ngates; ++i) hist[gates[i].kind]++;
        for (int k = 0; k < 12; ++k) c->cnt.gate_hist[k] += hist[k];
        p->last_t = t;
        const double ts_hist = since();
        rc = sk_program_read_record(p, outcomes, deterministic);
        if (dbg) fprintf(stderr, "sk_sim host ms: validate %.2f scan %.2f alloc+tableau %.2f first segment ready %.2f all enqueued %.2f workers joined %.2f histogram %.2f record read (device done) %.2f | %u threads, %zu segments in %zu uploads\n",
                         ts_val, ts_scan, ts_alloc, ts_first, ts_enq, ts_join, ts_hist, since(), nthreads, segs.size(), nbatches);
    } else cudaStreamSynchronize(c->stream);
    sk_program_destroy(p);
    if (rc) { sk_tableau_destroy(t); return rc; }
    *out_t = t;
    return SK_OK;
}

extern "C" int32_t sk_sim(sk_ctx* c, uint64_t n, const sk_gate* gates, size_t ngates,
                          const uint32_t* marks, size_t nmarks, int mode, uint64_t seed,
                          sk_tableau** out_t, uint8_t* outcomes, uint8_t* deterministic, uint32_t* warnings) {
    if (!c || !out_t || (!gates && ngates) || (!marks && nmarks)) return SK_EARG;
    *out_t = nullptr;
    if (warnings) *warnings = 0;
    if (n == 0) SK_FAIL(c, SK_EDIM, "circuit has zero qubits");
    for (size_t k = 0; k < nmarks; ++k)
        if (marks[k] >= ngates || (k && marks[k] <= marks[k - 1])) SK_FAIL(c, SK_EARG, "chunk_marks must be strictly increasing and < gate count (SPEC:238)");
    if (mode == 0 || nmarks == 0) return sim_pipelined(c, n, gates, ngates, seed, out_t, outcomes, deterministic);
    sk_program* p = nullptr; sk_tableau* t = nullptr;
    int32_t rc = sk_program_create(c, n, gates, ngates, marks, nmarks, mode, &p, warnings);
    if (rc) return rc;
    rc = sk_tableau_create(c, n, &t);
    if (!rc) rc = sk_program_run(p, t, seed);
    if (!rc) rc = sk_program_read_record(p, outcomes, deterministic);
    sk_program_destroy(p);
    if (rc) { sk_tableau_destroy(t); return rc; }
    *out_t = t;
    return SK_OK;
}

#include "sk_rows_impl.cuh"
#include "sk_shard_impl.cuh"
