// kernels_measure.cuh -- K2/K3/K4: a block of consecutive Z measurements executed by
// ONE persistent cooperative kernel (no host round trips; branches are data dependent).
// Exact CHP semantics (Algorithm 1): the tableau, signs and
// record are bit-identical to measuring one qubit at a time, in order.
//
// Two modes inside the kernel.
//
// WAVE mode (deterministic prefixes).  Over a window of pending measurements:
//   P1  pivot search = scan of the stabilizer half of column x_q in the C form (contiguous;
//       ffs + warp min) -- K2; the index r0 of the first random measurement is min-reduced.
//                                                                         -- grid barrier --
//   P2  every j < r0 is deterministic and read-only: ordered product of the stabilizer
//       partners from the R form, phase by popcounts mod 4 -- K4 (a warp per measurement, a
//       whole CTA for long products).  A window without random measurements is done after
//       this single barrier (rounds 2..d of a memory experiment: one wave per round).
//
// PANEL mode (from the first random measurement to the end of the block): blocked
// elimination, the bit-matrix analogue of a right-looking LU panel factorisation.  A panel =
// the next B <= 64 measurements (B * RW words must fit in shared memory).
//   G   gather: the panel's B x-columns at the panel-start state, read from the R form.
//   F   factorise (CTA 0, panel in shared memory): the B measurements are simulated IN ORDER
//       on the panel's own bits only -- pivot (smallest stabilizer row), frozen
//       target mask m_l, update of the later panel columns, the two overwritten rows -- which
//       fixes, symbolically, every full-row operation sequential CHP would perform:
//         hist_l  = steps k < l that multiplied the pivot row p_l before it was used,
//         M_h     = steps l whose pivot is multiplied into row h,
//         D_j     = partner set of a deterministic step j (split into rows that are still
//                   panel-start stabilizers, N_j = parity of their histories, and rows that
//                   earlier steps turned into +-Z).
//   V   pivot values: P_l' = (prod_{k in hist_l} P_k') * row p_l  -- the value row p_l has when
//       it is used; word-parallel (a thread owns one word of all B rows), phases reduced later.
//   A   every touched row replays its own list   row_h := (prod_{l in M_h} P_l') * row_h
//       independently (warp per row); destabilizer p_l + n starts from P_l'; row p_l := +-Z_q
//       with the counter RNG bit of the measurement's ordinal.
//   D   deterministic outcomes: sign of  prod_{i in D_j} row_i(panel start) * prod_{l in N_j} P_l'
//       * prod (+-Z_{q_l}); equal to the sequential scratch-row product because all factors
//       are commuting Hermitian operators (P^2 = +I cancels repeated factors).
//   Every row undergoes exactly the multiplications of sequential CHP, in the same order;
//   tools/proto_panel.py checks the scheme against the oracle.  Panel mode updates only the R
//   form; before the kernel exits it re-derives the C form itself (tile transpose over all CTAs).
// Row i = p+n is never a rowsum target (SURVEY.md section 7 hazard): it is overwritten.
//
// Roofline: HBM/L2.  Algorithmic bytes: random  RW*8 + 16W + k*32W + 32W ;
// deterministic  RW*8/2 + k*16W  -- reported from the k counters kept here.
#pragma once
#include "common.cuh"
#include "kernels_transpose.cuh"

namespace skd {

constexpr int kPanelMax = 64;
constexpr int kRowK = 4, kRowThreads = 512;              // row-form factorisation: slots per thread, threads
constexpr int kRowSlots = kRowK * kRowThreads;            // 2048 rows incl. up to kPanelMax virtual ones
constexpr int kRowCap = kRowSlots - kPanelMax;

struct PanelInfo {      // global scratch describing the current panel (written by CTA 0 in F)
    u64 hist[kPanelMax];   // random step l: earlier random steps whose pivot was multiplied into row p_l
    u64 dN[kPanelMax];     // deterministic step j: pivot values to multiply (parity of partner histories; written by D part 1)
    u64 dZ[kPanelMax];     // deterministic step j: earlier steps whose +-Z row is a partner
    u32 piv[kPanelMax];    // pivot stabilizer row-bit, 0xffffffff = deterministic step
    u32 eph[2][kPanelMax]; // V: sum over words of the g contributions of P_l' (atomic, mod 4 matters); double-buffered by panel parity
    int dete[kPanelMax];   // D part 1: phase exponent of the panel-start partner product
    u64 randmask;          // steps that are random
    u64 osign;             // panel-start sign bits of the pivot rows
    u32 nt;                // touched rows (entries of tlist / tM)
    u32 acount;            // G: active rows of the panel being gathered (reset by F)
    u32 dmode;             // partners of the deterministic steps: 0 = bit columns in pan, 1 = lists in dpart
    u32 pad;
    u32 dcnt[kPanelMax];   // dmode 1: partners per deterministic step
    uint8_t outc[kPanelMax];   // outcome of the random steps (counter RNG)
    u32 lvcount[2];        // replicated path (kernels_panel.cuh): pairs in the two pair-list buffers
    // replicated path, D1 split over several CTAs: what parts 1..3 of a deterministic step found (part 0 stays in its CTA's shared memory)
    int dp_e[3][kPanelMax]; u64 dp_N[3][kPanelMax], dp_Z[3][kPanelMax];
};

struct MeasWs {
    // ---- first 32 bytes: zeroed by ONE memset before each launch
    u32 bar;            // grid barrier counter
    u32 progress;       // panel mode: factorisation steps published so far in this launch (monotone)
    u32 r0[4];          // per-wave ~index of the first random measurement (0 = none), max-reduced; 3 slots rotate
    u32 exitcnt;        // CTAs that have left the kernel: the last one re-zeroes this block for the next launch
    u32 wdone;          // k_wave_cols / k_wave_rows: CTAs that have finished (the last one publishes wpos / accounts, and re-zeroes this word and r0[3])
    // ---- persistent
    u32 err;            // bit0 odd phase (invariant), bit31 barrier timeout, bit30 TMA timeout
    u32 wpos;           // k_wave_cols -> k_wave_rows, k_measure_block: measurements [0, wpos) of the block are deterministic and left to k_wave_rows
    u64 n_rand, n_det, k_rand, k_det, waves;
    u64 prof[8];        // CTA-0 wall time (ns): P1, P2, gather, factorise, values+detA, apply+detB, barriers(wave), barriers(panel)
    u64 panels;
    u64 cprof[16];      // debug: SM cycles per step section, thread 0 [0..7] and thread 96 [8..15]: random {search+bar, gather+bar, update}, det {search+bar, gather+bar, rest}
    u64 ctaphase[160 * 4];   // debug: per-CTA own time (ns) in panel phases G, F, V+D1, A+D2 (excluding barrier waits)
    u64 fprof[8];       // factorise (CTA 0) ns: load, random steps, deterministic steps, tail ; [4] random steps, [5] deterministic steps
    u64 ptl[160 * 6];   // debug (SK_DEBUG_PROF): per panel of the last launch: start, last arrival at barrier 1, barrier 1 left, last arrival at barrier 2, barrier 2 left (ns)
    u64 trace[8 * 3 * 8];   // debug timeline (globaltimer ns): panels 20..27 of a launch x CTA {0, 1, last} x 8 events
};

constexpr int kMeasThreads = 512;
constexpr int kMeasWarps = kMeasThreads / 32;
constexpr int kSlotsPerWarp = 4;
constexpr int kColChunk = 6;         // column words per lane loaded back-to-back (192 words per chunk)
constexpr int kMaxTargets = 2048;    // partner-list capacity of the CTA-wide product (dense fallback above)
constexpr int kWarpDirect = 16;      // panel mode: longer partner products go to a whole CTA (<= 1 per CTA and panel)
constexpr int kWarpList = 64;        // rows a single warp multiplies from its list; longer products are tree-reduced by a CTA

struct MeasArgs {
    DMat m;             // tableau (C and R valid on entry)
    int n;              // qubits == rows per half
    int NS;             // row-bit offset of the destabilizer half (64*W)
    const u32* qubits;  // measurement list
    int count;
    uint64_t seed, ordinal0;
    uint8_t* outcomes;  // [count]
    uint8_t* dets;      // [count]
    MeasWs* ws;
    u32* wpiv;          // [2][window] pivot of a window slot (0xffffffff = deterministic), by wave parity
    u32* wl;            // [2*window][kWarpList] k_wave_cols -> k_wave_rows: partner stabilizers of each measurement
    u64* wsgn;          // [W] k_wave_cols -> k_wave_rows: the stabilizer signs at the time of the measurement block
    // panel mode scratch
    int B;              // panel width (<= kPanelMax)
    u64* pan;           // [B][RW] gathered panel ; after F: destabilizer halves of deterministic steps hold D_j
    u64* pivbuf;        // [B] rows in R layout: P_l' x words then z words
    u64* detacc;        // [B] rows in R layout: panel-start partner products of the deterministic steps
    PanelInfo* info;
    u32* tlist;         // [2][tcap] touched rows            } double-buffered by panel parity: the apply phase of panel k
    u64* tM;            // [2][tcap] their step masks        } retires the entries of panel k-1 while panel k+1 is prepared
    u32 tcap;           // entries per buffer
    u32* alist_h;       // [64*RW] G: active rows (row-bits) of the panel, row form
    u64* alist_b;       // [64*RW]    and their bits in the panel columns
    u32* dpart;         // [B][kRowSlots] row form: partner stabilizers of the deterministic steps
    u64* rowM;          // [2][64*RW] step mask by row-bit (zero for rows the panel does not touch), double-buffered likewise
    int prof;           // device-side phase timers (SK_DEBUG_PROF)
    u64* tbits;         // [RW] row-bits listed in tlist of the panel just factorised (the folded gather skips them)
    int fold;           // gather of the next panel folded into the apply phase (SK_NO_FOLD=1 disables)
    int row_cap;        // most active rows the row-form factorisation takes (kRowCap; SK_ROW_CAP lowers it for tests)
    int destab_stale;   // the R form holds only the stabilizer rows (host transposed that half): panel mode derives the rest itself
    int force_columns;  // SK_PANEL_COLUMNS=1: always use the column-form factorisation (testing aid)
    int lv_enable;      // replicated level-form panel path (kernels_panel.cuh); SK_PANEL_REPL=0 disables
    int from_wave;      // the wave kernels ran first: start at ws->wpos
    int seq_rows;       // SK_PANEL_SEQ=1: step-by-step row-form factorisation instead of the level form (A/B and testing aid)
};

__device__ __forceinline__ u64 gtime() { u64 t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
// normal kernel exit: the last CTA to leave (every other one is past all grid barriers) re-zeroes the launch-scoped words,
// so the host needs no memset between measurement blocks (it zeroes them itself after an error)
#define SK_MEAS_EXIT() do { __syncthreads(); if (threadIdx.x == 0) { __threadfence(); if (atomicAdd(&ws->exitcnt, 1u) == gridDim.x - 1) { \
        ws->bar = 0; ws->progress = 0; ws->r0[0] = 0; ws->r0[1] = 0; ws->r0[2] = 0; ws->r0[3] = 0; __threadfence(); ws->exitcnt = 0; } } } while (0)
#define SK_PROF(k) do { if (a.prof && blockIdx.x == 0 && tid == 0) { u64 _n = gtime(); ws->prof[k] += _n - t_prof; t_prof = _n; } } while (0)

__device__ __forceinline__ int sign_bit(const u64* sgn, int r) { return int((ldcg(sgn + (r >> 6)) >> (r & 63)) & 1ull); }
__device__ __forceinline__ void named_bar(int id, int nthreads) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory"); }
__device__ __forceinline__ void st_release(u32* p, u32 v) { asm volatile("st.release.gpu.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }
// bounded wait until *p >= target (monotone counter); false on timeout
__device__ __forceinline__ bool wait_geq(const u32* p, u32 target) {
    for (unsigned long long spins = 0; spins < (1ull << 22); ++spins) {
        if (int(ld_acquire(p) - target) >= 0) return true;
        __nanosleep(100);            // keep the polling traffic away from the producer's stores
    }
    return false;
}
__device__ __forceinline__ u64 warp_xor64(u64 v) {        // two REDUX instead of ten shuffles
    const u32 lo = __reduce_xor_sync(0xffffffffu, (u32)v), hi = __reduce_xor_sync(0xffffffffu, (u32)(v >> 32));
    return ((u64)hi << 32) | lo;
}

// Multiplies the rows listed in `list` (row indices into `base`, R layout: x words then z words,
// Wp each) into the warp-private accumulator acc_x/acc_z [Wp] (lane-strided words), each as the
// LEFT factor.  Returns this lane's share of the i-exponent (the caller adds the factors' sign
// bits and reduces with warp_sum).  All factors commute, so any grouping/order gives the same
// Hermitian product; 8 rows are loaded per step so their latencies overlap.
__device__ __forceinline__ int warp_mul_list(const u64* base, int W, int Wp, const u32* list, int cnt,
                                             u64* acc_x, u64* acc_z, int lane) {
    int e = 0;
    for (int i0 = 0; i0 < cnt; i0 += 8) {
        int s[8]; int ns = 0;
#pragma unroll
        for (int t = 0; t < 8; ++t) { const int i = i0 + t; if (i < cnt) { s[t] = int(list[i]); ns = t + 1; } else s[t] = 0; }
        for (int w = lane; w < W; w += 32) {
            u64 sx[8], sz[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) if (t < ns) {
                const u64* rx = base + (size_t)(2 * s[t]) * Wp;
                sx[t] = ldcg(rx + w); sz[t] = ldcg(rx + Wp + w);
            }
            u64 ax = acc_x[w], az = acc_z[w];
#pragma unroll
            for (int t = 0; t < 8; ++t) if (t < ns) {
                e += g_word(sx[t], sz[t], ax, az);      // rowsum(acc, s): left factor = row s
                ax ^= sx[t]; az ^= sz[t];
            }
            acc_x[w] = ax; acc_z[w] = az;
        }
    }
    return e;
}

// ---- CTA-wide building blocks (all kMeasThreads threads call them together) -------------
struct MeasSmem {
    u64* acc;       // [kMeasWarps][2*Wp] per-warp product accumulators (start of the dynamic region)
    int* pe; int* pk; u64* pn;
    int* cnt;       // list length
    u32* targets;   // [kMaxTargets] partner rows
};

// K4 by a whole CTA: the partner list (set bits of dcol[0..W), stabilizer indices) is compacted
// into shared memory, then thread (w, g) owns word w of the product for row group g and
// multiplies its share of the listed rows word by word, 8 row loads in flight; groups are folded
// and the per-word phase contributions block-reduced (popcounts mod 4).  Word-parallel evaluation
// is the same product: g is a sum over qubit positions; the list order is irrelevant because
// stabilizer rows commute.  Returns (CTA-uniform) the phase exponent mod 4 including the rows'
// signs; if out_x != nullptr the product words are stored there (R layout).  *total_out = #rows.
// sm.cnt[0] is zero on entry and on exit.
__device__ __forceinline__ int cta_det(const MeasArgs& a, const MeasSmem& sm, const u64* dcol, u64* out_x, int* total_out, const u64* rowM = nullptr, u64* n_out = nullptr,
                                       const u32* glist = nullptr, int gcount = 0) {
    const int Wp = a.m.Wp, W = a.m.W;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (glist) {          // partners given as a list (<= kMaxTargets entries) instead of a bit column
        for (int i = tid; i < gcount; i += kMeasThreads) sm.targets[i] = __ldcg(glist + i);
        if (tid == 0) sm.cnt[0] = gcount;
    }
    for (int w0 = 0; w0 < (glist ? 0 : W); w0 += kMeasThreads) {
        const int w = w0 + tid;
        u64 bits = (w < W) ? ldcg(dcol + w) : 0ull;
        const int pc = __popcll(bits);
        int incl = pc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) { const int v = __shfl_up_sync(0xffffffffu, incl, o); if (lane >= o) incl += v; }
        int base = 0;
        if (lane == 31 && incl) base = atomicAdd(&sm.cnt[0], incl);
        base = __shfl_sync(0xffffffffu, base, 31);
        int ti = base + incl - pc;
        while (bits) {
            const int b = __ffsll((long long)bits) - 1; bits &= bits - 1;
            if (ti < kMaxTargets) sm.targets[ti] = u32(w * 64 + b);
            ++ti;
        }
    }
    __syncthreads();
    const int total = sm.cnt[0];
    int e = 0;
    u64 nx = 0;                                           // XOR of the listed rows' step masks (panel mode)
    u64 ax = 0, az = 0;                                   // this thread's word of the running product
    const int Wq = (W + 31) & ~31;
    const int ngroups = max(1, min(kMeasThreads / Wq, (total + 7) / 8));
    const int myw = tid % Wq, myg = tid / Wq;
    auto multiply_list = [&](int cnt) {
        if (Wq <= kMeasThreads) {
            if (myw < W && myg < ngroups) {
                for (int i0 = myg; i0 < cnt; i0 += 8 * ngroups) {
                    u64 sx[8], sz[8];
#pragma unroll
                    for (int t = 0; t < 8; ++t) {
                        const int i = i0 + t * ngroups;
                        if (i < cnt) { const u64* rx = a.m.rows + (size_t)(2 * sm.targets[i]) * Wp; sx[t] = ldcg(rx + myw); sz[t] = ldcg(rx + Wp + myw); }
                        else { sx[t] = 0; sz[t] = 0; }
                    }
#pragma unroll
                    for (int t = 0; t < 8; ++t) { e += g_word(sx[t], sz[t], ax, az); ax ^= sx[t]; az ^= sz[t]; }
                }
            }
        }
        for (int i = tid; i < cnt; i += kMeasThreads) { e += 2 * sign_bit(a.m.sgn, int(sm.targets[i])); if (rowM) nx ^= ldcg(rowM + sm.targets[i]); }
    };
    if (Wq > kMeasThreads) {
        // very wide rows: a thread owns several words; the running product lives in out_x / sm.acc
        // (not needed below 2^15 qubits; kept simple: one row at a time)
        u64* px = out_x ? out_x : sm.acc;
        for (int w = tid; w < 2 * Wp; w += kMeasThreads) px[w] = 0;
        __syncthreads();
        for (int base = 0; base < total; base += kMaxTargets) {
            if (base) {     // refill the list with the next slice, in column order
                __syncthreads();
                if (tid == 0) {
                    int rank = 0, fill = 0;
                    for (int w = 0; w < W && fill < kMaxTargets; ++w) {
                        u64 bits = ldcg(dcol + w);
                        while (bits && fill < kMaxTargets) { const int b = __ffsll((long long)bits) - 1; bits &= bits - 1; if (rank >= base) sm.targets[fill++] = u32(w * 64 + b); ++rank; }
                    }
                }
                __syncthreads();
            }
            const int cnt = min(total - base, kMaxTargets);
            for (int w = tid; w < W; w += kMeasThreads) {
                u64 bx = px[w], bz = px[Wp + w];
                for (int i = 0; i < cnt; ++i) {
                    const u64* rx = a.m.rows + (size_t)(2 * sm.targets[i]) * Wp;
                    const u64 sx = ldcg(rx + w), sz = ldcg(rx + Wp + w);
                    e += g_word(sx, sz, bx, bz); bx ^= sx; bz ^= sz;
                }
                px[w] = bx; px[Wp + w] = bz;
            }
            for (int i = tid; i < cnt; i += kMeasThreads) { e += 2 * sign_bit(a.m.sgn, int(sm.targets[i])); if (rowM) nx ^= ldcg(rowM + sm.targets[i]); }
        }
    } else if (total <= kMaxTargets) {
        multiply_list(total);
    } else {
        // more partners than list slots (dense tableaux): column-order slices selected by rank
        for (int base = 0; base < total; base += kMaxTargets) {
            __syncthreads();
            int seen = 0;
            for (int w0 = 0; w0 < W; w0 += kMeasThreads) {
                const int w = w0 + tid;
                const u64 bits = (w < W) ? ldcg(dcol + w) : 0ull;
                const int pc = __popcll(bits);
                int incl = pc;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) { int v = __shfl_up_sync(0xffffffffu, incl, o); if (lane >= o) incl += v; }
                if (lane == 31) sm.pk[warp] = incl;
                __syncthreads();
                int woff = 0, chunk_total = 0;
                for (int t = 0; t < kMeasWarps; ++t) { if (t < warp) woff += sm.pk[t]; chunk_total += sm.pk[t]; }
                int rank = seen + woff + incl - pc;
                u64 bb = bits;
                while (bb) {
                    const int b = __ffsll((long long)bb) - 1; bb &= bb - 1;
                    if (rank >= base && rank < base + kMaxTargets) sm.targets[rank - base] = u32(w * 64 + b);
                    ++rank;
                }
                seen += chunk_total;
                __syncthreads();
            }
            multiply_list(min(total - base, kMaxTargets));
        }
    }
    if (Wq <= kMeasThreads) {
        // fold the row groups (each holds a partial product of its word) and reduce the phase
        if (ngroups > 1) {
            if (myw < W && myg > 0 && myg < ngroups) { sm.acc[(size_t)(myg - 1) * 2 * Wp + myw] = ax; sm.acc[(size_t)(myg - 1) * 2 * Wp + Wp + myw] = az; }
            __syncthreads();
            if (myw < W && myg == 0)
                for (int g = 1; g < ngroups; ++g) {
                    const u64 bx = sm.acc[(size_t)(g - 1) * 2 * Wp + myw], bz = sm.acc[(size_t)(g - 1) * 2 * Wp + Wp + myw];
                    e += g_word(bx, bz, ax, az); ax ^= bx; az ^= bz;
                }
        }
        if (out_x && myw < W && myg == 0) { __stcg(out_x + myw, ax); __stcg(out_x + Wp + myw, az); }
    }
    e = warp_sum(e);
    if (lane == 0) sm.pe[warp] = e;
    if (rowM) { nx = warp_xor64(nx); if (lane == 0) sm.pn[warp] = nx; }
    __syncthreads();
    int et = 0;
    for (int t = 0; t < kMeasWarps; ++t) et += sm.pe[t];
    if (rowM && n_out) { u64 nt = 0; for (int t = 0; t < kMeasWarps; ++t) nt ^= sm.pn[t]; *n_out = nt; }
    *total_out = total;
    __syncthreads();
    if (tid == 0) sm.cnt[0] = 0;
    __syncthreads();
    return et & 3;
}

// ------------------------------------------------------------------ panel mode ------------
// F: symbolic factorisation of one panel by CTA 0.  sp = dynamic smem: panel [Bn][RW] then the
// pivot mask [W] (stabilizer rows used as pivots so far).
struct PanelSmem {
    u32 piv[kPanelMax]; u64 hist[kPanelMax], pw[kPanelMax], dZ[kPanelMax], S[kPanelMax]; uint8_t outc[kPanelMax];
    u32 full32[2]; u32 nt; u32 krand; u32 kdet; int steps;
    u32 dcnt[kPanelMax]; u32 gmin[3]; u64 wbp[2][kRowThreads / 32], wmp[2][kRowThreads / 32]; u32 wcnt[kRowThreads / 32]; u64 psign; u32 podd; u32 pready;
};

// Common tail of the row-form factorisations: the pivots join the touched-row list, outcomes of the random steps
// (counter RNG), panel-start signs of the pivot rows, counters, and the panel description for the other CTAs.
__device__ __forceinline__ void panel_rows_tail(const MeasArgs& a, PanelSmem& ps, int pos, int Bn, u32* tlist, u64* tM) {
    const int tid = threadIdx.x, lane = tid & 31;
    constexpr u32 kInf = 0xffffffffu;
    u64 randmask = 0;
    for (int j = 0; j < Bn; ++j) if (ps.piv[j] != kInf) randmask |= 1ull << j;
    const int nrand = __popcll(randmask);
    const u32 ntr = ps.nt;
    if (tid < Bn && ((randmask >> tid) & 1ull)) {
        ps.outc[tid] = uint8_t(counter_bit(a.seed, a.ordinal0 + (uint64_t)(pos + tid)));
        const u32 at = ntr + (u32)__popcll(randmask & ((1ull << tid) - 1ull));
        __stcg(tlist + at, ps.piv[tid]); __stcg(tM + at, 0ull);          // the pivot itself: -> +-Z_q
        atomicOr(a.tbits + (ps.piv[tid] >> 6), 1ull << (ps.piv[tid] & 63));
    }
    if (tid < 64) {       // panel-start signs of the pivot rows (A overwrites them)
        const u32 pl = ps.piv[tid];
        const u32 bal = __ballot_sync(0xffffffffu, pl != kInf && sign_bit(a.m.sgn, int(pl)));
        if (lane == 0) ps.full32[tid >> 5] = bal;
        if (tid < Bn && pl == kInf) atomicAdd(&ps.kdet, ps.dcnt[tid] + (u32)__popcll(ps.dZ[tid]));
    }
    __syncthreads();
    PanelInfo* info = a.info;
    if (tid < kPanelMax) {
        info->hist[tid] = ps.hist[tid]; info->dZ[tid] = ps.dZ[tid]; info->dcnt[tid] = ps.dcnt[tid];
        info->piv[tid] = ps.piv[tid]; info->outc[tid] = ps.outc[tid];
    }
    if (tid == 0) {
        info->randmask = randmask; info->nt = ntr + (u32)nrand; info->dmode = 1; info->osign = (u64)ps.full32[0] | ((u64)ps.full32[1] << 32);
        atomicAdd(&a.ws->n_rand, (u64)nrand); atomicAdd(&a.ws->n_det, (u64)(Bn - nrand));
        atomicAdd(&a.ws->k_rand, (u64)ps.krand); atomicAdd(&a.ws->k_det, (u64)ps.kdet);
        atomicAdd(&a.ws->waves, 1ull); atomicAdd(&a.ws->panels, 1ull);
    }
}

// F, row form (the common case: <= kRowCap rows have an x in any of the panel's columns).  The active rows
// live in REGISTERS of kRowThreads/32 warps as (row-bit, panel bits, step mask M); sequential CHP on them is then
//   pivot  = min row-bit among stabilizer rows with bit j            (scan + REDUX, one smem hop across the warps)
//   random: every other row with bit j:  bits ^= bits_p ; M |= 1<<j  ; the pivot and its old partner retire;
//           the partner's new content (the old pivot row) becomes a fresh VIRTUAL row (born at step j)
//   deterministic: partners = destabilizer rows with bit j (virtual ones stand for the +-Z rows of earlier steps)
// which yields the same schedule (pivots, histories, step masks, partner sets) as the column form below.
template <int KT>       // slots per thread actually used (1, 2 or 4): fewer slots = fewer dependent instructions per step
__device__ __noinline__ void panel_factorise_rows(const MeasArgs& a, PanelSmem& ps, int pos, int Bn, u32 A, u64* rowM, u32* tlist, u64* tM, u32 pbase) {
    const int NS = a.NS;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr u32 kInf = 0xffffffffu;
    long long tc = clock64();
#define SK_RPROF(k) do { if (a.prof && tid == 0) { const long long _c = clock64(); a.ws->cprof[k] += (u64)(_c - tc); tc = _c; } } while (0)
    if (tid < kPanelMax) { ps.piv[tid] = kInf; ps.hist[tid] = 0; ps.dZ[tid] = 0; ps.outc[tid] = 0; ps.dcnt[tid] = 0; }
    if (tid == 0) { ps.nt = 0; ps.krand = 0; ps.kdet = 0; ps.steps = 0; ps.gmin[0] = kInf; ps.gmin[1] = kInf; ps.gmin[2] = kInf; a.info->dmode = 1; }
    __syncthreads();
    u64 randmask = 0;
    // Lookahead: every finished step is published at once (pivot, history, partner list, then a release store of the
    // progress counter), so the other CTAs compute pivot values and partner products while the recurrence continues.
    // only as many warps as the rows (plus the virtual rows still to come) need take part
    const int Tact = min(kRowThreads, int(((A + kPanelMax + KT - 1) / KT + 31) & ~31u));
    // Steps are published in groups of 8: the release (a fence) is paid once per group -- and by a helper warp (the
    // last one, when the recurrence does not need it), so that the fence latency stays off the recurrence's critical path.
    const bool helper = Tact <= kMeasThreads - 32;
    int published = 0;
    auto publish = [&](int upto) {        // steps [published, upto)
        PanelInfo* info = a.info;
        for (int jj = published; jj < upto; ++jj) { info->piv[jj] = ps.piv[jj]; info->hist[jj] = ps.hist[jj]; info->dcnt[jj] = ps.dcnt[jj]; info->dZ[jj] = ps.dZ[jj]; }
        st_release(&a.ws->progress, pbase + u32(upto));
        published = upto;
    };
    if (tid < Tact) {
        // slot state in scalars (kRowK == 4), so that it stays in registers: row-bit | (born step + 1) << 24 (kInf = empty), bits, M
        static_assert(kRowK == 4, "slot macros below are written for 4 slots per thread");
        u32 hh0 = kInf, hh1 = kInf, hh2 = kInf, hh3 = kInf; u64 bb0 = 0, bb1 = 0, bb2 = 0, bb3 = 0, mm0 = 0, mm1 = 0, mm2 = 0, mm3 = 0;
#define SK_SLOTS(X) X(0, hh0, bb0, mm0) if (KT > 1) { X(1, hh1, bb1, mm1) } if (KT > 2) { X(2, hh2, bb2, mm2) X(3, hh3, bb3, mm3) }
        int Kact = int((A + Tact - 1) / Tact);
#define SK_LOAD(k, hh, bb, mm) { const u32 i = u32(k) * Tact + tid; if (i < A) { hh = __ldcg(a.alist_h + i); bb = ldcg(a.alist_b + i); } }
        SK_SLOTS(SK_LOAD)
#undef SK_LOAD
        int ntarget = 0;
        int vt = int(A % (u32)Tact), vk = int(A / (u32)Tact);      // slot (thread, k) of the next virtual row
        SK_RPROF(0);
        for (int j = 0; j < Bn; ++j) {
            // which of this thread's slots have an x in column j
            u32 hit = 0;
#define SK_HIT(k, hh, bb, mm) hit |= (u32(bb >> j) & 1u) << k;
            SK_SLOTS(SK_HIT)
#undef SK_HIT
            // pivot candidate: smallest stabilizer row-bit among the hits, carried with its bits and step mask
            u32 mymin = kInf; u64 cb = 0, cm = 0;
            if (hit) {
#define SK_SCAN(k, hh, bb, mm) if (((hit >> k) & 1u) && hh < mymin && hh < (u32)NS) { mymin = hh; cb = bb; cm = mm; }
                SK_SLOTS(SK_SCAN)
#undef SK_SCAN
            }
            const u32 wm = __reduce_min_sync(0xffffffffu, mymin);
            // the CTA-wide minimum and the warp that holds it in ONE shared word: atomicMin of (row-bit << 5 | warp); row-bits are
            // unique, so exactly one lane of the CTA ends up as the owner.  Three slots rotate (the next one is re-armed here).
            if (mymin == wm && wm != kInf) { atomicMin(&ps.gmin[j % 3], (wm << 5) | (u32)warp); ps.wbp[j & 1][warp] = cb; ps.wmp[j & 1][warp] = cm; }
            if (tid == 0) ps.gmin[(j + 1) % 3] = kInf;
            named_bar(1, Tact);
            if (tid == 0) {                                    // all warps' writes of the steps before j precede this barrier
                if (helper) { if ((j & 7) == 0) { __threadfence_block(); *(volatile int*)&ps.steps = j; } }     // the helper publishes in groups of 8
                else if (j - published >= 8) publish(j);
            }
            const u32 gm = ps.gmin[j % 3];
            const u32 p = (gm == kInf) ? kInf : (gm >> 5);
            const int tw = int(gm & 31u);
            if (p == kInf) {
                // ---------------- deterministic step: partners = destabilizer rows with an x (virtual ones stand for +-Z rows)
                if (hit) {
                    u32 dzlo = 0, dzhi = 0;
#define SK_DET(k, hh, bb, mm) if ((hit >> k) & 1u) { \
                        const u32 born = hh >> 24; \
                        if (born) { if (born <= 32) dzlo |= 1u << (born - 1); else dzhi |= 1u << (born - 33); } \
                        else { const u32 at = atomicAdd(&ps.dcnt[j], 1u); __stcg(a.dpart + (size_t)j * kRowSlots + at, hh - (u32)NS); } }
                    SK_SLOTS(SK_DET)
#undef SK_DET
                    if (dzlo | dzhi) atomicOr(&ps.dZ[j], (u64)dzlo | ((u64)dzhi << 32));
                }
                continue;
            }
            // ---------------- random step
            const u32 pd = (u32)NS + p;
            const u64 bp = ps.wbp[j & 1][tw], Mp = ps.wmp[j & 1][tw];
            const u64 above = (j < 63) ? ~((2ull << j) - 1ull) : 0ull;
            // pivot -> +-Z_q (history kept for earlier deterministic steps); others with bit j: multiplied by the pivot row
            if (hit) {
#define SK_UPD(k, hh, bb, mm) if ((hit >> k) & 1u) { \
                    if (hh == p) { __stcg(rowM + p, mm); hh = kInf; bb = 0; } \
                    else if (hh != pd) { bb ^= bp; mm |= 1ull << j; ++ntarget; } }
                SK_SLOTS(SK_UPD)
#undef SK_UPD
            }
            // the old partner row is overwritten: its past is void (it may or may not have had an x in column j)
#define SK_RET(k, hh, bb, mm) if (hh == pd) { hh = kInf; bb = 0; }
            SK_SLOTS(SK_RET)
#undef SK_RET
            if (tid == vt) {                        // ... and its new content, the old pivot row, is a fresh virtual row
#define SK_NEW(k, hh, bb, mm) if (k == vk) { hh = pd | (u32(j + 1) << 24); bb = bp & above; mm = 0; }
                SK_SLOTS(SK_NEW)
#undef SK_NEW
            }
            Kact = max(Kact, vk + 1);
            if (++vt == Tact) { vt = 0; ++vk; }
            if (tid == 0) { ps.piv[j] = p; ps.hist[j] = Mp; }
            randmask |= 1ull << j;
        }
        named_bar(1, Tact);
        if (tid == 0) { if (helper) { __threadfence_block(); *(volatile int*)&ps.steps = Bn; } else publish(Bn); }
        SK_RPROF(1);
        // emit the touched rows (regular rows that were multiplied at least once, and every virtual row)
        int cnt = 0;
#define SK_CNT(k, hh, bb, mm) if (k < Kact && hh != kInf && (mm || (hh >> 24))) ++cnt;
        SK_SLOTS(SK_CNT)
#undef SK_CNT
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) { const int t = __shfl_up_sync(0xffffffffu, incl, o); if (lane >= o) incl += t; }
        if (lane == 31) ps.wcnt[warp] = incl;
        ntarget = warp_sum(ntarget);
        if (lane == 0 && ntarget) atomicAdd(&ps.krand, (u32)ntarget);
        named_bar(1, Tact);
        u32 at = incl - cnt;
        for (int t = 0; t < warp; ++t) at += ps.wcnt[t];
#define SK_EMIT(k, hh, bb, mm) if (k < Kact && hh != kInf && (mm || (hh >> 24))) { \
                const u32 row = hh & 0xffffffu; \
                __stcg(tlist + at, row); __stcg(tM + at, mm); atomicOr(a.tbits + (row >> 6), 1ull << (row & 63)); \
                if (!(hh >> 24) && row < (u32)NS) __stcg(rowM + row, mm); \
                ++at; }
        SK_SLOTS(SK_EMIT)
#undef SK_EMIT
#undef SK_SLOTS
        if (tid == Tact - 1) ps.nt = at;
        SK_RPROF(2);
    } else if (helper && tid == kMeasThreads - 32) {
        // lock-free hand-off through ps.steps (volatile + __threadfence_block on both sides): deliberate, and the only
        // shared-memory access pattern compute-sanitizer's racecheck reports for this kernel
        while (published < Bn) {
            const int st = *(volatile int*)&ps.steps;
            if (st - published >= 8 || (st == Bn && st > published)) { __threadfence_block(); publish(st); }
            else __nanosleep(200);
        }
    }
    __syncthreads();
    SK_RPROF(3);
    panel_rows_tail(a, ps, pos, Bn, tlist, tM);
    SK_RPROF(4);
#undef SK_RPROF
}

// F, level form (the default for <= row_cap active rows).  The same symbolic elimination as the row form above, but the
// steps of a panel are not walked one by one: in every ROUND all steps whose outcome no earlier unfinished step can
// influence are executed together (a level-set / wavefront schedule of the elimination DAG).  A surface-code panel needs
// 1-2 rounds instead of 64 dependent steps (d=71: 306 rounds for 10 081 measurements).
//
// State: the active rows are joined into PAIRS (stabilizer i, destabilizer n+i) by a shared-memory hash; a pair slot
// holds the two rows' bits in the panel columns (sb, db), their step masks (Ms, Md) and `born` (step+1 that overwrote the
// destabilizer with a pivot row: from then on it stands for the +-Z row of that step).  U = unfinished steps.
// One round:
//   1  every stabilizer row offers itself as pivot candidate of its unfinished columns (atomicMin: smallest row)
//      and records what an elimination with it could touch: A_j |= (sb | db) & above(j)   (rows with more than kLevelK
//      bits do so for their lowest column only and force that column to count as a contributor, which covers the rest);
//   2  one warp, a lane per column: T_j = bits of the candidate pivot (and of its partner, which step j overwrites) above j,
//      J_j = the same below j.  A step is HARMLESS if it is ready and T_j = 0 (it changes no unfinished column).
//      ready(l)  <=>  l not in the union of A_j over the unfinished non-harmless j  (nothing can alter column l before l),
//                     J_l only holds harmless steps (the pivot row and its partner arrive at step l unchanged; those
//                     steps only add themselves to the pivot's history), and the candidate is not also the candidate
//                     of one of them.  Fixpoint over the harmless set (monotone, usually 1-2 sweeps of ballots + REDUX).
//      The lowest unfinished step is always ready, so every round makes progress.
//   3  every pair applies all ready steps at once: pivots retire (sb := 0, db := pivot bits above l, born := l+1), hit rows
//      XOR the pivots' bits and extend their step masks, deterministic steps collect their partners.
// Ready steps touch pairwise disjoint pivot rows and never flip each other's column bits, so executing them together
// equals executing them in index order; tools/proto_levels.py checks the rule against sequential elimination.
constexpr int kLevelK = 4;
__host__ __device__ inline int level_pair_cap(int NS) { return NS < kRowSlots ? NS : kRowSlots; }
__host__ __device__ inline int level_hash_size(int NS) { int h = 64; while (h < 2 * level_pair_cap(NS)) h <<= 1; return h; }
__host__ __device__ inline size_t level_smem_bytes(int NS) { return (size_t)level_pair_cap(NS) * (4 * 8 + 4 + 2) + (size_t)level_hash_size(NS) * (4 + 2) + 64; }

__device__ __forceinline__ u64 bits_above(int l) { return (l < 63) ? ~((2ull << l) - 1ull) : 0ull; }
__device__ __forceinline__ u64 bits_below(int l) { return (1ull << l) - 1ull; }
// 64-bit OR into shared memory as two native 32-bit reductions (a 64-bit shared atomic is a CAS spin loop)
__device__ __forceinline__ void smem_or64(u64* p, u64 v) {
    u32* q = reinterpret_cast<u32*>(p);
    if ((u32)v) atomicOr(q, (u32)v);
    if ((u32)(v >> 32)) atomicOr(q + 1, (u32)(v >> 32));
}
__device__ __forceinline__ u64 warp_or64(u64 v) {
    const u32 lo = __reduce_or_sync(0xffffffffu, (u32)v), hi = __reduce_or_sync(0xffffffffu, (u32)(v >> 32));
    return ((u64)hi << 32) | lo;
}

struct LevelSmem {
    u32 piv[kPanelMax], dcnt[kPanelMax], cand[kPanelMax], pslot[kPanelMax]; u64 hist[kPanelMax], dZ[kPanelMax], Aany[kPanelMax], bpA[kPanelMax];
    u64 ready, forced; u32 npairs, rounds, nt, krand, kdet; u32 wcnt[kMeasThreads / 32]; long long tacc[8];
};
// (not inlined: the function gets a register allocation of its own instead of adding to the pressure of the kernel body)
__device__ __noinline__ void panel_factorise_levels(const MeasArgs& a, int pos, int Bn, u32 A, u64* rowM, u32* tlist, u64* tM, u32 pbase) {
    const int NS = a.NS;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr u32 kInf = 0xffffffffu;
    constexpr int T = kMeasThreads;
    extern __shared__ __align__(16) u64 sp[];          // the kernel's dynamic shared memory (free in CTA 0 during F)
    __shared__ LevelSmem ps;
    const int Pc = level_pair_cap(NS), HS = level_hash_size(NS);
    u64* sb = sp; u64* db = sb + Pc; u64* Ms = db + Pc; u64* Md = Ms + Pc;
    u32* id = reinterpret_cast<u32*>(Md + Pc); u32* hkey = id + Pc;
    unsigned short* hslot = reinterpret_cast<unsigned short*>(hkey + HS);
    uint8_t* born = reinterpret_cast<uint8_t*>(hslot + HS); uint8_t* pvd = born + Pc;
    long long tc = clock64();
    if (tid < 8) ps.tacc[tid] = 0;
#define SK_LPROF(k) do { if (a.prof && tid == 0) { const long long _c = clock64(); ps.tacc[k] += _c - tc; tc = _c; } } while (0)
    // the active rows (issued first: one L2 round trip overlapped with the initialisation)
    u32 eh[kRowK]; u64 eb[kRowK];
#pragma unroll
    for (int k = 0; k < kRowK; ++k) { const u32 i = u32(k) * T + tid; eh[k] = kInf; eb[k] = 0; if (i < A) { eh[k] = __ldcg(a.alist_h + i); eb[k] = ldcg(a.alist_b + i); } }
    for (int i = tid; i < Pc; i += T) { sb[i] = 0; db[i] = 0; Ms[i] = 0; Md[i] = 0; born[i] = 0; pvd[i] = 0; }
    for (int i = tid; i < HS; i += T) hkey[i] = 0;
    if (tid < kPanelMax) { ps.piv[tid] = kInf; ps.hist[tid] = 0; ps.dZ[tid] = 0; ps.dcnt[tid] = 0; ps.cand[tid] = kInf; ps.Aany[tid] = 0; }
    if (tid == 0) { ps.nt = 0; ps.krand = 0; ps.kdet = 0; ps.npairs = 0; ps.forced = 0; ps.rounds = 0; a.info->dmode = 1; }
    __syncthreads();
    // pair join: key = stabilizer index + 1, open addressing
    u32 epos[kRowK]; bool ewon[kRowK];
#pragma unroll
    for (int k = 0; k < kRowK; ++k) {
        epos[k] = 0; ewon[k] = false;
        if (eh[k] == kInf) continue;
        const u32 pid = eh[k] < (u32)NS ? eh[k] : eh[k] - (u32)NS;
        u32 at = (pid * 2654435761u) >> 7 & u32(HS - 1);
        for (;;) {
            const u32 old = atomicCAS(&hkey[at], 0u, pid + 1u);
            if (old == 0u) { ewon[k] = true; break; }
            if (old == pid + 1u) break;
            at = (at + 1u) & u32(HS - 1);
        }
        epos[k] = at;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kRowK; ++k) if (ewon[k]) {
        const u32 slot = atomicAdd(&ps.npairs, 1u);
        hslot[epos[k]] = (unsigned short)slot; id[slot] = eh[k] < (u32)NS ? eh[k] : eh[k] - (u32)NS;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kRowK; ++k) if (eh[k] != kInf) { const u32 slot = hslot[epos[k]]; if (eh[k] < (u32)NS) sb[slot] = eb[k]; else db[slot] = eb[k]; }
    __syncthreads();
    const int P = int(ps.npairs);
    SK_LPROF(0);
    u64 U = (Bn < 64) ? ((1ull << Bn) - 1ull) : ~0ull;
    int ntarget = 0;
    bool isr[2] = {false, false}; u64 sgw[2] = {0, 0}; u32 spid[2] = {0, 0};      // warp 0: this lane's columns that turned out random
    while (U) {
        // ---- 1: pivot candidates and reach sets
        for (int s = tid; s < P; s += T) {
            const u64 sv = sb[s] & U;
            if (!sv) continue;
            const u64 all = sv | (db[s] & U);
            const u32 key = (id[s] << 11) | u32(s);
            if (__popcll(sv) > kLevelK) {
                const int low = __ffsll((long long)sv) - 1;
                atomicMin(&ps.cand[low], key); smem_or64(&ps.Aany[low], all & bits_above(low)); smem_or64(&ps.forced, 1ull << low);
            } else {
                u64 t = sv;
                while (t) {
                    const int j = __ffsll((long long)t) - 1; t &= t - 1;
                    atomicMin(&ps.cand[j], key);
                    const u64 r = all & bits_above(j);
                    smem_or64(&ps.Aany[j], r);
                }
            }
        }
        __syncthreads();
        SK_LPROF(4);
        // ---- 2: which steps are ready (warp 0; lane owns columns lane and lane + 32)
        if (warp == 0) {
            u64 Tm[2], Jm[2], Am[2], Js[2]; u32 cd[2]; bool inU[2], rnd[2], conf[2], hb[2];
            const u64 forced = ps.forced;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int j = lane + 32 * h;
                inU[h] = (U >> j) & 1ull; cd[h] = ps.cand[j]; rnd[h] = inU[h] && cd[h] != kInf;
                Tm[h] = 0; Jm[h] = 0; Am[h] = 0; Js[h] = 0; conf[h] = false;
                if (rnd[h]) {
                    const u32 slot = cd[h] & 2047u;
                    const u64 sv = sb[slot] & U, all = sv | (db[slot] & U);
                    Tm[h] = all & bits_above(j); Jm[h] = all & bits_below(j); Js[h] = sv & bits_below(j); Am[h] = ps.Aany[j];
                    u64 t = Js[h];
                    while (t) { const int j2 = __ffsll((long long)t) - 1; t &= t - 1; if (ps.cand[j2] == cd[h]) conf[h] = true; }
                }
                hb[h] = inU[h] && (!rnd[h] || (Tm[h] == 0 && !((forced >> j) & 1ull)));
            }
            u64 H = (u64)__ballot_sync(0xffffffffu, hb[0]) | ((u64)__ballot_sync(0xffffffffu, hb[1]) << 32);
            u64 acc = warp_or64(((inU[0] && !hb[0]) ? Am[0] : 0ull) | ((inU[1] && !hb[1]) ? Am[1] : 0ull));
            u64 ready;
            bool rd[2];
            for (;;) {
#pragma unroll
                for (int h = 0; h < 2; ++h) { const int j = lane + 32 * h; rd[h] = inU[h] && !((acc >> j) & 1ull) && !conf[h] && (Jm[h] & ~H) == 0; }
                ready = (u64)__ballot_sync(0xffffffffu, rd[0]) | ((u64)__ballot_sync(0xffffffffu, rd[1]) << 32);
                const u64 newH = H & ready;
                if (newH == H) break;
                const u64 drop = H & ~newH;
                acc |= warp_or64((((drop >> lane) & 1ull) ? Am[0] : 0ull) | (((drop >> (lane + 32)) & 1ull) ? Am[1] : 0ull));
                H = newH;
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int j = lane + 32 * h;
                if (!rd[h]) continue;
                if (rnd[h]) {
                    const u32 slot = cd[h] & 2047u;
                    const u64 hist = Ms[slot] | Js[h];
                    ps.pslot[j] = slot; ps.bpA[j] = sb[slot] & bits_above(j);
                    ps.piv[j] = id[slot]; ps.hist[j] = hist;
                    __stcg(rowM + id[slot], hist);
                    isr[h] = true; spid[h] = id[slot]; sgw[h] = ldcg(a.m.sgn + (id[slot] >> 6));
                } else ps.pslot[j] = kInf;
            }
            if (lane == 0) { ps.ready = ready; ps.rounds++; }
        }
        __syncthreads();
        SK_LPROF(5);
        // ---- 3: all ready steps at once
        const u64 ready = ps.ready;
        for (int s = tid; s < P; s += T) {
            const u64 sv = sb[s], dv = db[s];
            const u64 sh = sv & ready, dh = dv & ready;
            if (!(sh | dh)) continue;
            int pl = -1;
            { u64 t = sh; while (t) { const int l = __ffsll((long long)t) - 1; t &= t - 1; if (ps.pslot[l] == (u32)s) { pl = l; break; } } }
            const u32 bo = born[s];
            if (pl >= 0) {
                // pivot of step pl: the ready steps below pl multiplied this row (they are in its history) and read or
                // multiplied its old partner, which step pl then overwrites with the pivot row
                ntarget += __popcll(sh & bits_below(pl));
                u64 t = dh & bits_below(pl);
                while (t) {
                    const int l2 = __ffsll((long long)t) - 1; t &= t - 1;
                    if (ps.pslot[l2] != kInf) ++ntarget;
                    else if (bo) smem_or64(&ps.dZ[l2], 1ull << (bo - 1));
                    else { const u32 at = atomicAdd(&ps.dcnt[l2], 1u); __stcg(a.dpart + (size_t)l2 * kRowSlots + at, id[s]); }
                }
                sb[s] = 0; db[s] = sv & bits_above(pl); Ms[s] = ps.hist[pl]; Md[s] = 0; born[s] = uint8_t(pl + 1); pvd[s] = 1;
            } else {
                if (sh) {
                    u64 v = sv, t = sh;
                    while (t) { const int l = __ffsll((long long)t) - 1; t &= t - 1; v ^= ps.bpA[l]; }
                    sb[s] = v; Ms[s] |= sh; ntarget += __popcll(sh);
                }
                if (dh) {
                    u64 v = dv, t = dh, md = 0;
                    while (t) {
                        const int l = __ffsll((long long)t) - 1; t &= t - 1;
                        if (ps.pslot[l] != kInf) { v ^= ps.bpA[l]; md |= 1ull << l; ++ntarget; }
                        else if (bo) smem_or64(&ps.dZ[l], 1ull << (bo - 1));
                        else { const u32 at = atomicAdd(&ps.dcnt[l], 1u); __stcg(a.dpart + (size_t)l * kRowSlots + at, id[s]); }
                    }
                    db[s] = v; Md[s] |= md;
                }
            }
        }
        U &= ~ready;
        if (tid < kPanelMax) { ps.cand[tid] = kInf; ps.Aany[tid] = 0; }
        if (tid == 0) ps.forced = 0;
        __syncthreads();
        SK_LPROF(6);
    }
    // ---- touched rows: regular rows that were multiplied at least once, and every overwritten destabilizer
    int cnt = 0;
    for (int s = tid; s < P; s += T) { cnt += (!pvd[s] && Ms[s]) ? 1 : 0; cnt += (born[s] || Md[s]) ? 1 : 0; }
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { const int t = __shfl_up_sync(0xffffffffu, incl, o); if (lane >= o) incl += t; }
    if (lane == 31) ps.wcnt[warp] = incl;
    ntarget = warp_sum(ntarget);
    if (lane == 0 && ntarget) atomicAdd(&ps.krand, (u32)ntarget);
    if (warp == 0) {      // random steps and the panel-start signs of their pivot rows (loaded when the pivots were fixed)
        const u64 rm = (u64)__ballot_sync(0xffffffffu, isr[0]) | ((u64)__ballot_sync(0xffffffffu, isr[1]) << 32);
        const u64 os = (u64)__ballot_sync(0xffffffffu, isr[0] && ((sgw[0] >> (spid[0] & 63)) & 1ull)) | ((u64)__ballot_sync(0xffffffffu, isr[1] && ((sgw[1] >> (spid[1] & 63)) & 1ull)) << 32);
        if (lane == 0) { ps.ready = rm; ps.forced = os; }
    }
    __syncthreads();
    u32 at = incl - cnt, ntr = 0;
    for (int t = 0; t < T / 32; ++t) { const u32 c = ps.wcnt[t]; if (t < warp) at += c; ntr += c; }
    for (int s = tid; s < P; s += T) {
        const u32 pid = id[s];
        if (!pvd[s] && Ms[s]) {
            __stcg(tlist + at, pid); __stcg(tM + at, Ms[s]); atomicOr(a.tbits + (pid >> 6), 1ull << (pid & 63)); __stcg(rowM + pid, Ms[s]); ++at;
        }
        if (born[s] || Md[s]) {
            const u32 row = (u32)NS + pid;
            __stcg(tlist + at, row); __stcg(tM + at, Md[s]); atomicOr(a.tbits + (row >> 6), 1ull << (row & 63)); ++at;
        }
    }
    const u64 randmask = ps.ready, osign = ps.forced;
    const int nrand = __popcll(randmask);
    PanelInfo* info = a.info;
    if (tid < kPanelMax) {
        uint8_t oc = 0;
        if (tid < Bn) {
            if ((randmask >> tid) & 1ull) {       // the pivot itself joins the touched rows: -> +-Z_q with the counter RNG bit
                oc = uint8_t(counter_bit(a.seed, a.ordinal0 + (uint64_t)(pos + tid)));
                const u32 pt = ntr + (u32)__popcll(randmask & ((1ull << tid) - 1ull));
                __stcg(tlist + pt, ps.piv[tid]); __stcg(tM + pt, 0ull);
                atomicOr(a.tbits + (ps.piv[tid] >> 6), 1ull << (ps.piv[tid] & 63));
            } else atomicAdd(&ps.kdet, ps.dcnt[tid] + (u32)__popcll(ps.dZ[tid]));
        }
        info->hist[tid] = ps.hist[tid]; info->dZ[tid] = ps.dZ[tid]; info->dcnt[tid] = ps.dcnt[tid];
        info->piv[tid] = ps.piv[tid]; info->outc[tid] = oc;
    }
    if (tid == 64) { info->randmask = randmask; info->nt = ntr + (u32)nrand; info->dmode = 1; info->osign = osign; }
    SK_LPROF(2);
    __syncthreads();
    if (tid == 0) {
        st_release(&a.ws->progress, pbase + u32(Bn));         // everything is published at once (cumulative over the barrier)
        atomicAdd(&a.ws->n_rand, (u64)nrand); atomicAdd(&a.ws->n_det, (u64)(Bn - nrand));
        atomicAdd(&a.ws->k_rand, (u64)ps.krand); atomicAdd(&a.ws->k_det, (u64)ps.kdet);
        atomicAdd(&a.ws->waves, 1ull); atomicAdd(&a.ws->panels, 1ull);
    }
    SK_LPROF(3);
    if (a.prof && tid == 0) { a.ws->cprof[10] += ps.rounds; for (int k = 0; k < 7; ++k) atomicAdd(&a.ws->cprof[k], (u64)ps.tacc[k]); }
#undef SK_LPROF
}

// F: symbolic factorisation of one panel by CTA 0 (see the file header).
// Shared-memory panel: column j = words [j*CS, j*CS + RW] with CS = RW + 2; word RW holds the VIRTUAL rows:
// when random step l overwrites destabilizer p_l + n with the old pivot row, the old row-bit is retired and
// the new content lives on as virtual row l (bit l of word RW), so overwritten rows need no special casing:
// retired bits (pivots, which become +-Z_q and never carry an x again, and their old partners) are masked off.
// Left-looking elimination: column j is brought up to date only when step j needs it,
//   cur_j = (orig_j ^ XOR_{l in S_j} m_l) & ~retired,   S_j = earlier random steps whose pivot row has an x
// in column j (S_j bit l = pw_l bit j; the virtual word starts as S_j itself), sparse in the word index
// through nzm.  m_l = column l at step l minus the pivot and its partner = the rows step l multiplies.
__device__ __noinline__ void panel_factorise(const MeasArgs& a, u64* sp, PanelSmem& ps, u32* s_rows, u64* mbar, u32& tma_parity, int pos, int Bn, u64* rowM, u32* tlist, u64* tM, u32 pbase) {
    const int RW = a.m.RW, W = a.m.W, NS = a.NS;
    const int CS = RW + 2, RV = RW + 1;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    u64* nzm = sp + (size_t)Bn * CS;            // [RV] steps l whose frozen mask has a non-zero word here
    u64* ret = nzm + RV;                        // [RV] retired row-bits
    u64 tf = a.prof ? gtime() : 0;
#define SK_FPROF(k) do { if (a.prof && tid == 0) { u64 _n = gtime(); a.ws->fprof[k] += _n - tf; tf = _n; } } while (0)
    // the gathered panel arrives by TMA bulk copies (UBLKCP), one per column, on one mbarrier
    if (warp == 0) {
        asm volatile("fence.proxy.async;" ::: "memory");
        if (lane == 0) mbar_expect_tx(mbar, u32(Bn * RW * 8));
        for (int j = lane; j < Bn; j += 32) tma_load_1d(sp + (size_t)j * CS, a.pan + (size_t)j * RW, u32(RW * 8), mbar);
    }
    for (int w = tid; w < 2 * RV; w += kMeasThreads) nzm[w] = 0;      // nzm | ret are contiguous
    if (tid < Bn) { sp[(size_t)tid * CS + RW] = 0; sp[(size_t)tid * CS + RW + 1] = 0; }
    if (tid < kPanelMax) { ps.piv[tid] = 0xffffffffu; ps.hist[tid] = 0; ps.pw[tid] = 0; ps.dZ[tid] = 0; ps.outc[tid] = 0; }
    if (tid == 0) { ps.nt = 0; ps.krand = 0; ps.kdet = 0; }
    if (!mbar_wait(mbar, tma_parity)) { if (tid == 0) atomicOr(&a.ws->err, 0x40000000u); }
    tma_parity ^= 1;
    __syncthreads();
    SK_FPROF(0);
    // ---- control warp: the serial recurrence lives on the STABILIZER half only (pivots, pivot-row bits pw, histories);
    // warp-synchronous, no CTA barriers.  Lane owns words lane, lane+32, ...
    long long cp[6] = {0, 0, 0, 0, 0, 0};
    if (warp == 0) {
        u64 randmask = 0;
        for (int j = 0; j < Bn; ++j) {
            const long long c0 = clock64();
            u64* cj = sp + (size_t)j * CS;
            // S_j: lane l holds pw of steps l and l+32
            const u64 a0 = (lane < j) ? ps.pw[lane] : 0ull, a1 = (lane + 32 < j) ? ps.pw[lane + 32] : 0ull;
            const u64 S = (u64)__ballot_sync(0xffffffffu, (a0 >> j) & 1ull) | ((u64)__ballot_sync(0xffffffffu, (a1 >> j) & 1ull) << 32);
            u32 cand = 0xffffffffu;
            u64 nzw = 0;                 // which of this lane's words are non-zero in the materialised column
            int k = 0;
            for (int w0 = 0; w0 < W; w0 += 32, ++k) {
                const int w = w0 + lane;
                const bool valid = w < W;
                const u64 old = valid ? cj[w] : 0ull;
                u64 cur = old;
                const u64 bits = valid ? (S & nzm[w]) : 0ull;
                const int nb = __popcll(bits);
                if (nb && nb <= 3) { u64 b = bits; while (b) { const int l = __ffsll((long long)b) - 1; b &= b - 1; cur ^= sp[(size_t)l * CS + w]; } }
                // hot words (the same rows are targets again and again): the whole warp reduces one word at a time,
                // lane l loading the masks of steps l and l+32; 32-bit halves combined with REDUX
                u32 hot = __ballot_sync(0xffffffffu, nb > 3);
                while (hot) {
                    const int src = __ffs(hot) - 1; hot &= hot - 1;
                    const u64 sb = __shfl_sync(0xffffffffu, bits, src);
                    const int ws = w0 + src;
                    u64 x = 0;
                    if ((sb >> lane) & 1ull) x ^= sp[(size_t)lane * CS + ws];
                    if ((sb >> (lane + 32)) & 1ull) x ^= sp[(size_t)(lane + 32) * CS + ws];
                    const u32 lo = __reduce_xor_sync(0xffffffffu, (u32)x), hi = __reduce_xor_sync(0xffffffffu, (u32)(x >> 32));
                    if (lane == src) cur ^= (u64)lo | ((u64)hi << 32);
                }
                if (valid) {
                    cur &= ~ret[w];
                    if (cur != old) cj[w] = cur;
                    if (cur) { if (k < 64) nzw |= 1ull << k; if (cand == 0xffffffffu) cand = u32(w * 64 + __ffsll((long long)cur) - 1); }   // words ascend with k
                }
            }
            const u32 p = __reduce_min_sync(0xffffffffu, cand);
            if (lane == 0) ps.S[j] = S;
            const long long c1 = clock64();
            if (p != 0xffffffffu) {
                // ---------------- random step
                __syncwarp();         // the materialised column is visible to the bit gather
                const u32 b0 = (lane < Bn) ? u32((sp[(size_t)lane * CS + (p >> 6)] >> (p & 63)) & 1ull) : 0u;
                const u32 b1 = (lane + 32 < Bn) ? u32((sp[(size_t)(lane + 32) * CS + (p >> 6)] >> (p & 63)) & 1ull) : 0u;
                // bit p of every panel column: frozen masks for c < j (history), panel-start bits for c > j
                const u64 full = (u64)__ballot_sync(0xffffffffu, b0) | ((u64)__ballot_sync(0xffffffffu, b1) << 32);
                const u64 above = (j < 63) ? ~((2ull << j) - 1ull) : 0ull;
                const u64 hist = full & randmask & ((1ull << j) - 1ull);
                // x bits of the pivot row at the later columns = its panel-start bits ^ those of the pivot rows multiplied into it
                u64 x = 0;
                if ((hist >> lane) & 1ull) x ^= ps.pw[lane];
                if ((hist >> (lane + 32)) & 1ull) x ^= ps.pw[lane + 32];
                const u32 lo = __reduce_xor_sync(0xffffffffu, (u32)x), hi = __reduce_xor_sync(0xffffffffu, (u32)(x >> 32));
                const u64 pw = (full ^ ((u64)lo | ((u64)hi << 32))) & above;
                const long long c2 = clock64();
                // freeze m_j (stabilizer half): the pivot is not multiplied into itself; its row-bit retires
                k = 0;
                for (int w0 = 0; w0 < W; w0 += 32, ++k) {
                    const int w = w0 + lane;
                    if (k < 64 ? !((nzw >> k) & 1ull) : (w >= W || cj[w] == 0)) continue;     // (beyond 2048 words per half: re-read)
                    if (w == int(p >> 6)) {
                        const u64 bit = 1ull << (p & 63);
                        const u64 m = cj[w] & ~bit;
                        cj[w] = m; ret[w] |= bit;
                        if (!m) continue;
                    }
                    nzm[w] |= 1ull << j;
                }
                if (lane == 0) { ps.piv[j] = p; ps.hist[j] = hist; ps.pw[j] = pw; }
                randmask |= 1ull << j;
                { const long long c3 = clock64(); cp[0] += c1 - c0; cp[1] += c2 - c1; cp[2] += c3 - c2; }
            } else {
                { const long long c3 = clock64(); cp[3] += c1 - c0; cp[5] += c3 - c1; }
            }
            __syncwarp();
        }
    }
    if (a.prof && tid == 0) for (int k = 0; k < 6; ++k) a.ws->cprof[k] += (u64)cp[k];
    __syncthreads();
    SK_FPROF(1);
    // ---- destabilizer half + virtual word: they never influence the recurrence, so every word replays the B steps
    // on its own (thread per word, no synchronisation): same materialise / freeze rule with S_j and p_j from above
    for (int w = W + tid; w < RV; w += kMeasThreads) {
        u64 nz = 0, rt = 0;
        for (int j = 0; j < Bn; ++j) {
            const u64 S = ps.S[j];
            const u32 p = ps.piv[j];
            u64* cj = sp + (size_t)j * CS;
            const u64 old = cj[w];
            u64 cur = (w == RW) ? S : old;
            u64 bits = S & nz;
            while (bits) { const int l = __ffsll((long long)bits) - 1; bits &= bits - 1; cur ^= sp[(size_t)l * CS + w]; }
            cur &= ~rt;
            if (p != 0xffffffffu) {
                const u32 pd = u32(NS) + p;
                if (w == int(pd >> 6)) { const u64 bit = 1ull << (pd & 63); cur &= ~bit; rt |= bit; }
                if (cur) nz |= 1ull << j;
            }
            if (cur != old) cj[w] = cur;
        }
        nzm[w] = nz; ret[w] = rt;
    }
    __syncthreads();
    SK_FPROF(2);
    u64 randmask;
    randmask = 0;
    for (int j = 0; j < Bn; ++j) if (ps.piv[j] != 0xffffffffu) randmask |= 1ull << j;
    const int nrand = __popcll(randmask);
    long long tc0 = clock64();
#define SK_TPROF(k) do { if (a.prof && tid == 0) { const long long _c = clock64(); a.ws->cprof[k] += (u64)(_c - tc0); tc0 = _c; } } while (0)
    if (tid < Bn && ((randmask >> tid) & 1ull)) ps.outc[tid] = uint8_t(counter_bit(a.seed, a.ordinal0 + (uint64_t)(pos + tid)));
    // regular touched rows: targets of any random step that were not retired later
    int kr = 0;
    for (int w0 = 0; w0 < RV; w0 += kMeasThreads) {
        const int w = w0 + tid;
        u64 tw = 0;
        if (w < RV) {
            const u64 nz = nzm[w];
            if (nz) {
                const u64* col = sp + w;
                u64 bits = nz;
                for (int l0 = 0; l0 < Bn; l0 += 8, col += 8 * (size_t)CS, bits >>= 8) {
                    if ((bits & 0xffull) == 0) continue;
                    u64 v[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) v[u] = (l0 + u < Bn && ((bits >> u) & 1ull)) ? col[(size_t)u * CS] : 0ull;
#pragma unroll
                    for (int u = 0; u < 8; ++u) { tw |= v[u]; kr += __popcll(v[u]); }
                }
            }
            tw = (w < RW) ? (tw & ~ret[w]) : 0ull;        // virtual rows are listed with the overwritten destabilizers below
        }
        const int pc = __popcll(tw);
        int incl = pc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) { const int v = __shfl_up_sync(0xffffffffu, incl, o); if (lane >= o) incl += v; }
        u32 base = 0;
        if (lane == 31 && incl) base = atomicAdd(&ps.nt, (u32)incl);
        base = __shfl_sync(0xffffffffu, base, 31);
        u32 ti = base + incl - pc;
        while (tw) {
            const int b = __ffsll((long long)tw) - 1; tw &= tw - 1;
            const u32 h = u32(w * 64 + b);
            if (ti < (u32)kMaxTargets) s_rows[ti] = h;
            __stcg(tlist + ti, h); atomicOr(a.tbits + (h >> 6), 1ull << (h & 63));
            ++ti;
        }
    }
    kr = warp_sum(kr);
    if (lane == 0 && kr) atomicAdd(&ps.krand, (u32)kr);
    SK_TPROF(6);
    // deterministic steps: partner sets for phase D (real destabilizer words -> panel-start stabilizers; virtual word -> +-Z rows)
    for (int j = warp; j < Bn; j += kMeasWarps)
        if (!((randmask >> j) & 1ull)) {
            int kd = 0;
            for (int w = lane; w < W; w += 32) { const u64 v = sp[(size_t)j * CS + W + w]; kd += __popcll(v); __stcg(a.pan + (size_t)j * RW + W + w, v); }
            kd = warp_sum(kd);
            if (lane == 0) { const u64 z = sp[(size_t)j * CS + RW] & randmask; ps.dZ[j] = z; atomicAdd(&ps.kdet, (u32)(kd + __popcll(z))); }
        }
    if (tid < 64) {       // panel-start signs of the pivot rows (A overwrites them)
        const u32 pl = ps.piv[tid];
        const u32 bal = __ballot_sync(0xffffffffu, pl != 0xffffffffu && sign_bit(a.m.sgn, int(pl)));
        if (lane == 0) ps.full32[tid >> 5] = bal;
    }
    __syncthreads();
    SK_TPROF(7);
    // step masks M_h of the regular rows: a lane per row sweeps the random steps, 8 loads in flight
    const u32 ntr = ps.nt;
    if (a.prof && tid == 0) { a.ws->cprof[4] += ntr; a.ws->cprof[12] += ps.krand; }
    for (u32 i = tid; i < ntr; i += kMeasThreads) {
        const u32 h = (i < (u32)kMaxTargets) ? s_rows[i] : __ldcg(tlist + i);
        const u64* col = sp + (h >> 6);
        const int sh = int(h & 63);
        u64 M = 0, bits = randmask;
        for (int l0 = 0; l0 < Bn; l0 += 8, col += 8 * (size_t)CS, bits >>= 8) {
            if ((bits & 0xffull) == 0) continue;
            u64 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = (l0 + u < Bn) ? col[(size_t)u * CS] : 0ull;
#pragma unroll
            for (int u = 0; u < 8; ++u) M |= ((v[u] >> sh) & (bits >> u) & 1ull) << (l0 + u);
        }
        __stcg(tM + i, M); __stcg(rowM + h, M);
    }
    SK_TPROF(14);
    // the two rows every random step l overwrites: pivot p_l (-> +-Z_q) and partner p_l + n (-> P_l', then the steps
    // that multiply virtual row l)
    if (tid < 64 && ((randmask >> tid) & 1ull)) {
        const int l = tid;
        const u32 pl = ps.piv[l];
        u64 Mv = 0;
        const u64* col = sp + RW;
        for (int c0 = 0; c0 < Bn; c0 += 8, col += 8 * (size_t)CS) {
            u64 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = (c0 + u < Bn) ? col[(size_t)u * CS] : 0ull;
#pragma unroll
            for (int u = 0; u < 8; ++u) Mv |= ((v[u] >> l) & 1ull) << (c0 + u);
        }
        Mv &= randmask & ((l < 63) ? ~((2ull << l) - 1ull) : 0ull);
        const u32 at = ntr + 2u * (u32)__popcll(randmask & ((1ull << l) - 1ull));
        __stcg(tlist + at, pl); __stcg(tM + at, 0ull);
        __stcg(rowM + pl, ps.hist[l]);     // a deterministic step before l may still have row p_l as a partner
        __stcg(tlist + at + 1, u32(NS) + pl); __stcg(tM + at + 1, Mv);
        atomicOr(a.tbits + (pl >> 6), 1ull << (pl & 63)); atomicOr(a.tbits + ((u32(NS) + pl) >> 6), 1ull << ((u32(NS) + pl) & 63));
    }
    PanelInfo* info = a.info;
    if (tid < kPanelMax) {
        info->hist[tid] = ps.hist[tid]; info->dZ[tid] = ps.dZ[tid];
        info->piv[tid] = ps.piv[tid]; info->outc[tid] = ps.outc[tid];
    }
    if (tid == 0) {
        info->randmask = randmask; info->nt = ntr + 2u * (u32)nrand; info->dmode = 0; info->osign = (u64)ps.full32[0] | ((u64)ps.full32[1] << 32);
        atomicAdd(&a.ws->n_rand, (u64)nrand); atomicAdd(&a.ws->n_det, (u64)(Bn - nrand));
        atomicAdd(&a.ws->k_rand, (u64)ps.krand); atomicAdd(&a.ws->k_det, (u64)ps.kdet);
        atomicAdd(&a.ws->waves, 1ull); atomicAdd(&a.ws->panels, 1ull);
    }
    SK_TPROF(15);
#undef SK_TPROF
    __syncthreads();
    if (tid == 0) { __threadfence(); st_release(&a.ws->progress, pbase + u32(Bn)); }      // column form: everything is published at the end
    SK_FPROF(3);
#undef SK_FPROF
}


// Product of the listed rows (R layout) with the running product in REGISTERS: every lane owns NWL lane-strided words and the
// words of two rows are in flight together, so a short list costs one L2 round trip instead of one per word chunk.
// Returns this lane's share of the i-exponent (row signs not included).
template <int NWL, int ROWS = 2>      // ROWS = partner rows in flight (2, or 1 where registers are scarce)
__device__ __forceinline__ int warp_mul_wide(const u64* __restrict__ base, int W, int Wp, const u32* list, int cnt, int lane) {
    u64 ax[NWL], az[NWL];
#pragma unroll
    for (int k = 0; k < NWL; ++k) { ax[k] = 0; az[k] = 0; }
    int e = 0;
    if (ROWS == 1) {
        for (int i0 = 0; i0 < cnt; ++i0) {
            const u64* r0 = base + (size_t)(2 * list[i0]) * Wp;
            u64 x0[NWL], z0[NWL];
#pragma unroll
            for (int k = 0; k < NWL; ++k) { const int w = lane + 32 * k; const bool ok = w < W; x0[k] = ok ? ldcg(r0 + w) : 0ull; z0[k] = ok ? ldcg(r0 + Wp + w) : 0ull; }
#pragma unroll
            for (int k = 0; k < NWL; ++k) { e += g_word(x0[k], z0[k], ax[k], az[k]); ax[k] ^= x0[k]; az[k] ^= z0[k]; }
        }
        return e;
    }
    for (int i0 = 0; i0 < cnt; i0 += 2) {
        const bool two = i0 + 1 < cnt;
        const u64* r0 = base + (size_t)(2 * list[i0]) * Wp;
        const u64* r1 = base + (size_t)(2 * list[two ? i0 + 1 : i0]) * Wp;
        u64 x0[NWL], z0[NWL], x1[NWL], z1[NWL];
#pragma unroll
        for (int k = 0; k < NWL; ++k) {
            const int w = lane + 32 * k;
            const bool ok = w < W;
            x0[k] = ok ? ldcg(r0 + w) : 0ull; z0[k] = ok ? ldcg(r0 + Wp + w) : 0ull;
            x1[k] = (ok && two) ? ldcg(r1 + w) : 0ull; z1[k] = (ok && two) ? ldcg(r1 + Wp + w) : 0ull;
        }
#pragma unroll
        for (int k = 0; k < NWL; ++k) {
            e += g_word(x0[k], z0[k], ax[k], az[k]); ax[k] ^= x0[k]; az[k] ^= z0[k];
            e += g_word(x1[k], z1[k], ax[k], az[k]); ax[k] ^= x1[k]; az[k] ^= z1[k];
        }
    }
    return e;
}

// Wave mode, this warp's slots of the window [pos, wend): K2 pivot search over the stabilizer half of the C column and -- when it
// is empty -- K4, the product of the partner stabilizers (destabilizer half of the same column -> rows of the R form).
// Results per slot go to recj/recn (measurement index or -1, partner count | odd-phase flag << 30); products with more than
// kWarpList partners are left to the whole CTA (slot pushed to heavy[]).
__device__ __noinline__ void wave_slots(const MeasArgs& a, int pos, int wend, u32 wave, int gw, int GW, u32* wlist, int* nheavy, int* heavy,
                                        int* recj, int* recn, u64* acc_x, u64* acc_z) {
    const int lane = threadIdx.x & 31;
    const int W = a.m.W, Wp = a.m.Wp, RW = a.m.RW;
    const int nwl = (W + 31) / 32;
    if (lane < kSlotsPerWarp) recj[lane] = -1;
    u32* r0slot = &a.ws->r0[wave % 3];
    __syncwarp();
    int rec = 0;
    const bool trc = a.prof && lane == 0 && (gw == 0 || gw == GW / 2) && pos == 0;
    const int tb = (gw == 0) ? 0 : 96;
#define WV_TRACE(ev) do { if (trc && rec < 3) a.ws->trace[tb + rec * 8 + (ev)] = gtime(); } while (0)
    for (int slot = gw; pos + slot < wend; slot += GW, ++rec) {
        const int j = pos + slot;
        WV_TRACE(0);
        const u64* xcol = a.m.cols + (size_t)(2 * a.qubits[j]) * RW;
        u32 piv = 0xffffffffu;
        int npart = 0;
        for (int w0 = 0; w0 < W; w0 += 32 * kColChunk) {        // both halves of the column in one round trip per chunk
            u64 sv[kColChunk], dv[kColChunk];
#pragma unroll
            for (int t = 0; t < kColChunk; ++t) { const int w = w0 + 32 * t + lane; sv[t] = (w < W) ? ldcg(xcol + w) : 0ull; dv[t] = (w < W) ? ldcg(xcol + W + w) : 0ull; }
            int mine = 0;
#pragma unroll
            for (int t = 0; t < kColChunk; ++t) {
                const int w = w0 + 32 * t + lane;
                if (sv[t]) piv = min(piv, u32(w * 64 + __ffsll((long long)sv[t]) - 1));
                mine += __popcll(dv[t]);
            }
            // partner list: exclusive prefix of the lanes' counts
            int incl = mine;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) { const int v = __shfl_up_sync(0xffffffffu, incl, o); if (lane >= o) incl += v; }
            int ti = npart + incl - mine;
            npart += __shfl_sync(0xffffffffu, incl, 31);
#pragma unroll
            for (int t = 0; t < kColChunk; ++t) {
                const int w = w0 + 32 * t + lane;
                u64 v = dv[t];
                while (v) { const int b = __ffsll((long long)v) - 1; v &= v - 1; if (ti < kWarpList) wlist[ti] = u32(w * 64 + b); ++ti; }
            }
        }
        piv = warp_min(piv);
        __syncwarp();
        WV_TRACE(1);
        if (piv != 0xffffffffu) {       // random: the first one of the window ends the deterministic prefix
            if (lane == 0) atomicMax(r0slot, ~(u32)j);      // stored inverted: zero-initialised, max = smallest index
            continue;
        }
        if (npart > kWarpList) {                  // tree-reduced by the whole CTA
            if (lane == 0) { const int h = atomicAdd(nheavy, 1); heavy[h] = slot; }
            continue;
        }
        int e;
        constexpr int RIF = 2;
        if (nwl <= 1) e = warp_mul_wide<1, RIF>(a.m.rows, W, Wp, wlist, npart, lane);
        else if (nwl <= 2) e = warp_mul_wide<2, RIF>(a.m.rows, W, Wp, wlist, npart, lane);
        else if (nwl <= 4) e = warp_mul_wide<4, RIF>(a.m.rows, W, Wp, wlist, npart, lane);
        else if (nwl <= 6) e = warp_mul_wide<6, RIF>(a.m.rows, W, Wp, wlist, npart, lane);
        else {
            for (int w = lane; w < Wp; w += 32) { acc_x[w] = 0; acc_z[w] = 0; }
            e = warp_mul_list(a.m.rows, W, Wp, wlist, npart, acc_x, acc_z, lane);
        }
        WV_TRACE(2);
        for (int i = lane; i < npart; i += 32) e += 2 * sign_bit(a.m.sgn, int(wlist[i]));
        e = warp_sum(e) & 3;
        WV_TRACE(3);
        if (lane == 0) {
            a.outcomes[j] = uint8_t(e >> 1); a.dets[j] = 1;
            if (rec < kSlotsPerWarp) { recj[rec] = j; recn[rec] = npart | ((e & 1) << 30); }
        }
        __syncwarp();
    }
}


// Wave mode as two kernels of their own (launched in front of k_measure_block for long measurement blocks): ordinary grids with
// one warp per pending measurement instead of the one-CTA-per-SM cooperative grid whose warps walk three slots each, so the
// deterministic rounds of a memory experiment are two short passes -- and, being split by the FORM they read, they leave the
// critical path:
//   k_wave_cols  reads only the gate (C) form: pivot search on the stabilizer half of each measured x column, partner list from
//                the destabilizer half (written to a.wl), the stabilizer signs copied to a.wsgn.  Shares a launch with the
//                C -> R transposition, which reads the same columns (k_transpose_wave).
//   k_wave_rows  reads only the row (R) form, the lists and the sign copy: the partner products and the outcomes.  Nothing the
//                next run of gate layers writes (C form, live signs), so it runs on the side stream UNDER those layers.
// Speculative like the in-kernel wave: k_wave_cols evaluates every slot and its last CTA leaves in ws->wpos where k_measure_block
// has to start: at the end of the block when no measurement was random or too long for a warp (k_measure_block then exits at once
// and k_wave_rows owns the block); otherwise at 0 when the two overlap (`pipe`: k_wave_rows then does nothing, the cooperative
// kernel is about to change rows) or at the first such measurement when they run in order (k_wave_rows does the prefix).
constexpr int kWaveThreads = 256;
// CTA `cta` of `nctas` (any grid shape)
__device__ __forceinline__ void wave_cols_body(const MeasArgs& a, int wend, int pipe, int cta, int nctas) {
    __shared__ int s_last;
    MeasWs* ws = a.ws;
    const int tid = threadIdx.x, lane = tid & 31;
    const int W = a.m.W, RW = a.m.RW;
    const int nwl = (W + 31) / 32;
    const int GW = nctas * (kWaveThreads / 32);
    if (cta == 0) for (int w = tid; w < W; w += kWaveThreads) a.wsgn[w] = ldcg(a.m.sgn + w);
    for (int j = cta * (kWaveThreads / 32) + (tid >> 5); j < wend; j += GW) {
        const u64* xcol = a.m.cols + (size_t)(2 * a.qubits[j]) * RW;
        u32* wl = a.wl + (size_t)j * kWarpList;
        u32 piv = 0xffffffffu;
        int npart = 0;
        for (int w0 = 0; w0 < W; w0 += 32 * kColChunk) {        // both halves of the column in one round trip per chunk
            u64 sv[kColChunk], dv[kColChunk];
#pragma unroll
            for (int t = 0; t < kColChunk; ++t) { const int w = w0 + 32 * t + lane; sv[t] = (w < W) ? ldcg(xcol + w) : 0ull; dv[t] = (w < W) ? ldcg(xcol + W + w) : 0ull; }
            int mine = 0;
#pragma unroll
            for (int t = 0; t < kColChunk; ++t) {
                const int w = w0 + 32 * t + lane;
                if (sv[t]) piv = min(piv, u32(w * 64 + __ffsll((long long)sv[t]) - 1));
                mine += __popcll(dv[t]);
            }
            int incl = mine;                                    // partner list: exclusive prefix of the lanes' counts
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) { const int v = __shfl_up_sync(0xffffffffu, incl, o); if (lane >= o) incl += v; }
            int ti = npart + incl - mine;
            npart += __shfl_sync(0xffffffffu, incl, 31);
#pragma unroll
            for (int t = 0; t < kColChunk; ++t) {
                const int w = w0 + 32 * t + lane;
                u64 v = dv[t];
                while (v) { const int b = __ffsll((long long)v) - 1; v &= v - 1; if (ti < kWarpList) wl[ti] = u32(w * 64 + b); ++ti; }
            }
        }
        piv = warp_min(piv);
        if (lane == 0) {
            const bool hard = piv != 0xffffffffu || npart > kWarpList || nwl > 6;
            if (hard) atomicMax(&ws->r0[3], ~(u32)j);           // stored inverted: zero-initialised, max = smallest index
            a.wpiv[j] = hard ? 0x80000000u : u32(npart);
        }
    }
    __syncthreads();
    if (tid == 0) { __threadfence(); s_last = atomicAdd(&ws->wdone, 1u) == u32(nctas) - 1 ? 1 : 0; }
    __syncthreads();
    if (!s_last || tid) return;
    __threadfence();
    const u32 r0 = ~__ldcg(&ws->r0[3]);
    ws->wpos = (r0 == 0xffffffffu) ? u32(wend) : (pipe ? 0u : r0);
    ws->r0[3] = 0u; ws->wdone = 0u;
}

__global__ void __launch_bounds__(kWaveThreads, 4)
k_wave_cols(const __grid_constant__ MeasArgs a, int wend, int pipe) { wave_cols_body(a, wend, pipe, blockIdx.x, gridDim.x); }

// The C -> R transposition (x and z halves: planes 1 and 2 of the grid) and k_wave_cols (plane 0, scheduled first: its chains of
// dependent loads are the longer ones) as ONE launch: both only read the gate form, so they share the machine instead of a place
// each on the critical path of a round.
__global__ void __launch_bounds__(256, 4)
k_transpose_wave(const u32* __restrict__ src, size_t src_stride, int src_rows, int src_words,
                 u32* __restrict__ dst, size_t dst_stride, int dst_rows, int dst_words,
                 size_t src_zoff, size_t dst_zoff, const __grid_constant__ MeasArgs a, int wend, int pipe) {
    __shared__ __align__(16) u32 tin[kTrSmemWords];
    pdl_trigger();
    pdl_wait();
    if (blockIdx.z == 0) { wave_cols_body(a, wend, pipe, blockIdx.y * gridDim.x + blockIdx.x, gridDim.x * gridDim.y); return; }
    const int z = blockIdx.z - 1;
    transpose_tile_regs(src + (size_t)z * src_zoff, src_stride, src_rows, src_words, dst + (size_t)z * dst_zoff, dst_stride, dst_rows, dst_words,
                        blockIdx.x, blockIdx.y, tin);
}

__global__ void __launch_bounds__(kWaveThreads, 4)
k_wave_rows(const __grid_constant__ MeasArgs a, int wend) {
    __shared__ u32 s_wlist[kWaveThreads / 32][kWarpList];
    __shared__ int s_last;
    __shared__ unsigned long long s_kd;
    __shared__ u32 s_odd;
    MeasWs* ws = a.ws;
    wend = int(__ldcg(&ws->wpos));                            // deterministic prefix; 0: the cooperative kernel owns this block
    if (wend == 0) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int W = a.m.W, Wp = a.m.Wp;
    const int nwl = (W + 31) / 32;
    const int GW = gridDim.x * (kWaveThreads / 32);
    u32* wlist = s_wlist[warp];
    unsigned long long kd = 0; u32 odd = 0;
    for (int j = blockIdx.x * (kWaveThreads / 32) + warp; j < wend; j += GW) {
        const int npart = int(__ldcg(a.wpiv + j));
        const u32* wl = a.wl + (size_t)j * kWarpList;
        for (int i = lane; i < npart; i += 32) wlist[i] = __ldcg(wl + i);
        __syncwarp();
        int e;
        if (nwl <= 1) e = warp_mul_wide<1, 1>(a.m.rows, W, Wp, wlist, npart, lane);
        else if (nwl <= 2) e = warp_mul_wide<2, 1>(a.m.rows, W, Wp, wlist, npart, lane);
        else if (nwl <= 4) e = warp_mul_wide<4, 1>(a.m.rows, W, Wp, wlist, npart, lane);
        else e = warp_mul_wide<6, 1>(a.m.rows, W, Wp, wlist, npart, lane);
        for (int i = lane; i < npart; i += 32) e += 2 * sign_bit(a.wsgn, int(wlist[i]));
        e = warp_sum(e) & 3;
        if (lane == 0) { a.outcomes[j] = uint8_t(e >> 1); a.dets[j] = 1; kd += (unsigned long long)npart; odd |= u32(e & 1); }
        __syncwarp();
    }
    if (tid == 0) { s_kd = 0; s_odd = 0; }
    __syncthreads();
    if (lane == 0) { if (kd) atomicAdd(&s_kd, kd); if (odd) atomicOr(&s_odd, 1u); }
    __syncthreads();
    if (tid) return;
    if (s_kd) atomicAdd(&ws->k_det, (u64)s_kd);
    if (s_odd) atomicOr(&ws->err, 1u);
    __threadfence();
    if (atomicAdd(&ws->wdone, 1u) == gridDim.x - 1) { atomicAdd(&ws->n_det, (u64)wend); atomicAdd(&ws->waves, 1ull); ws->wdone = 0u; }
}

}  // namespace skd
#include "kernels_panel.cuh"
namespace skd {

// dynamic smem (u64): max( acc[kMeasWarps][2*Wp] + values scratch, panel [B][RW] + pivmask [W] )
__global__ void __launch_bounds__(kMeasThreads, 1)
k_measure_block(const __grid_constant__ MeasArgs a) {
    // the wave kernels own the whole block (every deterministic round of a memory experiment): nothing of this launch's state was
    // touched, so there is nothing to re-zero on the way out either
    if (a.from_wave && int(__ldcg(&a.ws->wpos)) >= a.count) return;
    extern __shared__ __align__(16) u64 smem[];
    __shared__ int s_nheavy, s_heavy[kMeasWarps * kSlotsPerWarp], s_pe[kMeasWarps], s_pk[kMeasWarps];
    __shared__ int s_wcnt[kMeasWarps];
    __shared__ int s_recj[kMeasWarps][kSlotsPerWarp], s_recn[kMeasWarps][kSlotsPerWarp], s_heavyj[kMeasWarps * kSlotsPerWarp];
    __shared__ u64 s_pn[kMeasWarps];
    __shared__ u32 s_wlist[kMeasWarps][kWarpList];
    __shared__ int s_cnt1, s_fast;
    __shared__ u32 s_targets[kMaxTargets];
    __shared__ PanelSmem ps;
    __shared__ PanelInfo s_info;
    __shared__ u32 s_q[kPanelMax], s_q2[kPanelMax];
    __shared__ __align__(8) u64 s_mbar;
    const int RW = a.m.RW, Wp = a.m.Wp, W = a.m.W;
    MeasSmem sm;
    sm.acc = smem; sm.pe = s_pe; sm.pk = s_pk; sm.pn = s_pn; sm.cnt = &s_cnt1; sm.targets = s_targets;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x;
    const int GW = G * kMeasWarps;
    const int WS = GW * kSlotsPerWarp;              // window size
    const int gw = blockIdx.x * kMeasWarps + warp;
    MeasWs* ws = a.ws;
    u32 epoch = 0;
    u32 tma_parity = 0;
    if (tid == 0) { s_cnt1 = 0; mbar_init(&s_mbar, 1); ps.pready = 0; }
    __syncthreads();

    u64* acc_x = sm.acc + (size_t)warp * 2 * Wp;
    u64* acc_z = acc_x + Wp;

    int pos = a.from_wave ? int(__ldcg(&ws->wpos)) : 0;        // the wave kernels own the deterministic prefix of the block
    u32 wave = 1;
    bool panel_mode = false;
    u64 t_prof = a.prof ? gtime() : 0;
    // =============================================================== wave mode =====
    while (pos < a.count) {
        const int wend = min(a.count, pos + WS);
        // ---- one fused pass: pivot search (K2) and, for every slot whose stabilizer half is empty, the deterministic product (K4)
        // -- speculatively for the slots behind a random measurement too: the pass only reads the tableau, and the outcomes of
        // [r0, wend) are written again by panel mode.  Counters and the odd-phase check are applied after the barrier, below r0.
        if (blockIdx.x == 0 && tid == 0) ws->r0[(wave + 1) % 3] = 0u;
        if (tid == 0) s_nheavy = 0;
        __syncthreads();
        wave_slots(a, pos, wend, wave, gw, GW, s_wlist[warp], &s_nheavy, s_heavy, s_recj[warp], s_recn[warp], acc_x, acc_z);
        __syncthreads();
        const int nheavy = s_nheavy;
        for (int h = 0; h < nheavy; ++h) {
            const int j = pos + s_heavy[h];
            int total;
            const int e = cta_det(a, sm, a.m.cols + (size_t)(2 * a.qubits[j]) * RW + W, nullptr, &total);
            if (tid == 0) { a.outcomes[j] = uint8_t(e >> 1); a.dets[j] = 1; s_heavyj[h] = j; s_heavy[h] = total | ((e & 1) << 30); }
        }
        SK_PROF(0);
        if (!grid_barrier(&ws->bar, epoch, &ws->err)) return;
        SK_PROF(6);
        const u32 r0 = ~__ldcg(&ws->r0[wave % 3]);                               // 0xffffffff = no random measurement in the window
        const int dend = (r0 == 0xffffffffu) ? wend : int(r0);      // [pos, dend) are deterministic and final
        if (lane == 0) {
            u32 nd = 0, kd = 0, odd = 0;
            for (int k = 0; k < kSlotsPerWarp; ++k) {
                const int j = s_recj[warp][k];
                if (j >= 0 && j < dend) { ++nd; kd += u32(s_recn[warp][k] & 0x3fffffff); odd |= u32(s_recn[warp][k] >> 30) & 1u; }
            }
            if (warp == 0) for (int h = 0; h < nheavy; ++h) {
                // (the slot index of a heavy product was replaced by its partner count above; it is below dend iff it was recorded ...
                //  heavy products are rare: their position is re-derived from the record)
                const int j = s_heavyj[h];
                if (j < dend) { ++nd; kd += u32(s_heavy[h] & 0x3fffffff); odd |= u32(s_heavy[h] >> 30) & 1u; }
            }
            if (nd) { atomicAdd(&ws->n_det, (u64)nd); atomicAdd(&ws->k_det, (u64)kd); }
            if (odd) atomicOr(&ws->err, 1u);
        }
        if (blockIdx.x == 0 && tid == 0) atomicAdd(&ws->waves, 1ull);
        SK_PROF(1);
        ++wave;
        pos = dend;
        if (r0 != 0xffffffffu) { panel_mode = true; break; }
    }
    if (!panel_mode) { SK_MEAS_EXIT(); return; }
#ifdef SK_PANEL_TRACE
#define SK_STAGE(k) do { if (a.prof && blockIdx.x == 0 && tid == 0) ws->cprof[8 + (k)] = gtime(); } while (0)
#else
#define SK_STAGE(k) do { } while (0)
#endif
    SK_STAGE(0);

    // =============================================================== panel mode =====
    // (the P2 reads above touch nothing that is written before the next grid barrier)
    if (a.destab_stale) {
        // The host transposed only the stabilizer half C -> R (all a deterministic block needs).  Panel mode works on whole
        // rows: derive the destabilizer rows now, two 256 x 256-bit tiles per CTA at a time (same tile move as k_transpose_bits).
        const int half = tid >> 8, t = tid & 255;
        u32 (*tin)[9] = reinterpret_cast<u32 (*)[9]>(smem) + (size_t)half * 512;
        u32 (*tout)[9] = tin + 256;
        const int nbx = (a.n + 255) / 256, by_lo = RW / 8, nby = (2 * RW + 7) / 8 - by_lo;      // u32 words [RW, 2*RW) of a column = destabilizer rows
        const int ntiles = nbx * nby * 2;
        for (int tile = blockIdx.x * 2 + half; tile < ntiles; tile += 2 * G) {
            const int z = tile / (nbx * nby), r = tile - z * nbx * nby, by = by_lo + r / nbx, bx = r - (r / nbx) * nbx;
            transpose_tile_256(reinterpret_cast<const u32*>(a.m.cols) + (size_t)z * 2 * RW, (size_t)4 * RW, a.n, 2 * RW,
                               reinterpret_cast<u32*>(a.m.rows) + (size_t)z * 2 * Wp, (size_t)4 * Wp, 64 * RW, 2 * Wp,
                               bx * 256, by * 8, t, 2 + half, tin, tout);
        }
        if (!grid_barrier(&ws->bar, epoch, &ws->err)) return;
    }
    SK_STAGE(1);
    if (a.lv_enable) { pos = panel_levels_loop(a, pos, epoch); if (pos < 0) return; }
    SK_STAGE(2);
    const int B = a.B;
    PanelInfo* info = a.info;
    const int gwi = warp * G + blockIdx.x;           // item index interleaved over the CTAs
    u32 prev_nt = 0;
    u32 pbase = 0;                      // progress counter value at the start of this panel attempt (monotone across attempts)
    int kpar = 0;                       // parity of the panel being processed: selects tlist / tM / rowM / eph buffers
    bool have_list = false;             // the active-row list of this panel was already built by the previous apply phase
    const size_t rowcap = (size_t)64 * RW;
    u64 t_cta = 0;
#define SK_CSTART() do { if (a.prof && tid == 0) t_cta = gtime(); } while (0)
#define SK_CPROF(k) do { if (a.prof && tid == 0 && blockIdx.x < 160) ws->ctaphase[blockIdx.x * 4 + k] += gtime() - t_cta; } while (0)
    int pidx = 0;                       // panel index within this launch
    const int tsel = (blockIdx.x == 0) ? 0 : (blockIdx.x == 1) ? 1 : (blockIdx.x == gridDim.x - 1) ? 2 : -1;
#define SK_TRACE(ev) do { if (a.prof && tid == 0 && tsel >= 0 && pidx >= 20 && pidx < 28) ws->trace[((pidx - 20) * 3 + tsel) * 8 + (ev)] = gtime(); } while (0)
    while (pos < a.count) {
        const int Bn = min(B, a.count - pos);
        SK_CSTART(); SK_TRACE(0);
        u64* rowM = a.rowM + (size_t)kpar * rowcap;
        u32* tlist = a.tlist + (size_t)kpar * a.tcap;
        u64* tM = a.tM + (size_t)kpar * a.tcap;
        if (tid < kPanelMax) s_q[tid] = (tid < Bn) ? a.qubits[pos + tid] : 0xffffffffu;
        __syncthreads();
        if (!have_list) {
        // ---- G: gather the panel columns from the R form: warp per group of 32 row-bits
        {
            u32* pan32 = reinterpret_cast<u32*>(a.pan);
            for (int g = gwi; g < 2 * RW; g += GW) {
                const int h = 32 * g + lane;
                const u64* rx = a.m.rows + (size_t)(2 * h) * Wp;
                u32 lo = 0, hi = 0;
                u64 rb = 0;                       // this lane's row: its bits in the panel columns (row form)
                int lastw = -1; u64 lastv = 0;
                for (int j0 = 0; j0 < Bn; j0 += 8) {
                    u32 qq[8]; u64 v[8];
#pragma unroll
                    for (int t = 0; t < 8; ++t) qq[t] = s_q[j0 + t];
#pragma unroll
                    for (int t = 0; t < 8; ++t) {
                        const int wq = int(qq[t] >> 6), prev = t ? int(qq[t - 1] >> 6) : lastw;
                        v[t] = (qq[t] != 0xffffffffu && wq != prev) ? ldcg(rx + wq) : 0ull;
                    }
#pragma unroll
                    for (int t = 0; t < 8; ++t) {
                        if (qq[t] == 0xffffffffu) continue;
                        const int wq = int(qq[t] >> 6);
                        if (wq == lastw) v[t] = lastv; else { lastv = v[t]; lastw = wq; }
                        const u64 bit = (v[t] >> (qq[t] & 63)) & 1ull;
                        const u32 bal = __ballot_sync(0xffffffffu, bit);
                        const int j = j0 + t;
                        rb |= bit << j;
                        if (lane == (j & 31)) { if (j < 32) lo = bal; else hi = bal; }
                    }
                }
                if (lane < Bn) pan32[(size_t)lane * 2 * RW + g] = lo;
                if (lane + 32 < Bn) pan32[(size_t)(lane + 32) * 2 * RW + g] = hi;
                // active rows (any x bit in the panel's columns), compacted in arbitrary order
                const u32 am = __ballot_sync(0xffffffffu, rb != 0);
                if (am) {
                    u32 base = 0;
                    if (lane == 0) base = atomicAdd(&info->acount, (u32)__popc(am));
                    base = __shfl_sync(0xffffffffu, base, 0);
                    if (rb) { const u32 at = base + __popc(am & ((1u << lane) - 1u)); __stcg(a.alist_h + at, (u32)h); __stcg(a.alist_b + at, rb); }
                }
            }
        }
        SK_PROF(2); SK_CPROF(0);
        if (!grid_barrier(&ws->bar, epoch, &ws->err)) return;
        SK_PROF(7); SK_CSTART();
        }   // standalone gather
        // ---- F: symbolic factorisation (CTA 0)
        if (blockIdx.x == 0) {
            const u32 A = __ldcg(&info->acount);
            for (int w = tid; w < RW; w += kMeasThreads) a.tbits[w] = 0;
            __syncthreads();
            if (tid == 0) { info->acount = 0; if (a.prof) { ws->cprof[8] += A; if (A > ws->cprof[9]) ws->cprof[9] = A; } }
            if (A <= (u32)a.row_cap && !a.force_columns && !a.seq_rows) panel_factorise_levels(a, pos, Bn, A, rowM, tlist, tM, pbase);
            else if (A <= (u32)a.row_cap && !a.force_columns) {
                if (A + kPanelMax <= (u32)kRowThreads) panel_factorise_rows<1>(a, ps, pos, Bn, A, rowM, tlist, tM, pbase);
                else if (A + kPanelMax <= 2u * kRowThreads) panel_factorise_rows<2>(a, ps, pos, Bn, A, rowM, tlist, tM, pbase);
                else panel_factorise_rows<4>(a, ps, pos, Bn, A, rowM, tlist, tM, pbase);
            }
            else if (!have_list) panel_factorise(a, smem, ps, s_targets, &s_mbar, tma_parity, pos, Bn, rowM, tlist, tM, pbase);
            else {
                // too many active rows for the row form, and the folded gather made no bit columns: ask for a full gather
                if (tid == 0) { info->dmode = 2; __threadfence(); st_release(&ws->progress, pbase + u32(Bn)); }
            }
        }
        SK_PROF(3); SK_CPROF(1);
        if (blockIdx.x == 0) SK_TRACE(1);
        // ---- consumers (every CTA but 0, which is busy factorising): V pivot values + D part 1, fed step by step
        const int nC = max(1, G - 1);
        const int cidx = (G == 1) ? 0 : int(blockIdx.x) - 1;
        if (G == 1 || blockIdx.x != 0) {
        SK_CSTART();
        { int bad = 0; if (tid == 0) { bad = wait_geq(&ws->progress, pbase + 1u) ? 0 : 1; if (bad) atomicOr(&ws->err, 0x80000000u); }
          if (__syncthreads_or(bad)) return; }
        SK_TRACE(1);
        const u32 dmode = __ldcg(&info->dmode);         // written before the first publication
        const int wpc = (W + nC - 1) / nC;
        const int wlo = min(W, cidx * wpc), whi = min(W, wlo + wpc);
        const int nw = whi - wlo;
        const int nvw = min(kMeasWarps - 1, (nw + 31) / 32);    // warps busy with V (a thread may own several words)
        u64* vs = smem + (size_t)kMeasWarps * 2 * Wp;           // [Bn][2][wpc] after the accumulators
        if (dmode == 1) {
            // The level form publishes the whole panel at once: then the description is staged in shared memory and the
            // pivot rows' words are loaded by the whole CTA, all in flight together (two L2 round trips for the whole phase).
            if (tid == 0) s_fast = int(ld_acquire(&ws->progress) - pbase) >= Bn ? 1 : 0;
            __syncthreads();
            const bool fast = s_fast != 0;
            if (fast) {
                for (int i = tid; i < int(sizeof(PanelInfo) / 8); i += kMeasThreads) reinterpret_cast<u64*>(&s_info)[i] = ldcg(reinterpret_cast<const u64*>(info) + i);
                __syncthreads();
                {   // stage the panel-start words [wlo, whi) of every pivot row: the whole CTA loads, 4 items in flight per thread
                    const int nitems = Bn * 2 * nw;
                    for (int i0 = tid; i0 < nitems; i0 += 4 * kMeasThreads) {
                        u64 v[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int i = i0 + u * kMeasThreads;
                            v[u] = 0;
                            if (i < nitems) {
                                const int k = i / (2 * nw), r = i - k * 2 * nw, half = r / nw, t = r - half * nw;
                                const u32 pk = s_info.piv[k];
                                if (pk != 0xffffffffu) v[u] = ldcg(a.m.rows + (size_t)(2 * pk + half) * Wp + wlo + t);
                            }
                        }
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int i = i0 + u * kMeasThreads;
                            if (i < nitems) { const int k = i / (2 * nw), r = i - k * 2 * nw, half = r / nw, t = r - half * nw; vs[(size_t)(2 * k + half) * wpc + t] = v[u]; }
                        }
                    }
                }
                __syncthreads();
                if (warp < nvw) {
                    const int nvt = 32 * nvw;
                    for (int t = tid; t < nw; t += nvt) {
                        const int w = wlo + t;
                        for (int k = 0; k < Bn; ++k) {
                            if (s_info.piv[k] == 0xffffffffu) continue;
                            u64 ax = vs[(size_t)(2 * k) * wpc + t], az = vs[(size_t)(2 * k + 1) * wpc + t], hb = s_info.hist[k];
                            int e = 0;
                            while (hb) {
                                const int l = __ffsll((long long)hb) - 1; hb &= hb - 1;
                                const u64 bx = vs[(size_t)(2 * l) * wpc + t], bz = vs[(size_t)(2 * l + 1) * wpc + t];
                                e += g_word(bx, bz, ax, az); ax ^= bx; az ^= bz;
                            }
                            vs[(size_t)(2 * k) * wpc + t] = ax; vs[(size_t)(2 * k + 1) * wpc + t] = az;
                            __stcg(a.pivbuf + (size_t)(2 * k) * Wp + w, ax); __stcg(a.pivbuf + (size_t)(2 * k + 1) * Wp + w, az);
                            if (e & 3) atomicAdd(&info->eph[kpar][k], (u32)(e & 3));
                        }
                    }
                }
            } else
            // ---------- streaming: V consumes the published steps in chunks of 8 (two L2 round trips per chunk)
            if (warp < nvw) {
                const int nvt = 32 * nvw;
                for (int done = 0; done < Bn;) {
                    const int target = min(Bn, done + 8);
                    if (!wait_geq(&ws->progress, pbase + u32(target))) { atomicOr(&ws->err, 0x80000000u); break; }
                    for (int t = tid; t < nw; t += nvt) {
                        const int w = wlo + t;
                        u32 pk[8]; u64 hk[8], lx[8], lz[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) pk[u] = (done + u < target) ? __ldcg(&info->piv[done + u]) : 0xffffffffu;
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            lx[u] = 0; lz[u] = 0; hk[u] = 0;
                            if (pk[u] != 0xffffffffu) { const u64* rp = a.m.rows + (size_t)(2 * pk[u]) * Wp + w; lx[u] = ldcg(rp); lz[u] = ldcg(rp + Wp); hk[u] = ldcg(&info->hist[done + u]); }
                        }
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            if (pk[u] == 0xffffffffu) continue;
                            const int k = done + u;
                            u64 ax = lx[u], az = lz[u], hb = hk[u];
                            int e = 0;
                            while (hb) {
                                const int l = __ffsll((long long)hb) - 1; hb &= hb - 1;
                                const u64 bx = vs[(size_t)(2 * l) * wpc + t], bz = vs[(size_t)(2 * l + 1) * wpc + t];
                                e += g_word(bx, bz, ax, az); ax ^= bx; az ^= bz;
                            }
                            vs[(size_t)(2 * k) * wpc + t] = ax; vs[(size_t)(2 * k + 1) * wpc + t] = az;
                            __stcg(a.pivbuf + (size_t)(2 * k) * Wp + w, ax); __stcg(a.pivbuf + (size_t)(2 * k + 1) * Wp + w, az);
                            if (e & 3) atomicAdd(&info->eph[kpar][k], (u32)(e & 3));
                        }
                    }
                    done = target;
                }
            }
            if (nvw) __syncthreads();
            SK_TRACE(2);
            // ---------- streaming D part 1: step j belongs to consumer nC-1 - j % nC (from the far end: V uses the first ones);
            // the step masks N_j are taken in D part 2, when the factorisation has finished
            for (int j = nC - 1 - cidx; j < Bn; j += nC) {
                if (!fast) {
                    int bad = 0; if (tid == 0) { bad = wait_geq(&ws->progress, pbase + u32(j + 1)) ? 0 : 1; if (bad) atomicOr(&ws->err, 0x80000000u); }
                    if (__syncthreads_or(bad)) return;
                }
                if ((fast ? s_info.piv[j] : __ldcg(&info->piv[j])) != 0xffffffffu) continue;
                const int cnt = int(fast ? s_info.dcnt[j] : __ldcg(&info->dcnt[j]));
                const u32* gl = a.dpart + (size_t)j * kRowSlots;
                u64* dx = a.detacc + (size_t)(2 * j) * Wp;
                if (cnt <= kWarpDirect) {
                    if (warp == 0) {
                        for (int i = lane; i < cnt; i += 32) s_wlist[0][i] = __ldcg(gl + i);
                        for (int w = lane; w < Wp; w += 32) { acc_x[w] = 0; acc_z[w] = 0; }
                        __syncwarp();
                        int e = warp_mul_list(a.m.rows, W, Wp, s_wlist[0], cnt, acc_x, acc_z, lane);
                        for (int i = lane; i < cnt; i += 32) e += 2 * sign_bit(a.m.sgn, int(s_wlist[0][i]));
                        e = warp_sum(e) & 3;
                        for (int w = lane; w < W; w += 32) { __stcg(dx + w, acc_x[w]); __stcg(dx + Wp + w, acc_z[w]); }
                        if (lane == 0) info->dete[j] = e;
                    }
                } else {
                    int total;
                    const int e = cta_det(a, sm, a.pan, dx, &total, nullptr, nullptr, gl, cnt);
                    if (tid == 0) info->dete[j] = e;
                }
                __syncthreads();
            }
        } else if (dmode == 0) {
        // ---------- column form: nothing is published before the end; V and D part 1 (with N_j) as one phase
        { int bad = 0; if (tid == 0) { bad = wait_geq(&ws->progress, pbase + u32(Bn)) ? 0 : 1; if (bad) atomicOr(&ws->err, 0x80000000u); }
          if (__syncthreads_or(bad)) return; }
        for (int i = tid; i < int(sizeof(PanelInfo) / 8); i += kMeasThreads) reinterpret_cast<u64*>(&s_info)[i] = ldcg(reinterpret_cast<const u64*>(info) + i);
        __syncthreads();
        const u64 randmask = s_info.randmask;
        const u64 allmask = (Bn < 64) ? ((1ull << Bn) - 1ull) : ~0ull;
        const u64 detmask = ~randmask & allmask;
        if (tid == 0) s_nheavy = 0;
        __syncthreads();
        {
            // V: words [wlo, whi) of every pivot value belong to this CTA; thread t owns word wlo + t
            if (warp < nvw) {
                // stage the panel-start pivot rows' words: items (step k, word t), 4 items (8 loads) in flight per thread
                const int nitems = Bn * nw, nvt = 32 * nvw;
                for (int i0 = tid; i0 < nitems; i0 += 4 * nvt) {
                    u64 lx[4], lz[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int i = i0 + u * nvt;
                        lx[u] = 0; lz[u] = 0;
                        if (i < nitems) {
                            const int k = i / nw, t = i - k * nw;
                            const u32 pk = s_info.piv[k];
                            if (pk != 0xffffffffu) { const u64* rp = a.m.rows + (size_t)(2 * pk) * Wp + wlo + t; lx[u] = ldcg(rp); lz[u] = ldcg(rp + Wp); }
                        }
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int i = i0 + u * nvt;
                        if (i < nitems) { const int k = i / nw, t = i - k * nw; vs[(size_t)(2 * k) * wpc + t] = lx[u]; vs[(size_t)(2 * k + 1) * wpc + t] = lz[u]; }
                    }
                }
                if (nvw == 1) __syncwarp(); else named_bar(2, 32 * nvw);
                for (int t = tid; t < nw; t += nvt) {
                    const int w = wlo + t;
                    u64 bits = randmask;
                    while (bits) {
                        const int k = __ffsll((long long)bits) - 1; bits &= bits - 1;
                        u64 ax = vs[(size_t)(2 * k) * wpc + t], az = vs[(size_t)(2 * k + 1) * wpc + t];
                        u64 hb = s_info.hist[k];
                        int e = 0;
                        while (hb) {
                            const int l = __ffsll((long long)hb) - 1; hb &= hb - 1;
                            const u64 bx = vs[(size_t)(2 * l) * wpc + t], bz = vs[(size_t)(2 * l + 1) * wpc + t];
                            e += g_word(bx, bz, ax, az); ax ^= bx; az ^= bz;
                        }
                        vs[(size_t)(2 * k) * wpc + t] = ax; vs[(size_t)(2 * k + 1) * wpc + t] = az;
                        __stcg(a.pivbuf + (size_t)(2 * k) * Wp + w, ax); __stcg(a.pivbuf + (size_t)(2 * k + 1) * Wp + w, az);
                        if (e & 3) atomicAdd(&info->eph[kpar][k], (u32)(e & 3));
                    }
                }
            } else {
                // D part 1: product of the panel-start partner rows of every deterministic step; the idx-th
                // deterministic step goes to consumer nC-1 - idx % nC, warp (idx / nC) % nwd of the non-V warps
                const int nwd = kMeasWarps - nvw;
                u64 bits = detmask; int idx = 0;
                while (bits) {
                    const int j = __ffsll((long long)bits) - 1; bits &= bits - 1;
                    const int my = idx++;
                    if (nC - 1 - my % nC != cidx || (my / nC) % nwd != warp - nvw) continue;    // from the far end: V uses the first consumers
                    const u64* dcol = a.pan + (size_t)j * RW + W;
                    if (lane == 0) s_wcnt[warp] = 0;
                    __syncwarp();
                    if (s_info.dmode) {          // partner list written by the row-form factorisation
                        const int n = int(s_info.dcnt[j]);
                        const u32* gl = a.dpart + (size_t)j * kRowSlots;
                        if (n <= kWarpDirect) for (int i = lane; i < n; i += 32) s_wlist[warp][i] = __ldcg(gl + i);
                        if (lane == 0) s_wcnt[warp] = n;
                    } else
                    for (int w0 = 0; w0 < W; w0 += 32 * kColChunk) {
                        u64 cv[kColChunk];
#pragma unroll
                        for (int t = 0; t < kColChunk; ++t) { const int w = w0 + 32 * t + lane; cv[t] = (w < W) ? ldcg(dcol + w) : 0ull; }
#pragma unroll
                        for (int t = 0; t < kColChunk; ++t) {
                            const int w = w0 + 32 * t + lane;
                            u64 v = cv[t];
                            while (v) {
                                const int b = __ffsll((long long)v) - 1; v &= v - 1;
                                const int ti = atomicAdd(&s_wcnt[warp], 1);
                                if (ti < kWarpList) s_wlist[warp][ti] = u32(w * 64 + b);
                            }
                        }
                    }
                    __syncwarp();
                    const int npart = s_wcnt[warp];
                    if (npart > kWarpDirect) {                // tree-reduced by the whole CTA below
                        if (lane == 0) { int h = atomicAdd(&s_nheavy, 1); s_heavy[h] = j; }
                        continue;
                    }
                    for (int w = lane; w < Wp; w += 32) { acc_x[w] = 0; acc_z[w] = 0; }
                    int e = warp_mul_list(a.m.rows, W, Wp, s_wlist[warp], npart, acc_x, acc_z, lane);
                    for (int i = lane; i < npart; i += 32) e += 2 * sign_bit(a.m.sgn, int(s_wlist[warp][i]));
                    e = warp_sum(e) & 3;
                    u64 N = 0;
                    for (int i = lane; i < npart; i += 32) N ^= ldcg(rowM + s_wlist[warp][i]);
                    N = warp_xor64(N) & randmask & ((1ull << j) - 1ull);
                    u64* dx = a.detacc + (size_t)(2 * j) * Wp;
                    for (int w = lane; w < W; w += 32) { __stcg(dx + w, acc_x[w]); __stcg(dx + Wp + w, acc_z[w]); }
                    if (lane == 0) { info->dete[j] = e; info->dN[j] = N; }
                    __syncwarp();
                }
            }
            __syncthreads();
            for (int h = 0; h < s_nheavy; ++h) {
                const int j = s_heavy[h];
                int total;
                u64 N = 0;
                const int e = cta_det(a, sm, a.pan + (size_t)j * RW + W, a.detacc + (size_t)(2 * j) * Wp, &total, rowM, &N,
                                      s_info.dmode ? a.dpart + (size_t)j * kRowSlots : nullptr, int(s_info.dcnt[j]));
                if (tid == 0) { info->dete[j] = e; info->dN[j] = N & randmask & ((1ull << j) - 1ull); }
            }
        }
        }   // column form
        SK_CPROF(2);
        }   // consumers
        SK_PROF(4); SK_TRACE(3);
        if (!grid_barrier(&ws->bar, epoch, &ws->err)) return;
        SK_PROF(7); SK_CSTART(); SK_TRACE(4);
        // ---- the finished panel description (one round trip), then the signs of the pivot values
        // (triangular GF(2) recurrence; every CTA solves it itself)
        for (int i = tid; i < int(sizeof(PanelInfo) / 8); i += kMeasThreads) reinterpret_cast<u64*>(&s_info)[i] = ldcg(reinterpret_cast<const u64*>(info) + i);
        const int Bn2 = min(B, a.count - pos - Bn);
        if (tid < kPanelMax) {        // next panel's qubits for the folded gather (same round trip as the description above)
            const bool f = a.fold && Bn2 > 0 && __ldcg(&info->dmode) == 1u;
            s_q2[tid] = (f && tid < Bn2) ? a.qubits[pos + Bn + tid] : 0xffffffffu;
        }
        __syncthreads();
        if (s_info.dmode == 2) { have_list = false; pbase += u32(Bn); continue; }      // regather: same panel again, with the full (row + column) gather
        const u64 randmask = s_info.randmask;
        const u64 allmask = (Bn < 64) ? ((1ull << Bn) - 1ull) : ~0ull;
        const u64 detmask = ~randmask & allmask;
        // The gather of the NEXT panel is folded into this phase when the row form is in use: touched rows emit their new
        // bits as they are written, the untouched ones (not in tbits) are read here -- no separate phase, no grid barrier.
        const bool do_fold = a.fold && s_info.dmode == 1 && Bn2 > 0;
        // housekeeping: retire the previous panel's step-mask entries (its D part 2 was their last reader) and phase sums
        {
            const u32* ptl = a.tlist + (size_t)(kpar ^ 1) * a.tcap;
            u64* prm = a.rowM + (size_t)(kpar ^ 1) * rowcap;
            for (u32 i = blockIdx.x * kMeasThreads + tid; i < prev_nt; i += G * kMeasThreads) __stcg(prm + __ldcg(ptl + i), 0ull);
            if (blockIdx.x == 0 && tid < kPanelMax) info->eph[kpar ^ 1][tid] = 0;
        }
        const u32 pseq = pbase + u32(Bn);            // unique per panel attempt, never 0
        if (tid == 0) {
            u64 psign = 0; u32 odd = 0;
            u64 bits = randmask;
            while (bits) {
                const int k = __ffsll((long long)bits) - 1; bits &= bits - 1;
                const u32 ek = s_info.eph[kpar][k] + 2u * (u32)((s_info.osign >> k) & 1ull) + 2u * (u32)__popcll(s_info.hist[k] & psign);
                odd |= ek & 1u;
                psign |= (u64)((ek >> 1) & 1u) << k;
            }
            ps.psign = psign; ps.podd = odd;
            __threadfence_block();
            *(volatile u32*)&ps.pready = pseq;          // the warps pick the signs up when they first need them (end of their first item)
            if (odd) atomicOr(&ws->err, 1u);
        }
        bool ps_have = false; u64 ps_val = 0;
        auto get_psign = [&]() -> u64 {
            if (!ps_have) {
                if (lane == 0) { while (*(volatile u32*)&ps.pready != pseq) {} }
                __syncwarp();
                ps_val = *(volatile u64*)&ps.psign; ps_have = true;
            }
            return ps_val;
        };
        // ---- D part 2 + A: items = deterministic steps, then touched rows; warp per item
        {
            const int nd = __popcll(detmask);
            const int nt = int(s_info.nt);
            // next panel's bits of a row whose new x words sit in this warp's accumulator
            auto emit_next = [&](u32 h) {
                if (!do_fold) return;
                __syncwarp();
                const u32 q0 = s_q2[lane], q1 = s_q2[lane + 32];
                const u32 b0 = (q0 != 0xffffffffu) ? u32((acc_x[q0 >> 6] >> (q0 & 63)) & 1ull) : 0u;
                const u32 b1 = (q1 != 0xffffffffu) ? u32((acc_x[q1 >> 6] >> (q1 & 63)) & 1ull) : 0u;
                const u64 rb = (u64)__ballot_sync(0xffffffffu, b0) | ((u64)__ballot_sync(0xffffffffu, b1) << 32);
                if (rb && lane == 0) { const u32 at = atomicAdd(&info->acount, 1u); __stcg(a.alist_h + at, h); __stcg(a.alist_b + at, rb); }
                __syncwarp();
            };
            for (int it = gwi; it < nd + nt; it += GW) {
                if (it < nd) {
                    // deterministic step: j = it-th set bit of detmask
                    u64 bits = detmask; for (int s = 0; s < it; ++s) bits &= bits - 1;
                    const int j = __ffsll((long long)bits) - 1;
                    const u64* dx = a.detacc + (size_t)(2 * j) * Wp;
                    for (int w = lane; w < W; w += 32) { acc_x[w] = ldcg(dx + w); acc_z[w] = ldcg(dx + Wp + w); }
                    u64 N;
                    if (s_info.dmode) {        // XOR of the partners' step masks, restricted to the steps before j
                        N = 0;
                        const int cnt = int(s_info.dcnt[j]);
                        const u32* gl = a.dpart + (size_t)j * kRowSlots;
                        for (int i = lane; i < cnt; i += 32) N ^= ldcg(rowM + __ldcg(gl + i));
                        N = warp_xor64(N) & randmask & ((1ull << j) - 1ull);
                    } else N = ldcg(&info->dN[j]);
                    const u64 Z = s_info.dZ[j];
                    int cnt = 0;
                    { u64 b = N; while (b) { const int l = __ffsll((long long)b) - 1; b &= b - 1; if (lane == 0) s_wlist[warp][cnt] = u32(l); ++cnt; } }
                    __syncwarp();
                    int e = warp_mul_list(a.pivbuf, W, Wp, s_wlist[warp], cnt, acc_x, acc_z, lane);
                    __syncwarp();
                    const u64 sgd = get_psign();
                    if (lane == 0) {
                        e += __ldcg(&info->dete[j]) + 2 * __popcll(N & sgd);
                        u64 b = Z;
                        while (b) {        // (+-Z_{q_l}) * acc
                            const int l = __ffsll((long long)b) - 1; b &= b - 1;
                            const u32 ql = s_q[l];
                            const u64 zb = 1ull << (ql & 63);
                            e += g_word(0ull, zb, acc_x[ql >> 6], acc_z[ql >> 6]) + 2 * int(s_info.outc[l]);
                            acc_z[ql >> 6] ^= zb;
                        }
                    }
                    e = warp_sum(e) & 3;
                    if (lane == 0) {
                        if (e & 1) atomicOr(&ws->err, 1u);
                        a.outcomes[pos + j] = uint8_t(e >> 1); a.dets[pos + j] = 1;
                    }
                    __syncwarp();
                } else {
                    const int i = it - nd;
                    const u32 h = __ldcg(tlist + i);
                    u64 M = ldcg(tM + i);
                    // is h a pivot of this panel, or the destabilizer partner of one?
                    int kp = -1, ko = -1;
                    {
                        const u32 p0 = (lane < Bn) ? s_info.piv[lane] : 0xffffffffu, p1 = (lane + 32 < Bn) ? s_info.piv[lane + 32] : 0xffffffffu;
                        const u32 b0 = __ballot_sync(0xffffffffu, p0 == h), b1 = __ballot_sync(0xffffffffu, p1 == h);
                        const u32 c0 = __ballot_sync(0xffffffffu, p0 != 0xffffffffu && p0 + (u32)a.NS == h), c1 = __ballot_sync(0xffffffffu, p1 != 0xffffffffu && p1 + (u32)a.NS == h);
                        if (b0) kp = __ffs(b0) - 1; else if (b1) kp = 32 + __ffs(b1) - 1;
                        if (c0) ko = __ffs(c0) - 1; else if (c1) ko = 32 + __ffs(c1) - 1;
                    }
                    u64* tx = a.m.rows + (size_t)(2 * h) * Wp;
                    u64* sg = a.m.sgn + (h >> 6);
                    const u64 hb = 1ull << (h & 63);
                    if (kp >= 0) {                // row p := +-Z_q
                        const u32 q = s_q[kp];
                        for (int w = lane; w < 2 * Wp; w += 32) __stcg(tx + w, (w == Wp + int(q >> 6)) ? (1ull << (q & 63)) : 0ull);
                        if (lane == 0) { if (s_info.outc[kp]) atomicOr(sg, hb); else atomicAnd(sg, ~hb); a.outcomes[pos + kp] = s_info.outc[kp]; a.dets[pos + kp] = 0; }
                        continue;
                    }
                    int e;
                    if (ko >= 0) {                // row p+n := P_ko', then the later steps
                        const u64* sx = a.pivbuf + (size_t)(2 * ko) * Wp;
                        for (int w = lane; w < W; w += 32) { acc_x[w] = ldcg(sx + w); acc_z[w] = ldcg(sx + Wp + w); }
                        M &= (ko < 63) ? ~((2ull << ko) - 1ull) : 0ull;
                        e = 0;                       // (+ the sign of P_ko', added with the other pivot signs below)
                    } else {
                        for (int w = lane; w < W; w += 32) { acc_x[w] = ldcg(tx + w); acc_z[w] = ldcg(tx + Wp + w); }
                        e = (lane == 0) ? 2 * int((ldcg(sg) >> (h & 63)) & 1ull) : 0;
                        if (M == 0) { emit_next(h); continue; }
                    }
                    int cnt = 0;
                    { u64 b = M; while (b) { const int l = __ffsll((long long)b) - 1; b &= b - 1; if (lane == 0) s_wlist[warp][cnt] = u32(l); ++cnt; } }
                    __syncwarp();
                    e += warp_mul_list(a.pivbuf, W, Wp, s_wlist[warp], cnt, acc_x, acc_z, lane);
                    { const u64 sg_ = get_psign(); if (lane == 0) e += 2 * __popcll(M & sg_) + (ko >= 0 ? 2 * int((sg_ >> ko) & 1ull) : 0); }
                    e = warp_sum(e) & 3;
                    for (int w = lane; w < W; w += 32) { __stcg(tx + w, acc_x[w]); __stcg(tx + Wp + w, acc_z[w]); }
                    if (lane == 0) {
                        if (e & 1) atomicOr(&ws->err, 1u);
                        if (e >> 1) atomicOr(sg, hb); else atomicAnd(sg, ~hb);
                    }
                    emit_next(h);
                }
            }
            // folded gather, untouched rows: a lane per row, rows listed in tbits are skipped (their warps emitted them above)
            SK_TRACE(5);
            if (do_fold) {
                // groups are handed out from the far end of the warp index space: the item loop above keeps the first warps busy
                for (int g = GW - 1 - gwi; g < 2 * RW; g += GW) {
                    const int h = 32 * g + lane;
                    const bool skip = (ldcg(a.tbits + (h >> 6)) >> (h & 63)) & 1ull;
                    const u64* rx = a.m.rows + (size_t)(2 * h) * Wp;
                    u64 rb = 0;
                    int lastw = -1; u64 lastv = 0;
                    for (int j0 = 0; j0 < Bn2; j0 += 8) {
                        u32 qq[8]; u64 v[8];
#pragma unroll
                        for (int t = 0; t < 8; ++t) qq[t] = s_q2[j0 + t];
#pragma unroll
                        for (int t = 0; t < 8; ++t) {
                            const int wq = int(qq[t] >> 6), prev = t ? int(qq[t - 1] >> 6) : lastw;
                            v[t] = (!skip && qq[t] != 0xffffffffu && wq != prev) ? ldcg(rx + wq) : 0ull;
                        }
#pragma unroll
                        for (int t = 0; t < 8; ++t) {
                            if (qq[t] == 0xffffffffu) continue;
                            const int wq = int(qq[t] >> 6);
                            if (wq == lastw) v[t] = lastv; else { lastv = v[t]; lastw = wq; }
                            rb |= ((v[t] >> (qq[t] & 63)) & 1ull) << (j0 + t);
                        }
                    }
                    if (skip) rb = 0;
                    const u32 am = __ballot_sync(0xffffffffu, rb != 0);
                    if (am) {
                        u32 base = 0;
                        if (lane == 0) base = atomicAdd(&info->acount, (u32)__popc(am));
                        base = __shfl_sync(0xffffffffu, base, 0);
                        if (rb) { const u32 at = base + __popc(am & ((1u << lane) - 1u)); __stcg(a.alist_h + at, (u32)h); __stcg(a.alist_b + at, rb); }
                    }
                }
            }
        }
        SK_PROF(5); SK_CPROF(3); SK_TRACE(6);
        if (!grid_barrier(&ws->bar, epoch, &ws->err)) return;
        SK_PROF(7); SK_TRACE(7);
        ++pidx;
        prev_nt = s_info.nt;
        have_list = do_fold;
        kpar ^= 1;
        pbase += u32(Bn);
        pos += Bn;
    }
    SK_STAGE(3);
    {   // the last panel's entries (buffers of parity kpar ^ 1 after the final toggle)
        const u32* ptl = a.tlist + (size_t)(kpar ^ 1) * a.tcap;
        u64* prm = a.rowM + (size_t)(kpar ^ 1) * rowcap;
        for (u32 i = blockIdx.x * kMeasThreads + tid; i < prev_nt; i += G * kMeasThreads) __stcg(prm + __ldcg(ptl + i), 0ull);
        if (blockIdx.x == 0 && tid < kPanelMax) { info->eph[0][tid] = 0; info->eph[1][tid] = 0; }
    }
    // Panel mode kept only the R form current: re-derive the C form here (same tile move as k_transpose_bits, two tiles per
    // CTA at a time), so that the host never needs a conditional transpose after a measurement block.  Every row was final at
    // the last grid barrier.
    {
        const int half = tid >> 8, t = tid & 255;
        u32 (*tin)[9] = reinterpret_cast<u32 (*)[9]>(smem) + (size_t)half * 512;
        u32 (*tout)[9] = tin + 256;
        const int nbx = (64 * RW + 255) / 256, nby = (2 * Wp + 7) / 8;
        const int ntiles = nbx * nby * 2;
        __syncthreads();
        for (int tile = blockIdx.x * 2 + half; tile < ntiles; tile += 2 * G) {
            const int z = tile / (nbx * nby), r = tile - z * nbx * nby, by = r / nbx, bx = r - by * nbx;
            transpose_tile_256(reinterpret_cast<const u32*>(a.m.rows) + (size_t)z * 2 * Wp, (size_t)4 * Wp, 64 * RW, 2 * Wp,
                               reinterpret_cast<u32*>(a.m.cols) + (size_t)z * 2 * RW, (size_t)4 * RW, a.n, 2 * RW,
                               bx * 256, by * 8, t, 2 + half, tin, tout);
        }
    }
    SK_STAGE(4);
    SK_MEAS_EXIT();
}

// SPEC:165-173 rowsum(h, i) on the R form + C form fix-up, single CTA (API parity helper).
__global__ void __launch_bounds__(256)
k_rowsum_single(DMat m, int h, int i, u32* err) {
    __shared__ int s_e[8];
    const int Wp = m.Wp, W = m.W, RW = m.RW;
    u64* hx = m.rows + (size_t)(2 * h) * Wp; u64* hz = hx + Wp;
    const u64* ix = m.rows + (size_t)(2 * i) * Wp; const u64* iz = ix + Wp;
    int e = 0;
    for (int w = threadIdx.x; w < W; w += blockDim.x) {
        u64 ax = ix[w], az = iz[w], bx = hx[w], bz = hz[w];
        e += g_word(ax, az, bx, bz);
        hx[w] = bx ^ ax; hz[w] = bz ^ az;
        // C form: flip bit h of every column where row i is set
        u64 bits = ax;
        while (bits) { int b = __ffsll((long long)bits) - 1; bits &= bits - 1;
            atomicXor(m.cols + (size_t)(2 * (w * 64 + b)) * RW + (h >> 6), 1ull << (h & 63)); }
        bits = az;
        while (bits) { int b = __ffsll((long long)bits) - 1; bits &= bits - 1;
            atomicXor(m.cols + (size_t)(2 * (w * 64 + b) + 1) * RW + (h >> 6), 1ull << (h & 63)); }
    }
    e = warp_sum(e);
    if ((threadIdx.x & 31) == 0) s_e[threadIdx.x >> 5] = e;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0; for (int k = 0; k < int(blockDim.x >> 5); ++k) t += s_e[k];
        int rh = int((m.sgn[h >> 6] >> (h & 63)) & 1ull), ri = int((m.sgn[i >> 6] >> (i & 63)) & 1ull);
        int sum = (2 * rh + 2 * ri + t) & 3;
        if (sum & 1) { atomicOr(err, 1u); }
        else if ((sum >> 1) != rh) m.sgn[h >> 6] ^= 1ull << (h & 63);
    }
}

}  // namespace skd
