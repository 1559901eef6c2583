// kernels_measure.cuh -- K2/K3/K4: a block of consecutive Z measurements executed by
// ONE persistent cooperative kernel (no host round trips; branches are data dependent).
// Exact CHP semantics (Algorithm 1): the tableau, signs and
// record are bit-identical to measuring one qubit at a time, in order.
//
// Out-of-order wave scheduler.  The FOOTPRINT of a pending measurement j in the current
// state is the set of row slots F_j = {i mod n : x_iq = 1} (slot i = stabilizer i and its
// destabilizer partner; the pivot and its partner are in it by construction).  Two
// measurements with disjoint footprints act on disjoint rows, cannot change each other's
// column x_q, pivot, branch or phases, and therefore commute bit-exactly -- also with
// everything the earlier one may turn into once ITS predecessors have run (DESIGN.md,
// "independence of measurements"; tools/proto_waves.py checks the rule against the oracle).
// Per wave, over a window of pending measurements (kSlotsPerWarp per warp of the grid):
//
//   P1  pivot search = scan of the stabilizer half of column x_q in the C form (contiguous;
//       ffs + warp min) -- K2.  Every window member CLAIMS its slots with a 64-bit atomicMax
//       of (wave, ~j); the first random index r0 is min-reduced.           -- grid barrier --
//   P2  j < r0: deterministic and final (nothing before it writes).  j >= r0: runnable iff
//       no slot of F_j is claimed by a smaller index.  Runnable deterministic measurements
//       are evaluated at once from the read-only R form: ordered product of the stabilizer
//       partners, phase by popcounts mod 4 -- K4.                           -- grid barrier --
//   P3  runnable random measurements, one CTA each -- K3: column mask, pivot row P and old
//       destabilizer row D staged in shared memory by 1-D TMA bulk copies, then
//         B1 R form: rowsum(i, p) for every i in the mask (warp per row, P from smem)
//         B2 C form: column_j ^= mask for j in supp(P)            (word parallel, atomicXor)
//         B3 C form: bit fixes for the overwritten rows p and p+n ; sign bits ; record
//         B4 R form: row p+n := P ; row p := Z_q                            -- grid barrier --
//   A window without random measurements needs only the first barrier.  The first pending
//   measurement is always runnable, so every wave makes progress; RNG ordinal and record
//   slot are those of the measurement's position, never of its execution order.
// Both forms stay valid throughout.  Row i = p+n is skipped in B1 (it is overwritten;
// SURVEY.md section 7 "rowsum on the pivot's own destabilizer").
//
// Roofline: HBM/L2.  Algorithmic bytes: random  RW*8 + 16W + k*32W + 32W ;
// deterministic  RW*8/2 + k*16W  -- reported from the k counters kept here.
#pragma once
#include "common.cuh"

namespace skd {

struct MeasWs {
    u32 bar;            // grid barrier counter (zeroed before each launch)
    u32 err;            // bit0 odd phase (invariant), bit31 barrier timeout, bit30 tma timeout
    u32 r0[4];          // per-wave index of the first random measurement, min-reduced; 3 slots rotate
    u64 n_rand, n_det, k_rand, k_det, waves;
    u64 prof[8];        // block-0 wall time (ns) per phase: P1, barrier, P2, barrier, P3, barrier, sequential, window search
    u32 ncommit;        // measurements executed so far in this launch
    u32 pad;
    u64 dbg[8];         // SK_DEBUG_PROF: cta_random ns in {stage+lists, B1, B2, B3+B4+record}, sums of nt, nmw, nsup, calls
    u64 seqprof[8];     // sequential mode, CTA 0: inspect, det, random, fence ns ; [4] det count, [5] random count, [6] SM cycles, [7] ns
};

constexpr int kMeasThreads = 512;
constexpr int kMeasWarps = kMeasThreads / 32;
constexpr int kSlotsPerWarp = 4;
constexpr int kColChunk = 6;         // column words per lane loaded back-to-back (192 words per chunk)
constexpr int kNarrowWaves = 32;      // consecutive narrow waves before switching to sequential mode
constexpr int kSeqMin = 256, kSeqMax = 4096;   // sequential run length (doubles while waves stay narrow)
constexpr int kMaxTargets = 2048, kMaxMaskWords = 512, kMaxSupport = 4096;   // sparse work-list capacities (dense fallback above)
constexpr int kWarpList = 48;        // partner rows a single warp multiplies itself; longer products are tree-reduced by a CTA

struct MeasArgs {
    DMat m;             // tableau (C and R valid)
    int n;              // qubits == rows per half
    int NS;             // row-bit offset of the destabilizer half (64*W)
    const u32* qubits;  // measurement list
    int count;
    uint64_t seed, ordinal0;
    uint8_t* outcomes;  // [count]
    uint8_t* dets;      // [count]
    MeasWs* ws;
    u64* claim;         // [64*W] slot claims, zeroed before each launch
    u32* wpiv;          // [2][window] pivot of a window slot (0xffffffff = deterministic), by wave parity
    uint8_t* wrun;      // [2][window] 1 = runnable random measurement, by wave parity
    uint8_t* done;      // [count], zeroed before each launch
    int prof;           // SK_DEBUG_PROF: extra barriers + timers inside cta_random (debug only)
    int use_tma;        // stage mask/P/D with cp.async.bulk (1) or ld.global.cg (0)
    int seq_threshold;  // a wave committing fewer measurements than this switches to sequential mode (0 = never)
};

__device__ __forceinline__ u64 gtime() { u64 t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
#define SK_PROF(k) do { if (a.prof && blockIdx.x == 0 && tid == 0) { u64 _n = gtime(); ws->prof[k] += _n - t_prof; t_prof = _n; } } while (0)

__device__ __forceinline__ int sign_bit(const u64* sgn, int r) { return int((ldcg(sgn + (r >> 6)) >> (r & 63)) & 1ull); }

// K4: product of the stabilizer rows listed in `list` (entries part, part+nparts, ...), phase
// exponent mod 4 returned warp-uniform.  Stabilizer rows commute and Pauli multiplication is
// associative, so any grouping/order of the factors gives the same Hermitian product; 8 rows are
// loaded per step so their latencies overlap.  acc_x/acc_z [Wp] are private to the warp
// (lane-strided words).
__device__ __forceinline__ int det_list_partial(const DMat& m, const u32* list, int cnt, int part, int nparts,
                                                u64* acc_x, u64* acc_z, int lane, int* k_out) {
    const int W = m.W, Wp = m.Wp;
    for (int w = lane; w < Wp; w += 32) { acc_x[w] = 0; acc_z[w] = 0; }
    int e = 0, k = 0;
    for (int i0 = part; i0 < cnt; i0 += 8 * nparts) {
        int s[8]; int ns = 0;
#pragma unroll
        for (int t = 0; t < 8; ++t) { const int i = i0 + t * nparts; if (i < cnt) { s[t] = int(list[i]); ns = t + 1; } else s[t] = 0; }
        if (lane < ns) e += 2 * sign_bit(m.sgn, int(list[i0 + lane * nparts]));
        for (int w = lane; w < W; w += 32) {
            u64 sx[8], sz[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) if (t < ns) {
                const u64* rx = m.rows + (size_t)(2 * s[t]) * Wp;
                sx[t] = ldcg(rx + w); sz[t] = ldcg(rx + Wp + w);
            }
            u64 ax = acc_x[w], az = acc_z[w];
#pragma unroll
            for (int t = 0; t < 8; ++t) if (t < ns) {
                e += g_word(sx[t], sz[t], ax, az);      // rowsum(scratch, s): left factor = row s
                ax ^= sx[t]; az ^= sz[t];
            }
            acc_x[w] = ax; acc_z[w] = az;
        }
        k += ns;
    }
    *k_out = k;
    return warp_sum(e) & 3;
}

// ---- CTA-wide building blocks (all kMeasThreads threads call them together) -------------
struct MeasSmem {
    u64* mask;      // [RW]   column x_q (rows to update; pivot bits cleared)
    u64* P;         // [2*Wp] pivot row
    u64* D;         // [2*Wp] old destabilizer row of the pivot
    u64* acc;       // [kMeasWarps][2*Wp] per-warp product accumulators
    u64* mbar;
    int* pe; int* pk;
    int* cnt;                 // [3] list lengths
    u32* targets;             // [kMaxTargets] rows to rowsum
    unsigned short* mwords;   // [kMaxMaskWords] non-zero mask words
    u32* support;             // [kMaxSupport] (2*qubit + half) entries of supp(P)
};

// K3: one random measurement (index jr, qubit q, pivot stabilizer row-bit p) by one CTA.
__device__ __forceinline__ void cta_random(const MeasArgs& a, const MeasSmem& sm, int jr, u32 q, int p, u32& tma_parity, bool exclusive) {
    const int RW = a.m.RW, Wp = a.m.Wp, W = a.m.W;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    MeasWs* ws = a.ws;
    const int pd = a.NS + p;
    const u64* qcol = a.m.cols + (size_t)(2 * q) * RW;
    u64 tp_in = 0;
    if (a.prof && tid == 0) tp_in = gtime();
    const int sp = sign_bit(a.m.sgn, p), sd = sign_bit(a.m.sgn, pd);
    // one pass: stage mask | P | D into shared memory (contiguous) and, from the same registers,
    // compact the work lists: target rows + non-zero mask words (pivot bits removed), support of P.
    // sm.cnt[0..2] are zero on entry (reset at the end of the previous CTA-level operation).
    if (a.use_tma) {          // 1-D TMA bulk copies on one mbarrier (UBLKCP); lists are built from smem afterwards
        if (tid == 0) {
            asm volatile("fence.proxy.async;" ::: "memory");
            mbar_expect_tx(sm.mbar, u32(RW * 8 + 4 * Wp * 8));
            tma_load_1d(sm.mask, qcol, u32(RW * 8), sm.mbar);
            tma_load_1d(sm.P, a.m.rows + (size_t)(2 * p) * Wp, u32(2 * Wp * 8), sm.mbar);
            tma_load_1d(sm.D, a.m.rows + (size_t)(2 * pd) * Wp, u32(2 * Wp * 8), sm.mbar);
        }
        if (!mbar_wait(sm.mbar, tma_parity)) { if (tid == 0) atomicOr(&ws->err, 0x40000000u); }
        tma_parity ^= 1;
        __syncthreads();
    }
    {
        const u64* rp = a.m.rows + (size_t)(2 * p) * Wp;
        const u64* rd = a.m.rows + (size_t)(2 * pd) * Wp;
        const int total_words = RW + 4 * Wp;
        for (int w0 = 0; w0 < total_words; w0 += kMeasThreads) {       // whole warps iterate together (w0 + tid may overrun)
            const int w = w0 + tid;
            u64 v = 0;
            if (w < total_words)
                v = a.use_tma ? sm.mask[w]
                              : ((w < RW) ? ldcg(qcol + w) : (w < RW + 2 * Wp ? ldcg(rp + (w - RW)) : ldcg(rd + (w - RW - 2 * Wp))));
            int kind = 2;                                               // 0 mask word, 1 word of P, 2 neither
            if (w < RW) {
                kind = 0;
                if (w == (p >> 6)) v &= ~(1ull << (p & 63));
                if (w == (pd >> 6)) v &= ~(1ull << (pd & 63));
                sm.mask[w] = v;
            } else if (w < total_words) {
                if (!a.use_tma) sm.mask[w] = v;
                if (w - RW < 2 * Wp) kind = 1;
            }
            // warp-aggregated appends: one shared-memory atomic per warp and list
            const int pc = (kind == 2) ? 0 : __popcll(v);
            const int pc_t = kind == 0 ? pc : 0, pc_s = kind == 1 ? pc : 0;
            int in_t = pc_t, in_s = pc_s;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int vt = __shfl_up_sync(0xffffffffu, in_t, o), vs = __shfl_up_sync(0xffffffffu, in_s, o);
                if (lane >= o) { in_t += vt; in_s += vs; }
            }
            const u32 nzmask = __ballot_sync(0xffffffffu, kind == 0 && v != 0);
            int base_t = 0, base_s = 0, base_m = 0;
            if (lane == 31) {
                if (in_t) base_t = atomicAdd(&sm.cnt[0], in_t);
                if (in_s) base_s = atomicAdd(&sm.cnt[2], in_s);
                if (nzmask) base_m = atomicAdd(&sm.cnt[1], __popc(nzmask));
            }
            base_t = __shfl_sync(0xffffffffu, base_t, 31); base_s = __shfl_sync(0xffffffffu, base_s, 31); base_m = __shfl_sync(0xffffffffu, base_m, 31);
            if (kind == 0 && v) {
                const int mi = base_m + __popc(nzmask & ((1u << lane) - 1u));
                if (mi < kMaxMaskWords) sm.mwords[mi] = (unsigned short)w;
                int ti = base_t + in_t - pc_t;
                u64 bits = v;
                while (bits) {
                    const int b = __ffsll((long long)bits) - 1; bits &= bits - 1;
                    if (ti < kMaxTargets) sm.targets[ti] = u32(w * 64 + b);
                    ++ti;
                }
            } else if (kind == 1 && v) {
                const int u = w - RW, h = u >= Wp, pw = h ? u - Wp : u;
                int pi = base_s + in_s - pc_s;
                u64 bits = v;
                while (bits) {
                    const int b = __ffsll((long long)bits) - 1; bits &= bits - 1;
                    if (pi < kMaxSupport) sm.support[pi] = (u32(pw * 64 + b) << 1) | u32(h);
                    ++pi;
                }
            }
        }
    }
    __syncthreads();
    const int nt = sm.cnt[0], nmw = sm.cnt[1], nsup = sm.cnt[2];
    u64 tp0 = 0;
    if (a.prof && tid == 0) { tp0 = gtime(); ws->dbg[0] += tp0 - tp_in; ws->dbg[4] += nt; ws->dbg[5] += nmw; ws->dbg[6] += nsup; }
    const bool sparse = nt <= kMaxTargets && nmw <= kMaxMaskWords && nsup <= kMaxSupport;
    // B1: rowsum(i, p) for every target row i (warp per row, P from smem)
    auto rowsum_into = [&](int i) {
        u64* tx = a.m.rows + (size_t)(2 * i) * Wp;
        u64* tz = tx + Wp;
        int e = 0;
        for (int w0 = 0; w0 < W; w0 += 32 * kColChunk) {     // loads first, then phase + stores
            u64 xv[kColChunk], zv[kColChunk];
#pragma unroll
            for (int t = 0; t < kColChunk; ++t) {
                const int w = w0 + 32 * t + lane;
                xv[t] = (w < W) ? ldcg(tx + w) : 0ull; zv[t] = (w < W) ? ldcg(tz + w) : 0ull;
            }
#pragma unroll
            for (int t = 0; t < kColChunk; ++t) {
                const int w = w0 + 32 * t + lane;
                if (w >= W) continue;
                const u64 px = sm.P[w], pz = sm.P[Wp + w];
                e += g_word(px, pz, xv[t], zv[t]);             // left factor = pivot row
                if (px) __stcg(tx + w, xv[t] ^ px);
                if (pz) __stcg(tz + w, zv[t] ^ pz);
            }
        }
        e = warp_sum(e) & 3;
        if (lane == 0) {
            if (e & 1) atomicOr(&ws->err, 1u);
            if (sp ^ (e >> 1)) atomicXor(a.m.sgn + (i >> 6), 1ull << (i & 63));
        }
    };
    if (sparse) {
        for (int t = warp; t < nt; t += kMeasWarps) rowsum_into(int(sm.targets[t]));
        if (a.prof) { __syncthreads(); if (tid == 0) { u64 t = gtime(); ws->dbg[1] += t - tp0; tp0 = t; } }
        // B2: C form, column_j ^= mask for j in supp(P): warp per support entry, lanes over the non-zero mask words
        for (int e = warp; e < nsup; e += kMeasWarps) {
            const u32 ent = sm.support[e];
            u64* col = a.m.cols + (size_t)ent * RW;           // ent == 2*qubit + half
            if (exclusive) {      // no other CTA touches C (sequential mode): plain RMW, except the two words B3 also updates
                for (int i = lane; i < nmw; i += 32) {
                    const int w = sm.mwords[i];
                    if (w == (p >> 6) || w == (pd >> 6)) atomicXor(col + w, sm.mask[w]);
                    else __stcg(col + w, ldcg(col + w) ^ sm.mask[w]);
                }
            } else {
                for (int i = lane; i < nmw; i += 32) { const int w = sm.mwords[i]; atomicXor(col + w, sm.mask[w]); }
            }
        }
    } else {
        for (int mw = warp; mw < RW; mw += kMeasWarps) {
            u64 bits = sm.mask[mw];
            while (bits) { int b = __ffsll((long long)bits) - 1; bits &= bits - 1; rowsum_into(mw * 64 + b); }
        }
        for (int u = warp; u < 2 * W; u += kMeasWarps) {
            const int h = u >= W, pw = h ? u - W : u;
            u64 bits = sm.P[h * Wp + pw];
            while (bits) {
                int b = __ffsll((long long)bits) - 1; bits &= bits - 1;
                u64* col = a.m.cols + (size_t)(2 * (pw * 64 + b) + h) * RW;
                for (int w = lane; w < RW; w += 32) { u64 mv = sm.mask[w]; if (mv) atomicXor(col + w, mv); }
            }
        }
    }
    if (a.prof) { __syncthreads(); if (tid == 0) { u64 t = gtime(); ws->dbg[2] += t - tp0; tp0 = t; } }
    // B3: C form, single-bit fixes for rows p (-> Z_q) and p+n (-> P); thread per (list, word)
    {
        const u64 pbit = 1ull << (p & 63), dbit = 1ull << (pd & 63);
        for (int u = tid; u < 4 * W; u += kMeasThreads) {
            const int list = (u >= 2 * W) ? (u >= 3 * W ? 3 : 2) : (u >= W ? 1 : 0), pw = u - list * W;
            const int h = list & 1;
            u64 bits; int word; u64 bit;
            if (list < 2) {          // row p: old P -> Z_q
                bits = sm.P[h * Wp + pw];
                if (h == 1 && pw == int(q >> 6)) bits ^= 1ull << (q & 63);
                word = p >> 6; bit = pbit;
            } else {                 // row p+n: old D -> P
                bits = sm.D[h * Wp + pw] ^ sm.P[h * Wp + pw];
                word = pd >> 6; bit = dbit;
            }
            while (bits) {
                int b = __ffsll((long long)bits) - 1; bits &= bits - 1;
                atomicXor(a.m.cols + (size_t)(2 * (pw * 64 + b) + h) * RW + word, bit);
            }
        }
    }
    // B4: R form, row p+n := P ; row p := Z_q
    {
        u64* rp = a.m.rows + (size_t)(2 * p) * Wp;
        u64* rd = a.m.rows + (size_t)(2 * pd) * Wp;
        for (int w = tid; w < 2 * Wp; w += kMeasThreads) {
            __stcg(rd + w, sm.P[w]);
            u64 v = 0;
            if (w == Wp + int(q >> 6)) v = 1ull << (q & 63);
            __stcg(rp + w, v);
        }
    }
    // signs, record, counters
    if (warp == 0) {
        const int k = nt;
        if (lane == 0) {
            const int out = counter_bit(a.seed, a.ordinal0 + (uint64_t)jr);
            if (sp != out) atomicXor(a.m.sgn + (p >> 6), 1ull << (p & 63));
            if (sd != sp) atomicXor(a.m.sgn + (pd >> 6), 1ull << (pd & 63));
            a.outcomes[jr] = uint8_t(out);
            a.dets[jr] = 0; a.done[jr] = 1;
            atomicAdd(&ws->n_rand, 1ull); atomicAdd(&ws->k_rand, (u64)k); atomicAdd(&ws->ncommit, 1u);
        }
    }
    if (tid == 0) { sm.cnt[0] = 0; sm.cnt[1] = 0; sm.cnt[2] = 0; }
    __syncthreads();      // smem is restaged by the next measurement
    if (a.prof && tid == 0) { ws->dbg[3] += gtime() - tp0; ws->dbg[7] += 1; }
}

// K4 by a whole CTA: the partner list is compacted into shared memory, then thread (w, g) owns
// word w of the product for row group g and multiplies its share of the listed rows word by word,
// 8 row loads in flight; groups are folded and the per-word phase contributions block-reduced
// (popcounts mod 4).  Word-parallel evaluation is the same product: g is a sum over qubit
// positions; the list order is irrelevant because stabilizer rows commute.
// sm.cnt[0] is zero on entry and on exit.
__device__ __forceinline__ void cta_det(const MeasArgs& a, const MeasSmem& sm, int j, const u64* xcol) {
    const int Wp = a.m.Wp, W = a.m.W;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    MeasWs* ws = a.ws;
    for (int w0 = 0; w0 < W; w0 += kMeasThreads) {
        const int w = w0 + tid;
        u64 bits = (w < W) ? ldcg(xcol + W + w) : 0ull;
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
    u64 ax = 0, az = 0;                                   // this thread's word of the running product
    const int Wq = (W + 31) & ~31;
    const int ngroups = max(1, min(kMeasThreads / Wq, (total + 7) / 8));
    const int myw = tid % Wq, myg = tid / Wq;
    auto multiply_list = [&](int cnt) {
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
        for (int i = tid; i < cnt; i += kMeasThreads) e += 2 * sign_bit(a.m.sgn, int(sm.targets[i]));
    };
    if (total <= kMaxTargets) {
        multiply_list(total);
    } else {
        // more partners than list slots (dense tableaux): column-order slices selected by rank
        for (int base = 0; base < total; base += kMaxTargets) {
            __syncthreads();
            int seen = 0;
            for (int w0 = 0; w0 < W; w0 += kMeasThreads) {
                const int w = w0 + tid;
                const u64 bits = (w < W) ? ldcg(xcol + W + w) : 0ull;
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
    e = warp_sum(e);
    if (lane == 0) sm.pe[warp] = e;
    __syncthreads();
    if (tid == 0) {
        int et = 0;
        for (int t = 0; t < kMeasWarps; ++t) et += sm.pe[t];
        et &= 3;
        if (et & 1) atomicOr(&ws->err, 1u);
        a.outcomes[j] = uint8_t(et >> 1); a.dets[j] = 1; a.done[j] = 1;
        atomicAdd(&ws->n_det, 1ull); atomicAdd(&ws->k_det, (u64)total); atomicAdd(&ws->ncommit, 1u);
        sm.cnt[0] = 0;
    }
    __syncthreads();
}

// dynamic smem: mask[RW] | P[2*Wp] | D[2*Wp] | acc[kMeasWarps][2*Wp]   (u64 each)
__global__ void __launch_bounds__(kMeasThreads, 1)
k_measure_block(MeasArgs a) {
    extern __shared__ __align__(16) u64 smem[];
    __shared__ __align__(8) u64 s_mbar;
    __shared__ int s_red[2];
    __shared__ int s_nrun, s_run[kMeasWarps * kSlotsPerWarp];
    __shared__ int s_nheavy, s_heavy[kMeasWarps * kSlotsPerWarp], s_pe[kMeasWarps], s_pk[kMeasWarps];
    __shared__ u32 s_piv;
    __shared__ int s_wcnt[kMeasWarps];
    __shared__ u32 s_wlist[kMeasWarps][kWarpList];
    __shared__ int s_cnt3[3];
    __shared__ u32 s_targets[kMaxTargets], s_support[kMaxSupport];
    __shared__ unsigned short s_mwords[kMaxMaskWords];
    const int RW = a.m.RW, Wp = a.m.Wp, W = a.m.W;
    MeasSmem sm;
    sm.mask = smem; sm.P = sm.mask + RW; sm.D = sm.P + 2 * Wp; sm.acc = sm.D + 2 * Wp;
    sm.mbar = &s_mbar; sm.pe = s_pe; sm.pk = s_pk;
    sm.cnt = s_cnt3; sm.targets = s_targets; sm.mwords = s_mwords; sm.support = s_support;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x;
    const int GW = G * kMeasWarps;
    const int WS = GW * kSlotsPerWarp;              // window size
    const int gw = blockIdx.x * kMeasWarps + warp;
    MeasWs* ws = a.ws;
    u32 epoch = 0;
    u32 tma_parity = 0;
    if (tid == 0) { mbar_init(&s_mbar, 1); s_cnt3[0] = 0; s_cnt3[1] = 0; s_cnt3[2] = 0; s_piv = 0xffffffffu; }
    __syncthreads();

    u64* acc_x = sm.acc + (size_t)warp * 2 * Wp;
    u64* acc_z = acc_x + Wp;

    int pos = 0;
    u32 wave = 1;
    u32 commits_seen = 0;
    int seqlen = 0, narrow = 0;
    u64 t_prof = a.prof ? gtime() : 0;
    while (pos < a.count) {
        const int wend = min(a.count, pos + WS);
        const int par = int(wave & 1);
        u32* wpiv = a.wpiv + (size_t)par * WS;
        uint8_t* wrun = a.wrun + (size_t)par * WS;
        // ------------------------------------------------------------ P1 -----
        if (blockIdx.x == 0 && tid == 0) ws->r0[(wave + 1) % 3] = 0xffffffffu;
        for (int slot = gw; pos + slot < wend; slot += GW) {
            const int j = pos + slot;
            if (__ldcg(a.done + j)) { if (lane == 0) wpiv[slot] = 0xfffffffeu; continue; }       // executed in an earlier wave
            const u64* xcol = a.m.cols + (size_t)(2 * a.qubits[j]) * RW;
            const u64 key = ((u64)wave << 32) | (u64)(0xffffffffu - (u32)j);
            u32 piv = 0xffffffffu;
            for (int w0 = 0; w0 < RW; w0 += 32 * kColChunk) {        // loads first (one L2 round trip per chunk)
                u64 cv[kColChunk];
#pragma unroll
                for (int t = 0; t < kColChunk; ++t) { const int w = w0 + 32 * t + lane; cv[t] = (w < RW) ? ldcg(xcol + w) : 0ull; }
#pragma unroll
                for (int t = 0; t < kColChunk; ++t) {
                    const int w = w0 + 32 * t + lane;
                    u64 v = cv[t];
                    if (v && w < W) piv = min(piv, u32(w * 64 + __ffsll((long long)v) - 1));
                    const int base = (w < W ? w : w - W) * 64;
                    while (v) { int b = __ffsll((long long)v) - 1; v &= v - 1; atomicMax(a.claim + base + b, key); }
                }
            }
            piv = warp_min(piv);
            if (lane == 0) {
                wpiv[slot] = piv;
                if (piv != 0xffffffffu) atomicMin(&ws->r0[wave % 3], (u32)j);
            }
        }
        SK_PROF(0);
        if (!grid_barrier(&ws->bar, epoch, &ws->err)) return;
        SK_PROF(1);
        const u32 r0 = __ldcg(&ws->r0[wave % 3]);
        if (tid == 0) s_nheavy = 0;
        __syncthreads();
        // ------------------------------------------------------------ P2 (+K4) --
        for (int slot = gw; pos + slot < wend; slot += GW) {
            const int j = pos + slot;
            const u32 piv = __ldcg(wpiv + slot);      // written by this warp in P1
            if (piv == 0xfffffffeu) { if (lane == 0) wrun[slot] = 0; continue; }
            const u64* xcol = a.m.cols + (size_t)(2 * a.qubits[j]) * RW;
            bool blocked = false;
            const bool isdet = piv == 0xffffffffu;
            if (lane == 0) s_wcnt[warp] = 0;
            __syncwarp();
            for (int w0 = 0; w0 < RW; w0 += 32 * kColChunk) {
                u64 cv[kColChunk];
#pragma unroll
                for (int t = 0; t < kColChunk; ++t) { const int w = w0 + 32 * t + lane; cv[t] = (w < RW) ? ldcg(xcol + w) : 0ull; }
#pragma unroll
                for (int t = 0; t < kColChunk; ++t) {
                    const int w = w0 + 32 * t + lane;
                    u64 v = cv[t];
                    const int base = (w < W ? w : w - W) * 64;
                    const bool chk = (u32)j >= r0;
                    while (v) {
                        int b = __ffsll((long long)v) - 1; v &= v - 1;
                        if (isdet) { const int ti = atomicAdd(&s_wcnt[warp], 1); if (ti < kWarpList) s_wlist[warp][ti] = u32(base + b); }
                        if (chk) {
                            const u64 c = ldcg(a.claim + base + b);
                            if ((u32)(c >> 32) == wave && (0xffffffffu - (u32)c) < (u32)j) blocked = true;
                        }
                    }
                }
            }
            blocked = __any_sync(0xffffffffu, blocked);
            if (lane == 0) wrun[slot] = uint8_t(!blocked && !isdet);
            if (blocked || !isdet) continue;
            __syncwarp();
            const int npart = s_wcnt[warp];
            if (npart > kWarpList) {                  // tree-reduced by the whole CTA below
                if (lane == 0) { int h = atomicAdd(&s_nheavy, 1); s_heavy[h] = slot; }
                continue;
            }
            int k;
            const int e = det_list_partial(a.m, s_wlist[warp], npart, 0, 1, acc_x, acc_z, lane, &k);
            if (lane == 0) {
                if (e & 1) atomicOr(&ws->err, 1u);
                a.outcomes[j] = uint8_t(e >> 1); a.dets[j] = 1; a.done[j] = 1;
                atomicAdd(&ws->n_det, 1ull); atomicAdd(&ws->k_det, (u64)k); atomicAdd(&ws->ncommit, 1u);
            }
        }
        __syncthreads();
        for (int h = 0; h < s_nheavy; ++h) {
            const int j = pos + s_heavy[h];
            cta_det(a, sm, j, a.m.cols + (size_t)(2 * a.qubits[j]) * RW);
        }
        if (blockIdx.x == 0 && tid == 0) atomicAdd(&ws->waves, 1ull);
        SK_PROF(2);
        if (r0 == 0xffffffffu) { pos = wend; ++wave; commits_seen = 0xffffffffu; continue; }   // window was all deterministic: done
        if (!grid_barrier(&ws->bar, epoch, &ws->err)) return;          // reads of the wave-start state done
        SK_PROF(3);

        // ------------------------------------------------------------ P3: K3 ----
        // this CTA owns window slots blockIdx.x, +G, +2G, ...: gather the runnable ones in parallel
        if (tid == 0) s_nrun = 0;
        __syncthreads();
        for (int i = tid; pos + blockIdx.x + i * G < wend; i += kMeasThreads) {
            const int slot = blockIdx.x + i * G;
            if (__ldcg(wrun + slot)) { int h = atomicAdd(&s_nrun, 1); s_run[h] = slot; }
        }
        __syncthreads();
        for (int h = 0; h < s_nrun; ++h) {
            const int slot = s_run[h];
            cta_random(a, sm, pos + slot, a.qubits[pos + slot], int(__ldcg(wpiv + slot)), tma_parity, false);
        }
        SK_PROF(4);
        if (!grid_barrier(&ws->bar, epoch, &ws->err)) return;
        SK_PROF(5);
        // ---- sequential mode: when a wave commits only a handful of measurements the block is
        // dependency-limited; CTA 0 then runs the next `seqlen` measurements strictly in order
        // with CTA-level synchronisation only (no grid barriers), the other CTAs wait.
        {
            const u32 nc = __ldcg(&ws->ncommit);
            const u32 committed = (commits_seen == 0xffffffffu) ? 0xffffu : nc - commits_seen;
            // a narrow wave is normal while the dependency frontier is still widening (round 1 of a
            // memory experiment needs ~20 waves); only a long run of narrow waves means the block is
            // inherently sequential
            narrow = (committed < (u32)a.seq_threshold) ? narrow + 1 : 0;
            seqlen = (narrow >= kNarrowWaves) ? min(kSeqMax, max(kSeqMin, seqlen * 2)) : 0;
        }
        if (seqlen > 0) {
            if (blockIdx.x == 0) {
                int j = pos, ran = 0;
                u64 t0s = a.prof ? gtime() : 0; const long long c0 = clock64(); const u64 tseq0 = t0s;
                for (; j < a.count && ran < seqlen; ++j) {
                    if (__ldcg(a.done + j)) continue;                   // uniform: every thread reads the same byte
                    const u32 q = a.qubits[j];
                    const u64* xcol = a.m.cols + (size_t)(2 * q) * RW;
                    u32 piv = 0xffffffffu;                      // s_piv was reset at the end of the previous iteration
                    for (int w = tid; w < W; w += kMeasThreads) {
                        u64 v = ldcg(xcol + w);
                        if (v) piv = min(piv, u32(w * 64 + __ffsll((long long)v) - 1));
                    }
                    piv = warp_min(piv);
                    if (lane == 0 && piv != 0xffffffffu) atomicMin(&s_piv, piv);
                    __syncthreads();
                    piv = s_piv;
                    u64 t1 = 0, t2 = 0;
                    if (a.prof && tid == 0) { t1 = gtime(); ws->seqprof[0] += t1 - t0s; }
                    if (piv == 0xffffffffu) cta_det(a, sm, j, xcol);
                    else cta_random(a, sm, j, q, int(piv), tma_parity, true);
                    if (a.prof && tid == 0) { t2 = gtime(); ws->seqprof[piv == 0xffffffffu ? 1 : 2] += t2 - t1; ws->seqprof[piv == 0xffffffffu ? 4 : 5] += 1; }
                    __threadfence();                                    // this measurement's updates before the next column read
                    if (tid == 0) s_piv = 0xffffffffu;                  // (everyone read s_piv before the CTA op's barriers)
                    __syncthreads();
                    if (a.prof && tid == 0) { t0s = gtime(); ws->seqprof[3] += t0s - t2; }
                    ++ran;
                }
                if (tid == 0) { atomicAdd(&ws->waves, (u64)ran); if (a.prof) { ws->seqprof[6] += (u64)(clock64() - c0); ws->seqprof[7] += gtime() - tseq0; } }
            }
            SK_PROF(6);
            if (!grid_barrier(&ws->bar, epoch, &ws->err)) return;
        }
        commits_seen = __ldcg(&ws->ncommit);
        // next window starts at the first measurement not yet executed (same value in every CTA)
        int first = 0x7fffffff;
        for (int jj = pos + tid; jj < wend; jj += kMeasThreads) if (!__ldcg(a.done + jj)) first = min(first, jj);   // no early exit: loads overlap
        if (tid == 0) s_red[0] = 0x7fffffff;
        __syncthreads();
        if (first != 0x7fffffff) atomicMin(&s_red[0], first);
        __syncthreads();
        pos = min(s_red[0], wend);
        ++wave;
        SK_PROF(7);
    }
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
