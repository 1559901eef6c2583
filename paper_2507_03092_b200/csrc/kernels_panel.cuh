// kernels_panel.cuh -- panel mode of k_measure_block, REPLICATED level-form path (the default for sparse panels).
//
// Same blocked elimination as described in kernels_measure.cuh (exact CHP semantics), organised so
// that no CTA ever waits for another one's symbolic work:
//   * the active rows of a panel travel as PAIRS (stabilizer i, destabilizer n+i) with their bits in the panel's columns;
//   * EVERY CTA runs the level-form symbolic factorisation of the panel on its own copy of that list in shared memory
//     (a few hundred pairs, 1-2 rounds for a surface-code panel): pivots, pivot histories, step masks and deterministic
//     partner sets are then local knowledge -- nothing is published, nobody polls;
//   * V: the value pivot row k has when it is used is the product of the panel-start rows in the closure C_k of its history
//     (all of them stabilizer rows: commuting, Hermitian, so order and grouping are free) -- every (step, word) is
//     independent, no recurrence; D1: panel-start partner products of the deterministic steps;        -- grid barrier --
//   * A: every touched pair replays its own step list with a thread per row word (8 pivot rows in flight), writes the row
//     and emits the pair's bits in the NEXT panel's columns; untouched pairs are gathered from the R form in the same phase;
//     D2: outcomes of the deterministic steps.                                                        -- grid barrier --
// A panel whose pair list outgrows the shared-memory slots returns to the general path in kernels_measure.cuh.
#pragma once
#include "common.cuh"

namespace skd {

struct LvShared {
    u32 piv[kPanelMax], cand[2][kPanelMax], pslot[kPanelMax], q[kPanelMax], q2[kPanelMax], eph[kPanelMax];
    u64 hist[kPanelMax], C[kPanelMax], Aany[2][kPanelMax], bpA[kPanelMax];
    uint8_t outc[kPanelMax];
    u64 ready, rr, forced[2], randmask, osign, psign;
    u32 P, nlist, bail;
    u32 wcnt[kMeasThreads / 32];
    int gpe[kMeasThreads / 32];
    u64 wN[kMeasThreads / 32], wZ[kMeasThreads / 32];
    // this CTA's deterministic steps of the current panel (D1 -> D2 across the grid barrier)
    int dj[kPanelMax], de[kPanelMax]; u64 dN[kPanelMax], dZ[kPanelMax]; int nd, dparts;
};

// geometry of the thread-per-word groups of the apply phase
__host__ __device__ inline int lv_group_threads(int W) { const int t = ((W + 31) / 32) * 32; return t < 32 ? 32 : t; }
// dynamic shared memory (bytes) the replicated path needs for a tableau with W words per half row on a grid of G CTAs
__host__ __device__ inline size_t lv_smem_bytes(int NS, int W, int Wp, int G, int B) {
    const int Pc = level_pair_cap(NS);
    const int TW = lv_group_threads(W), ng = kMeasThreads / TW;
    const int wpc = (W + G - 1) / G;
    size_t words = (size_t)5 * Pc + (size_t)(Pc + 1) / 2 /*id*/ + (size_t)(2 * Pc + 7) / 8 /*born, pvd*/ + 2;
    words += (size_t)W + 2;                      // touched-pair bitmap
    words += (size_t)ng * 2 * Wp;                // per-group row words (x then z)
    words += (size_t)B * 2 * wpc + 2;            // V: staged panel-start words of the pivot rows
    words += (size_t)(Pc + 1) / 2 + 2;           // D1 partner list
    return words * 8 + sizeof(LvShared) + 16;
}
__host__ __device__ inline bool lv_supported(int W) { return W <= kMeasThreads; }

__device__ __forceinline__ void group_sync(int gid, int TW) {
    if (TW == 32) __syncwarp(); else asm volatile("bar.sync %0, %1;" ::"r"(gid + 1), "r"(TW) : "memory");
}

// Gathers the pairs' bits in the columns q[0..Bn) from the R form: warp per 32 pair ids, lane per pair (consecutive qubits share
// one 8-byte load).  Pairs whose bit is set in `skip` (shared memory, may be null) are left out.  Entries (pid, sb, db) with any
// bit set are appended to the list (lh, lb) through the global counter *cnt.
__device__ __forceinline__ void lv_gather_pairs(const MeasArgs& a, const u32* q, int Bn, const u64* skip, u32* lh, u64* lb, u32* cnt,
                                                int first, int stride) {
    const int lane = threadIdx.x & 31;
    const int Wp = a.m.Wp, NS = a.NS;
    for (int g = first; g < NS / 32; g += stride) {
        const int pid = 32 * g + lane;
        const bool sk = skip && ((skip[pid >> 6] >> (pid & 63)) & 1ull);
        const u64* rs = a.m.rows + (size_t)(2 * pid) * Wp;
        const u64* rd = a.m.rows + (size_t)(2 * (NS + pid)) * Wp;
        u64 sbits = 0, dbits = 0;
        int lastw = -1; u64 ls = 0, ld = 0;
        for (int j0 = 0; j0 < Bn; j0 += 8) {
            u32 qq[8]; u64 vs[8], vd[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) qq[t] = (j0 + t < Bn) ? q[j0 + t] : 0xffffffffu;
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                const int wq = int(qq[t] >> 6), prev = t ? int(qq[t - 1] >> 6) : lastw;
                const bool ldit = !sk && qq[t] != 0xffffffffu && wq != prev;
                vs[t] = ldit ? ldcg(rs + wq) : 0ull; vd[t] = ldit ? ldcg(rd + wq) : 0ull;
            }
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                if (qq[t] == 0xffffffffu) continue;
                const int wq = int(qq[t] >> 6);
                if (wq == lastw) { vs[t] = ls; vd[t] = ld; } else { ls = vs[t]; ld = vd[t]; lastw = wq; }
                sbits |= ((vs[t] >> (qq[t] & 63)) & 1ull) << (j0 + t);
                dbits |= ((vd[t] >> (qq[t] & 63)) & 1ull) << (j0 + t);
            }
        }
        if (sk) { sbits = 0; dbits = 0; }
        const u32 am = __ballot_sync(0xffffffffu, (sbits | dbits) != 0);
        if (am) {
            u32 base = 0;
            if (lane == 0) base = atomicAdd(cnt, (u32)__popc(am));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (sbits | dbits) {
                const u32 at = base + __popc(am & ((1u << lane) - 1u));
                __stcg(lh + at, (u32)pid); __stcg(lb + 2 * (size_t)at, sbits); __stcg(lb + 2 * (size_t)at + 1, dbits);
            }
        }
    }
}

// shared-memory layout and geometry of the panel loop, re-derived at the top of every phase function (registers, no argument struct)
#define LV_LOCALS \
    extern __shared__ __align__(16) u64 sp[]; \
    constexpr u32 kInf = 0xffffffffu; constexpr int T = kMeasThreads; \
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5; \
    const int G = gridDim.x, bid = blockIdx.x; \
    const int NS = a.NS, W = a.m.W, Wp = a.m.Wp, B = a.B; \
    MeasWs* ws = a.ws; PanelInfo* info = a.info; \
    LvShared& ps = *reinterpret_cast<LvShared*>(sp); \
    u64* const sl = sp + (sizeof(LvShared) + 7) / 8; \
    const int Pc = level_pair_cap(NS); \
    u64* sb = sl; u64* db = sb + Pc; u64* Ms = db + Pc; u64* Md = Ms + Pc; u64* Dm = Md + Pc; \
    u32* id = reinterpret_cast<u32*>(Dm + Pc); \
    uint8_t* born = reinterpret_cast<uint8_t*>(id + Pc + (Pc & 1)); uint8_t* pvd = born + Pc; \
    u64* tb = reinterpret_cast<u64*>(pvd + Pc + ((8 - (2 * Pc) % 8) % 8)); \
    const int TW = lv_group_threads(W), ngroups = T / TW; \
    u64* gw = tb + W + 1; \
    const int wpc = (W + G - 1) / G; \
    u64* vs = gw + (size_t)ngroups * 2 * Wp; \
    u32* dl = reinterpret_cast<u32*>(vs + (size_t)B * 2 * wpc + 1); \
    const int gid = tid / TW, gt = tid - gid * TW; \
    const int NG = G * ngroups; \
    const int gwi = warp * G + bid, GW = G * (T / 32); \
    const size_t lcap = (size_t)32 * a.m.RW; \
    (void)kInf; (void)lane; (void)warp; (void)bid; (void)ws; (void)info; (void)sb; (void)db; (void)Ms; (void)Md; (void)Dm; (void)id; (void)born; (void)pvd; \
    (void)tb; (void)gw; (void)vs; (void)dl; (void)gid; (void)gt; (void)NG; (void)gwi; (void)GW; (void)lcap; (void)ngroups; (void)wpc; (void)Wp; (void)B

// F: level-form symbolic factorisation of the panel (every CTA, identical result).  P pairs in list buffer kpar.
__device__ __noinline__ void lv_factorise(const MeasArgs& a, int pos, int Bn, int kpar, int P) {
    LV_LOCALS;
    const u32* lh = a.alist_h + (size_t)kpar * lcap; const u64* lb = a.alist_b + (size_t)kpar * 2 * lcap;
    // the pair list is fetched while the per-step arrays are still being cleared by the caller's barrier: slots first, two per thread in flight
    u64 U = (Bn < 64) ? ((1ull << Bn) - 1ull) : ~0ull;
    // candidates and reach sets of a row for the round that works on the unfinished steps Un (buffer cb)
    auto contribute = [&](int s, u64 svv, u64 dvv, u64 Un, int cb) {
        const u64 sv = svv & Un;
        if (!sv) return;
        const u64 all = sv | (dvv & Un);
        const u32 key = (id[s] << 11) | u32(s);
        if (__popcll(sv) > kLevelK) {
            const int low = __ffsll((long long)sv) - 1;
            atomicMin(&ps.cand[cb][low], key); smem_or64(&ps.Aany[cb][low], all & bits_above(low)); smem_or64(&ps.forced[cb], 1ull << low);
        } else {
            u64 t = sv;
            while (t) {
                const int j = __ffsll((long long)t) - 1; t &= t - 1;
                atomicMin(&ps.cand[cb][j], key);
                smem_or64(&ps.Aany[cb][j], all & bits_above(j));
            }
        }
    };
    for (int s0 = tid; s0 < P; s0 += 2 * T) {
        const int s1 = s0 + T;
        const u32 i0 = __ldcg(lh + s0); const u64 a0 = ldcg(lb + 2 * (size_t)s0), b0 = ldcg(lb + 2 * (size_t)s0 + 1);
        u32 i1 = 0; u64 a1 = 0, b1 = 0;
        if (s1 < P) { i1 = __ldcg(lh + s1); a1 = ldcg(lb + 2 * (size_t)s1); b1 = ldcg(lb + 2 * (size_t)s1 + 1); }
        id[s0] = i0; sb[s0] = a0; db[s0] = b0; Ms[s0] = 0; Md[s0] = 0; Dm[s0] = 0; born[s0] = 0; pvd[s0] = 0;
        contribute(s0, a0, b0, U, 0);
        if (s1 < P) { id[s1] = i1; sb[s1] = a1; db[s1] = b1; Ms[s1] = 0; Md[s1] = 0; Dm[s1] = 0; born[s1] = 0; pvd[s1] = 0; contribute(s1, a1, b1, U, 0); }
    }
    for (int w = tid; w < W; w += T) tb[w] = 0;
    __syncthreads();
    int ntarget = 0, kdet = 0;
    bool isr[2] = {false, false}; u64 sgw[2] = {0, 0}; u32 spid[2] = {0, 0};      // warp 0: this lane's columns that turned out random
    for (int cb = 0;; cb ^= 1) {
        // ---- which steps are ready (warp 0; lane owns columns lane and lane + 32)
        if (warp == 0) {
            u64 Tm[2], Jm[2], Am[2], Js[2]; u32 cd[2]; bool inU[2], rnd[2], conf[2], hb[2];
            const u64 forced = ps.forced[cb];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int j = lane + 32 * h;
                inU[h] = (U >> j) & 1ull; cd[h] = ps.cand[cb][j]; rnd[h] = inU[h] && cd[h] != kInf;
                Tm[h] = 0; Jm[h] = 0; Am[h] = 0; Js[h] = 0; conf[h] = false;
                if (rnd[h]) {
                    const u32 slot = cd[h] & 2047u;
                    const u64 sv = sb[slot] & U, all = sv | (db[slot] & U);
                    Tm[h] = all & bits_above(j); Jm[h] = all & bits_below(j); Js[h] = sv & bits_below(j); Am[h] = ps.Aany[cb][j];
                    u64 t = Js[h];
                    while (t) { const int j2 = __ffsll((long long)t) - 1; t &= t - 1; if (ps.cand[cb][j2] == cd[h]) conf[h] = true; }
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
                if (!(rd[h] && rnd[h])) continue;
                const u32 slot = cd[h] & 2047u;
                ps.pslot[j] = slot; ps.bpA[j] = sb[slot] & bits_above(j);
                ps.piv[j] = id[slot]; ps.hist[j] = Ms[slot] | Js[h];
                isr[h] = true; spid[h] = id[slot]; sgw[h] = ldcg(a.m.sgn + (id[slot] >> 6));
            }
            const u64 rr = (u64)__ballot_sync(0xffffffffu, rd[0] && rnd[0]) | ((u64)__ballot_sync(0xffffffffu, rd[1] && rnd[1]) << 32);
            if (lane == 0) { ps.ready = ready; ps.rr = rr; }
        }
        __syncthreads();
        // ---- all ready steps at once; the same sweep offers the rows as candidates of the next round (other buffer) or -- after
        // the last round -- marks the touched pairs
        const u64 ready = ps.ready, rr = ps.rr;
        const u64 Un = U & ~ready;
        if (tid < kPanelMax) { ps.cand[cb][tid] = kInf; ps.Aany[cb][tid] = 0; }      // read by this round's warp 0 only: free again
        if (tid == 0) ps.forced[cb] = 0;
        for (int s = tid; s < P; s += T) {
            u64 sv = sb[s], dv = db[s];
            const u64 sh = sv & ready, dh = dv & ready;
            if (sh | dh) {
                int pl = -1;
                { u64 t = sh; while (t) { const int l = __ffsll((long long)t) - 1; t &= t - 1; if (ps.pslot[l] == (u32)s) { pl = l; break; } } }
                if (pl >= 0) {
                    // pivot of step pl: the ready steps below pl multiplied this row (they are in its history) and read or
                    // multiplied its old partner, which step pl then overwrites with the pivot row
                    const u64 lo = bits_below(pl);
                    ntarget += __popcll(sh & lo) + __popcll(dh & lo & rr);
                    Dm[s] |= dh & lo & ~rr;
                    dv = sv & bits_above(pl); sv = 0;
                    sb[s] = 0; db[s] = dv; Ms[s] = ps.hist[pl]; Md[s] = 0; born[s] = uint8_t(pl + 1); pvd[s] = 1;
                } else {
                    if (sh) {
                        u64 t = sh;
                        while (t) { const int l = __ffsll((long long)t) - 1; t &= t - 1; sv ^= ps.bpA[l]; }
                        sb[s] = sv; Ms[s] |= sh; ntarget += __popcll(sh);
                    }
                    if (dh) {
                        u64 t = dh & rr;
                        while (t) { const int l = __ffsll((long long)t) - 1; t &= t - 1; dv ^= ps.bpA[l]; }
                        db[s] = dv; Md[s] |= dh & rr; Dm[s] |= dh & ~rr; ntarget += __popcll(dh & rr);
                    }
                }
            }
            if (Un) contribute(s, sv, dv, Un, cb ^ 1);
            else {
                if (pvd[s] || Ms[s] || Md[s] || born[s]) { const u32 pid = id[s]; atomicOr(reinterpret_cast<u32*>(tb) + (pid >> 5), 1u << (pid & 31)); }
                kdet += __popcll(Dm[s]);
            }
        }
        U = Un;
        __syncthreads();
        if (!U) break;
    }
    // ---- closure of the histories, random mask, panel-start signs of the pivot rows, touched pairs
    if (warp == 0) {
        const u64 rm = (u64)__ballot_sync(0xffffffffu, isr[0]) | ((u64)__ballot_sync(0xffffffffu, isr[1]) << 32);
        const u64 os = (u64)__ballot_sync(0xffffffffu, isr[0] && ((sgw[0] >> (spid[0] & 63)) & 1ull)) | ((u64)__ballot_sync(0xffffffffu, isr[1] && ((sgw[1] >> (spid[1] & 63)) & 1ull)) << 32);
        u64 C0 = isr[0] ? 1ull << lane : 0ull, C1 = isr[1] ? 1ull << (lane + 32) : 0ull;
        const u64 h0 = isr[0] ? ps.hist[lane] : 0ull, h1 = isr[1] ? ps.hist[lane + 32] : 0ull;
        u64 nzh = (u64)__ballot_sync(0xffffffffu, h0 != 0) | ((u64)__ballot_sync(0xffffffffu, h1 != 0) << 32);
        while (nzh) {        // ascending: the closures of the steps in hist_k are final when k is reached
            const int k = __ffsll((long long)nzh) - 1; nzh &= nzh - 1;
            const u64 hk = ps.hist[k];
            const u64 x = (((hk >> lane) & 1ull) ? C0 : 0ull) ^ (((hk >> (lane + 32)) & 1ull) ? C1 : 0ull);
            const u64 r = warp_xor64(x);
            if (lane == (k & 31)) { if (k < 32) C0 ^= r; else C1 ^= r; }
        }
        ps.C[lane] = C0; ps.C[lane + 32] = C1;
        if (isr[0]) ps.outc[lane] = uint8_t(counter_bit(a.seed, a.ordinal0 + (uint64_t)(pos + lane)));
        if (isr[1]) ps.outc[lane + 32] = uint8_t(counter_bit(a.seed, a.ordinal0 + (uint64_t)(pos + lane + 32)));
        if (lane == 0) { ps.randmask = rm; ps.osign = os; }
    }
    if (bid == 0) {      // counters: one CTA reports
        ntarget = warp_sum(ntarget); kdet = warp_sum(kdet);
        if (lane == 0) { if (ntarget) atomicAdd(&ws->k_rand, (u64)ntarget); if (kdet) atomicAdd(&ws->k_det, (u64)kdet); }
    }
    __syncthreads();
    const u64 randmask = ps.randmask;
    const u64 allmask = (Bn < 64) ? ((1ull << Bn) - 1ull) : ~0ull;
    const u64 detmask = ~randmask & allmask;
    if (bid == 0 && tid == 0) {
        const int nrand = __popcll(randmask);
        atomicAdd(&ws->n_rand, (u64)nrand); atomicAdd(&ws->n_det, (u64)(Bn - nrand)); atomicAdd(&ws->waves, 1ull); atomicAdd(&ws->panels, 1ull);
    }
}

// V + D1: pivot values (this CTA's words of every step) and the panel-start partner products of this CTA's deterministic steps
__device__ __noinline__ void lv_values(const MeasArgs& a, int pos, int Bn, int kpar, int P) {
    LV_LOCALS;
    const u64 randmask = ps.randmask;
    const u64 allmask = (Bn < 64) ? ((1ull << Bn) - 1ull) : ~0ull;
    const u64 detmask = ~randmask & allmask;
    // ================================================================ V: pivot values (words [wlo, whi) of every step) =====
    {
        const int wlo = min(W, bid * wpc), nw = min(W, wlo + wpc) - wlo;
        const int nitems = Bn * 2 * nw;
        for (int i0 = tid; i0 < nitems; i0 += 4 * T) {
            u64 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = i0 + u * T;
                v[u] = 0;
                if (i < nitems) {
                    const int k = i / (2 * nw), r = i - k * 2 * nw, half = r / nw, t = r - half * nw;
                    const u32 pk = ps.piv[k];
                    if (pk != kInf) v[u] = ldcg(a.m.rows + (size_t)(2 * pk + half) * Wp + wlo + t);
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = i0 + u * T;
                if (i < nitems) { const int k = i / (2 * nw), r = i - k * 2 * nw, half = r / nw, t = r - half * nw; vs[(size_t)(2 * k + half) * wpc + t] = v[u]; }
            }
        }
        __syncthreads();
        for (int i = tid; i < Bn * nw; i += T) {
            const int k = i / nw, t = i - k * nw;
            if (!((randmask >> k) & 1ull)) continue;
            u64 ax = 0, az = 0, c = ps.C[k];
            int e = 0;
            while (c) {
                const int l = __ffsll((long long)c) - 1; c &= c - 1;
                const u64 bx = vs[(size_t)(2 * l) * wpc + t], bz = vs[(size_t)(2 * l + 1) * wpc + t];
                e += g_word(bx, bz, ax, az); ax ^= bx; az ^= bz;
            }
            __stcg(a.pivbuf + (size_t)(2 * k) * Wp + wlo + t, ax); __stcg(a.pivbuf + (size_t)(2 * k + 1) * Wp + wlo + t, az);
            if (e & 3) atomicAdd(&info->eph[kpar][k], (u32)(e & 3));
        }
    }
    // ================================================================ D1: panel-start partner products =====
    // A deterministic step's product is cut into NP parts by the pair index (NP = 4 while there are CTAs for it): part p of the
    // idx-th step belongs to CTA G-1 - (p*ndet + idx) % G (from the far end: the first CTAs own the most V words and apply work).  The owner of
    // part 0 keeps its partial product in detacc[j] and its record in shared memory -- it also does D2 -- the others leave theirs
    // in detacc[p][j] and info->dp_*: all factors are stabilizer rows (commuting), D2 folds the parts in any order.
    {
        const int ndet = __popcll(detmask);
        const int NP = ndet ? max(1, min(4, G / ndet)) : 1;
        const int Pq = (P + NP - 1) / NP;
        const size_t part_stride = (size_t)B * 2 * Wp;
        if (tid == 0) ps.dparts = NP;
        // this CTA's items: G-1-bid, G-1-bid + G, .. (at most two: NP * ndet <= 256) -- no loop over everybody's items
        for (int it = G - 1 - bid; it < NP * ndet; it += G) {
            const int part = it / ndet, my = it - part * ndet;        // part-major: the owners of part 0 (who also do D2) are the last CTAs, which have the least apply work
            u64 bits = detmask;
            for (int i = 0; i < my; ++i) bits &= bits - 1;             // the my-th deterministic step
            const int j = __ffsll((long long)bits) - 1;
            {
            const int s_lo = part * Pq, s_hi = min(P, s_lo + Pq);
            // partner list: original destabilizers (their stabilizer's index), N = XOR of those stabilizers' step masks, Z = earlier
            // steps of this panel whose +-Z row is a partner
            __syncthreads();
            if (tid == 0) ps.nlist = 0;
            __syncthreads();
            u64 N = 0, Z = 0;
            for (int s0 = s_lo; s0 < s_hi; s0 += T) {
                const int s = s0 + tid;
                bool orig = false;
                if (s < s_hi && ((Dm[s] >> j) & 1ull)) {
                    const int b = born[s];
                    if (b == 0 || j < b - 1) { orig = true; N ^= Ms[s]; } else Z |= 1ull << (b - 1);
                }
                const u32 bal = __ballot_sync(0xffffffffu, orig);
                if (bal) {
                    u32 base = 0;
                    if (lane == 0) base = atomicAdd(&ps.nlist, (u32)__popc(bal));
                    base = __shfl_sync(0xffffffffu, base, 0);
                    if (orig) dl[base + __popc(bal & ((1u << lane) - 1u))] = id[s];
                }
            }
            N = warp_xor64(N); Z = warp_or64(Z);
            if (lane == 0) { ps.wN[warp] = N; ps.wZ[warp] = Z; }
            __syncthreads();
            const int cnt = int(ps.nlist);
            // the partners' sign words are requested before the rows, used after them: one round trip instead of two in a row
            const u64 sgw = tid < cnt ? ldcg(a.m.sgn + (dl[tid] >> 6)) : 0ull;
            // product of the listed stabilizer rows: the groups split the list, a thread owns one word, 8 rows in flight
            u64 ax = 0, az = 0; int e = 0;
            if (gid < ngroups && gt < W) {
                for (int i0 = gid; i0 < cnt; i0 += 8 * ngroups) {
                    u64 sx[8], sz[8];
#pragma unroll
                    for (int t = 0; t < 8; ++t) {
                        const int i = i0 + t * ngroups;
                        if (i < cnt) { const u64* rx = a.m.rows + (size_t)(2 * dl[i]) * Wp; sx[t] = ldcg(rx + gt); sz[t] = ldcg(rx + Wp + gt); }
                        else { sx[t] = 0; sz[t] = 0; }
                    }
#pragma unroll
                    for (int t = 0; t < 8; ++t) { e += g_word(sx[t], sz[t], ax, az); ax ^= sx[t]; az ^= sz[t]; }
                }
            }
            if (tid < cnt) e += 2 * int((sgw >> (dl[tid] & 63u)) & 1ull);
            for (int i = tid + T; i < cnt; i += T) e += 2 * sign_bit(a.m.sgn, int(dl[i]));
            if (ngroups > 1) {       // fold the groups' partial products (commuting factors: any grouping)
                if (gid > 0 && gid < ngroups && gt < W) { gw[(size_t)gid * 2 * Wp + gt] = ax; gw[(size_t)gid * 2 * Wp + Wp + gt] = az; }
                __syncthreads();
                if (gid == 0 && gt < W)
                    for (int g = 1; g < ngroups; ++g) {
                        const u64 bx = gw[(size_t)g * 2 * Wp + gt], bz = gw[(size_t)g * 2 * Wp + Wp + gt];
                        e += g_word(bx, bz, ax, az); ax ^= bx; az ^= bz;
                    }
            }
            u64* acc = a.detacc + (size_t)part * part_stride;
            if (gid == 0 && gt < W) { __stcg(acc + (size_t)(2 * j) * Wp + gt, ax); __stcg(acc + (size_t)(2 * j + 1) * Wp + gt, az); }
            e = warp_sum(e);
            if (lane == 0) ps.gpe[warp] = e;
            __syncthreads();
            if (tid == 0) {
                int et = 0; u64 Nt = 0, Zt = 0;
                for (int t = 0; t < T / 32; ++t) { et += ps.gpe[t]; Nt ^= ps.wN[t]; Zt |= ps.wZ[t]; }
                Nt &= randmask & bits_below(j);
                if (part == 0) { const int k = ps.nd++; ps.dj[k] = j; ps.de[k] = et & 3; ps.dN[k] = Nt; ps.dZ[k] = Zt; }
                else { info->dp_e[part - 1][j] = et & 3; info->dp_N[part - 1][j] = Nt; info->dp_Z[part - 1][j] = Zt; }
            }
            }
        }
    }
}

// after the first grid barrier: signs of the pivot values, D2 (outcomes of this CTA's deterministic steps), A (touched pairs)
__device__ __noinline__ void lv_apply(const MeasArgs& a, int pos, int Bn, int Bn2, int kpar, int P) {
    LV_LOCALS;
    const u64 randmask = ps.randmask;
    u32* lh2 = a.alist_h + (size_t)(kpar ^ 1) * lcap; u64* lb2 = a.alist_b + (size_t)(kpar ^ 1) * 2 * lcap;
    // ================================================================ after the barrier: signs of the pivot values =====
    if (tid < kPanelMax) {
        const bool r = (randmask >> tid) & 1ull;
        const u32 ek = r ? __ldcg(&info->eph[kpar][tid]) + 2u * (u32)__popcll(ps.C[tid] & ps.osign) : 0u;
        const u32 odd = __ballot_sync(0xffffffffu, r && (ek & 1u)), sg = __ballot_sync(0xffffffffu, r && ((ek >> 1) & 1u));
        if (lane == 0) { reinterpret_cast<u32*>(&ps.psign)[tid >> 5] = sg; if (odd) atomicOr(&ws->err, 1u); }
    }
    if (bid == 0) {       // housekeeping: the phase sums of the previous panel and the consumed list counter
        if (tid < kPanelMax) info->eph[kpar ^ 1][tid] = 0;
        if (tid == 0) info->lvcount[kpar] = 0;
    }
    __syncthreads();
    const u64 psign = ps.psign;
    // ================================================================ D2: outcomes of this CTA's deterministic steps =====
    const int NP = ps.dparts;
    for (int k = 0; k < ps.nd; ++k) {
        const int j = ps.dj[k];
        u64 N = ps.dN[k], Z = ps.dZ[k];
        int ep = 0;
        for (int p = 1; p < NP; ++p) { N ^= __ldcg(&info->dp_N[p - 1][j]); Z |= __ldcg(&info->dp_Z[p - 1][j]); ep += __ldcg(&info->dp_e[p - 1][j]); }
        u64 ax = 0, az = 0; int e = 0;
        if (gid == 0 && gt < W) {
            ax = ldcg(a.detacc + (size_t)(2 * j) * Wp + gt); az = ldcg(a.detacc + (size_t)(2 * j + 1) * Wp + gt);
            if (NP > 1) {          // the other CTAs' parts of the partner product (all loads in flight at once)
                u64 px[3], pz[3];
#pragma unroll
                for (int p = 1; p < 4; ++p) if (p < NP) { const u64* acc = a.detacc + (size_t)p * B * 2 * Wp; px[p - 1] = ldcg(acc + (size_t)(2 * j) * Wp + gt); pz[p - 1] = ldcg(acc + (size_t)(2 * j + 1) * Wp + gt); }
#pragma unroll
                for (int p = 1; p < 4; ++p) if (p < NP) { e += g_word(px[p - 1], pz[p - 1], ax, az); ax ^= px[p - 1]; az ^= pz[p - 1]; }
            }
            if (gt == 0) e += ep;
            u64 b = N;
            while (b) {
                const int l = __ffsll((long long)b) - 1; b &= b - 1;
                const u64 bx = ldcg(a.pivbuf + (size_t)(2 * l) * Wp + gt), bz = ldcg(a.pivbuf + (size_t)(2 * l + 1) * Wp + gt);
                e += g_word(bx, bz, ax, az); ax ^= bx; az ^= bz;
            }
            b = Z;
            while (b) {        // (+-Z_{q_l}) * acc
                const int l = __ffsll((long long)b) - 1; b &= b - 1;
                const u32 ql = ps.q[l];
                if (int(ql >> 6) == gt) { const u64 zb = 1ull << (ql & 63); e += g_word(0ull, zb, ax, az) + 2 * int(ps.outc[l]); az ^= zb; }
            }
            if (gt == 0) e += ps.de[k] + 2 * __popcll(N & psign);
        }
        e = warp_sum(e);
        if (lane == 0) ps.gpe[warp] = e;
        __syncthreads();
        if (tid == 0) {
            int et = 0;
            for (int t = 0; t < (TW + 31) / 32; ++t) et += ps.gpe[t];
            et &= 3;
            if (et & 1) atomicOr(&ws->err, 1u);
            a.outcomes[pos + j] = uint8_t(et >> 1); a.dets[pos + j] = 1;
        }
        __syncthreads();
    }
    // ================================================================ A: touched pairs, a group per pair =====
    if (gid < ngroups) {
        u64* gx = gw + (size_t)gid * 2 * Wp;        // this group's new x words (for the next panel's bits)
        const int gw0 = gid * (TW / 32);            // first warp of the group
        for (int s = bid * ngroups + gid; s < P; s += NG) {
            const bool pv = pvd[s] != 0;
            const int b = born[s];
            const u64 ms = Ms[s], md = Md[s];
            if (!(pv || ms || md || b)) continue;
#ifdef SK_PANEL_TRACE
            const u64 t_pair = a.prof ? gtime() : 0;
#endif
            const u32 pid = id[s];
            u64 rbs = 0, rbd = 0;
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                const u32 h = half ? (u32)NS + pid : pid;
                u64* tx = a.m.rows + (size_t)(2 * h) * Wp;
                u64* sg = a.m.sgn + (h >> 6);
                const u64 hbit = 1ull << (h & 63);
                u64 M = half ? md : ms;
                bool touched = true;
                u64 ax = 0, az = 0; int e = 0;
                if (!half && pv) {
                    // the pivot of step b-1: -> +-Z_q with the counter RNG bit of its ordinal
                    const int k = b - 1;
                    const u32 q = ps.q[k];
                    if (gt < W) { __stcg(tx + gt, 0ull); __stcg(tx + Wp + gt, (gt == int(q >> 6)) ? (1ull << (q & 63)) : 0ull); }
                    if (gt == 0) { if (ps.outc[k]) atomicOr(sg, hbit); else atomicAnd(sg, ~hbit); a.outcomes[pos + k] = ps.outc[k]; a.dets[pos + k] = 0; }
                    continue;       // no x bits: nothing to emit for the next panel
                } else if (half && b) {
                    // overwritten destabilizer: starts as the pivot value of step b-1, then the later steps
                    const int k = b - 1;
                    if (gt < W) { ax = ldcg(a.pivbuf + (size_t)(2 * k) * Wp + gt); az = ldcg(a.pivbuf + (size_t)(2 * k + 1) * Wp + gt); }
                    if (gt == 0) e = 2 * int((psign >> k) & 1ull);
                } else if (M) {
                    if (gt < W) { ax = ldcg(tx + gt); az = ldcg(tx + Wp + gt); }
                    if (gt == 0) e = 2 * int((ldcg(sg) >> (h & 63)) & 1ull);
                } else touched = false;
                if (touched) {
                    if (gt < W) {
                        u64 bits = M;
                        while (bits) {
                            int ls[8]; int nl = 0;
#pragma unroll
                            for (int t = 0; t < 8; ++t) { ls[t] = 0; if (bits) { ls[t] = __ffsll((long long)bits) - 1; bits &= bits - 1; nl = t + 1; } }
                            u64 bx[8], bz[8];
#pragma unroll
                            for (int t = 0; t < 8; ++t) { bx[t] = 0; bz[t] = 0; if (t < nl) { bx[t] = ldcg(a.pivbuf + (size_t)(2 * ls[t]) * Wp + gt); bz[t] = ldcg(a.pivbuf + (size_t)(2 * ls[t] + 1) * Wp + gt); } }
                            // the eight factors as a tree (pairs, quads, then onto the row): same product and, by associativity, the same
                            // phase exponent as one after the other -- with a dependency depth of four instead of eight
#pragma unroll
                            for (int t = 0; t < 8; t += 2) { e += g_word(bx[t + 1], bz[t + 1], bx[t], bz[t]); bx[t] ^= bx[t + 1]; bz[t] ^= bz[t + 1]; }
#pragma unroll
                            for (int t = 0; t < 8; t += 4) { e += g_word(bx[t + 2], bz[t + 2], bx[t], bz[t]); bx[t] ^= bx[t + 2]; bz[t] ^= bz[t + 2]; }
                            e += g_word(bx[0], bz[0], ax, az); ax ^= bx[0]; az ^= bz[0];
                            e += g_word(bx[4], bz[4], ax, az); ax ^= bx[4]; az ^= bz[4];
                        }
                        __stcg(tx + gt, ax); __stcg(tx + Wp + gt, az);
                        gx[gt] = ax;
                    }
                    if (gt == 0) e += 2 * __popcll(M & psign);
                    e = warp_sum(e);
                    if (lane == 0) ps.gpe[warp] = e;
                    group_sync(gid, TW);
                    if (gt == 0) {
                        int et = 0;
                        for (int t = 0; t < TW / 32; ++t) et += ps.gpe[gw0 + t];
                        et &= 3;
                        if (et & 1) atomicOr(&ws->err, 1u);
                        if (et >> 1) atomicOr(sg, hbit); else atomicAnd(sg, ~hbit);
                    }
                }
                // the row's bits in the next panel's columns: from the new x words, or from the R form if the row was not touched
                if (Bn2 > 0 && gt < 32) {
                    const u32 q0 = ps.q2[gt], q1 = ps.q2[gt + 32];
                    u32 b0 = 0, b1 = 0;
                    if (touched) {
                        if (q0 != kInf) b0 = u32((gx[q0 >> 6] >> (q0 & 63)) & 1ull);
                        if (q1 != kInf) b1 = u32((gx[q1 >> 6] >> (q1 & 63)) & 1ull);
                    } else {
                        if (q0 != kInf) b0 = u32((ldcg(tx + (q0 >> 6)) >> (q0 & 63)) & 1ull);
                        if (q1 != kInf) b1 = u32((ldcg(tx + (q1 >> 6)) >> (q1 & 63)) & 1ull);
                    }
                    const u64 rb = (u64)__ballot_sync(0xffffffffu, b0) | ((u64)__ballot_sync(0xffffffffu, b1) << 32);
                    if (half) rbd = rb; else rbs = rb;
                }
                group_sync(gid, TW);        // gx and gpe are reused by the next row
            }
#ifdef SK_PANEL_TRACE
            if (a.prof && gt == 0)      // debug: the longest pair of the launch: ns << 24 | steps of the stabilizer << 16 | of the destabilizer << 8 | born, pivot flags
                atomicMax((unsigned long long*)&ws->cprof[15], ((gtime() - t_pair) << 24) | ((u64)__popcll(ms) << 16) | ((u64)__popcll(md) << 8) | (u64)((b ? 2 : 0) | (pv ? 1 : 0)));
#endif
            if (gt == 0 && (rbs | rbd)) {
                const u32 at = atomicAdd(&info->lvcount[kpar ^ 1], 1u);
                __stcg(lh2 + at, pid); __stcg(lb2 + 2 * (size_t)at, rbs); __stcg(lb2 + 2 * (size_t)at + 1, rbd);
            }
        }
    }
}

// The panel loop.  Returns the position it stopped at: a.count when the block is finished, or the start of a panel that
// needs the general path (pair list larger than the slots).  All CTAs return the same value.
__device__ __noinline__ int panel_levels_loop(const MeasArgs& a, int pos, u32& epoch) {
    LV_LOCALS;
    int kpar = 0;
    bool have_list = false;
    u64 t_prof = a.prof ? gtime() : 0;
    u64 t_cta = 0;
#define LV_CSTART() do { if (a.prof && tid == 0) t_cta = gtime(); } while (0)
#define LV_CPROF(k) do { if (a.prof && tid == 0 && bid < 160) { const u64 _n = gtime(); ws->ctaphase[bid * 4 + (k)] += _n - t_cta; t_cta = _n; } } while (0)
#define LV_PROF(k) do { if (a.prof && bid == 0 && tid == 0) { const u64 _n = gtime(); ws->prof[k] += _n - t_prof; t_prof = _n; } } while (0)
    // debug timeline of panels 20..27 of the launch (SK_DEBUG_PROF): CTAs {0, G/2, G-1}: start, F done, V+D1 done, barrier 1 left, A done
    // (thread 0), barrier 2 left; row of CTA 0, slots 6 / 7: the last CTA's arrival at barrier 2 / 1; row of CTA G/2, slot 6: who that was
    // (compiled in with -DSK_PANEL_TRACE only: the extra code costs the production kernel registers -- 0.25 ms at d=71)
#ifdef SK_PANEL_TRACE
    const int tsel = bid == 0 ? 0 : (bid == G / 2 ? 1 : (bid == G - 1 ? 2 : -1));
    int pidx = 0;
#define LV_TRACE(ev) do { if (a.prof && tid == 0 && tsel >= 0 && pidx >= 20 && pidx < 28) ws->trace[((pidx - 20) * 3 + tsel) * 8 + (ev)] = gtime(); } while (0)
#define LV_PLOG(k) do { if (a.prof && tid == 0 && pidx < 160) { if ((k) & 1) atomicMax((unsigned long long*)&ws->ptl[pidx * 6 + (k)], (unsigned long long)gtime()); else if (bid == 0) ws->ptl[pidx * 6 + (k)] = gtime(); } } while (0)
#define LV_ARRIVE(slot) do { if (a.prof) { __syncthreads(); if (tid == 0 && pidx >= 20 && pidx < 28) { \
        atomicMax((unsigned long long*)&ws->trace[((pidx - 20) * 3) * 8 + (slot)], (unsigned long long)gtime()); \
        if ((slot) == 6) atomicMax((unsigned long long*)&ws->trace[((pidx - 20) * 3 + 1) * 8 + 6], ((unsigned long long)(gtime() & 0xffffffffffull) << 8) | (unsigned long long)bid); } } } while (0)
#else
#define LV_TRACE(ev) do { } while (0)
#define LV_PLOG(k) do { } while (0)
#define LV_ARRIVE(slot) do { } while (0)
#endif
    while (pos < a.count) {
        const int Bn = min(B, a.count - pos), Bn2 = min(B, a.count - pos - Bn);
        u32* lh = a.alist_h + (size_t)kpar * lcap; u64* lb = a.alist_b + (size_t)kpar * 2 * lcap;
        u32* lh2 = a.alist_h + (size_t)(kpar ^ 1) * lcap; u64* lb2 = a.alist_b + (size_t)(kpar ^ 1) * 2 * lcap;
        if (tid < kPanelMax) {
            ps.q[tid] = (tid < Bn) ? a.qubits[pos + tid] : kInf; ps.q2[tid] = (tid < Bn2) ? a.qubits[pos + Bn + tid] : kInf;
            ps.piv[tid] = kInf; ps.hist[tid] = 0; ps.C[tid] = 0; ps.cand[0][tid] = kInf; ps.cand[1][tid] = kInf; ps.Aany[0][tid] = 0; ps.Aany[1][tid] = 0; ps.outc[tid] = 0;
        }
        if (tid == 0) { ps.forced[0] = 0; ps.forced[1] = 0; ps.nd = 0; }
        __syncthreads();
        if (!have_list) {
            lv_gather_pairs(a, ps.q, Bn, nullptr, lh, lb, &info->lvcount[kpar], gwi, GW);
            LV_PROF(2);
            if (!grid_barrier(&ws->bar, epoch, &ws->err)) return -1;
            LV_PROF(7);
        }
        // ================================================================ F (every CTA, identical result) =====
        LV_CSTART(); LV_TRACE(0); LV_PLOG(0);
        const u32 A = __ldcg(&info->lvcount[kpar]);
        if (A > (u32)Pc || A > (u32)a.row_cap) {
            // too many active pairs for the slots: hand the panel to the general path (which gathers for itself)
            if (!grid_barrier(&ws->bar, epoch, &ws->err)) return -1;
            if (bid == 0) { if (tid == 0) info->lvcount[kpar] = 0; if (tid < kPanelMax) { info->eph[0][tid] = 0; info->eph[1][tid] = 0; } }
            return pos;
        }
        const int P = int(A);
#ifdef SK_PANEL_TRACE
        if (a.prof && bid == 0 && tid == 0 && pidx < 160) ws->ptl[pidx * 6 + 5] = (u64)P;
#endif
        lv_factorise(a, pos, Bn, kpar, P);
        LV_PROF(3); LV_CPROF(1); LV_TRACE(1);
        lv_values(a, pos, Bn, kpar, P);
        LV_PROF(4); LV_CPROF(2); LV_TRACE(2); LV_ARRIVE(7); LV_PLOG(1);
        if (!grid_barrier(&ws->bar, epoch, &ws->err)) return -1;
        LV_PROF(7); LV_CSTART(); LV_TRACE(3); LV_PLOG(2);
        lv_apply(a, pos, Bn, Bn2, kpar, P);
        LV_CPROF(3);
        // the untouched pairs' bits in the next panel's columns, straight from the R form (from the far end of the warp index space)
        if (Bn2 > 0) lv_gather_pairs(a, ps.q2, Bn2, tb, lh2, lb2, &info->lvcount[kpar ^ 1], GW - 1 - gwi, GW);
        LV_PROF(5); LV_CPROF(0); LV_TRACE(4); LV_ARRIVE(6); LV_PLOG(3);
        if (!grid_barrier(&ws->bar, epoch, &ws->err)) return -1;
        LV_PROF(7); LV_TRACE(5); LV_PLOG(4);
        have_list = Bn2 > 0;
        kpar ^= 1;
        pos += Bn;
#ifdef SK_PANEL_TRACE
        ++pidx;
#endif
    }
#undef LV_PROF
#undef LV_TRACE
#undef LV_PLOG
#undef LV_ARRIVE
#undef LV_CPROF
#undef LV_CSTART
    return pos;
}

}  // namespace skd
