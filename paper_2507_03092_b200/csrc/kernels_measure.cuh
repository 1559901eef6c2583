// kernels_measure.cuh -- K2/K3/K4: a block of consecutive Z measurements executed by
// ONE persistent cooperative kernel (no host round trips; the branch taken is
// data dependent).  Exact CHP semantics (Algorithm 1):
// results are bit-identical to measuring one qubit at a time, in order.
//
// Scheduler (per wave):
//   A  every warp takes one pending measurement j (window = #warps in the grid):
//      pivot search = scan of the stabilizer half of column x_q in the C form
//      (contiguous, warp ballot + min) -- K2.  If there is no pivot the
//      measurement is deterministic and the warp evaluates it at once from the
//      read-only R form: ordered product of the stabilizer partners of the
//      destabilizers with x_q = 1, phase by popcounts (mod 4) -- K4.  A random
//      one only publishes (j, pivot) with a 64-bit atomicMin.
//   -- grid barrier --
//      f = first random measurement of the window.  Everything before f is final
//      (deterministic measurements do not modify the tableau).
//   B  if f exists, the whole grid performs that one random measurement -- K3:
//      stage column mask + pivot row P + old destabilizer row D in shared memory
//      (1-D TMA bulk copies, mbarrier), barrier, then concurrently
//        B1 R form: rowsum(i, p) for every i in the mask (warp per row, P from smem)
//        B2 C form: column_j ^= mask for every j in supp(P)   (word parallel)
//        B3 C form: bit fixes for the overwritten rows p and p+n ; sign bits ; record
//        B4 R form: row p+n := P ; row p := Z_q
//      barrier; the next window starts at f+1.
// Both forms stay valid, so later measurements (and gate layers) need no
// re-transposition.  Row i = p+n is skipped in B1 (it is overwritten; SURVEY.md
// section 7 "rowsum on the pivot's own destabilizer").
//
// Roofline: HBM/L2.  Algorithmic bytes: random  RW*8 + 16W + k*32W + 32W ;
// deterministic  RW*8/2 + k*16W  -- reported from the k counters kept here.
#pragma once
#include "common.cuh"

namespace skd {

struct MeasWs {
    u32 bar;            // grid barrier counter (zeroed before each launch)
    u32 err;            // bit0 odd phase (invariant), bit31 barrier timeout, bit30 tma timeout
    u64 first[3];       // per-wave (j << 32 | pivot), min-reduced; 3 slots rotate
    u64 n_rand, n_det, k_rand, k_det, waves;
};

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
};

constexpr int kMeasThreads = 512;
constexpr int kMeasWarps = kMeasThreads / 32;

// dynamic smem: mask[RW] | P[2*Wp] | D[2*Wp] | acc[kMeasWarps][2*Wp]   (u64 each)
__global__ void __launch_bounds__(kMeasThreads, 1)
k_measure_block(MeasArgs a) {
    extern __shared__ __align__(16) u64 smem[];
    __shared__ __align__(8) u64 s_mbar;
    const int RW = a.m.RW, Wp = a.m.Wp, W = a.m.W, NS = a.NS;
    u64* s_mask = smem;
    u64* s_P = s_mask + RW;
    u64* s_D = s_P + 2 * Wp;
    u64* s_acc = s_D + 2 * Wp;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int GW = gridDim.x * kMeasWarps;
    const int gw = blockIdx.x * kMeasWarps + warp;
    MeasWs* ws = a.ws;
    u32 epoch = 0;
    u32 tma_parity = 0;
    if (tid == 0) mbar_init(&s_mbar, 1);
    __syncthreads();

    u64* acc_x = s_acc + (size_t)warp * 2 * Wp;
    u64* acc_z = acc_x + Wp;

    int pos = 0;
    u32 wave = 0;
    while (pos < a.count) {
        // ------------------------------------------------ phase A -------------
        if (blockIdx.x == 0 && tid == 0) { ws->first[(wave + 1) % 3] = ~0ull; }
        const int j = pos + gw;
        int my_det = 0, my_k = 0;
        if (j < a.count) {
            const u32 q = a.qubits[j];
            const u64* xcol = a.m.cols + (size_t)(2 * q) * RW;
            // K2: pivot = smallest stabilizer row with x_q = 1
            u32 best = 0xffffffffu;
            for (int w = lane; w < W; w += 32) {
                u64 v = ldcg(xcol + w);
                if (v) best = min(best, u32(w * 64 + __ffsll((long long)v) - 1));
            }
            best = warp_min(best);
            if (best != 0xffffffffu) {
                if (lane == 0) atomicMin(&ws->first[wave % 3], ((u64)(u32)j << 32) | best);
            } else {
                // K4: deterministic.  scratch := product of stabilizer rows s with destab x_{s,q} = 1
                my_det = 1;
                for (int w = lane; w < Wp; w += 32) { acc_x[w] = 0; acc_z[w] = 0; }
                int e = 0;
                for (int c = 0; c < W; c += 32) {
                    u64 v = (c + lane < W) ? ldcg(xcol + W + c + lane) : 0ull;
                    u32 nz = __ballot_sync(0xffffffffu, v != 0);
                    while (nz) {
                        int l = __ffs(nz) - 1; nz &= nz - 1;
                        u64 word = __shfl_sync(0xffffffffu, v, l);
                        while (word) {
                            int b = __ffsll((long long)word) - 1; word &= word - 1;
                            const int s = (c + l) * 64 + b;            // stabilizer row-bit
                            const u64* rx = a.m.rows + (size_t)(2 * s) * Wp;
                            const u64* rz = rx + Wp;
                            if (lane == 0) e += 2 * int((ldcg(a.m.sgn + (s >> 6)) >> (s & 63)) & 1ull);
                            for (int w = lane; w < W; w += 32) {
                                u64 sx = ldcg(rx + w), sz = ldcg(rz + w);
                                u64 ax = acc_x[w], az = acc_z[w];
                                e += g_word(sx, sz, ax, az);            // rowsum(scratch, s): left factor = row s
                                acc_x[w] = ax ^ sx; acc_z[w] = az ^ sz;
                            }
                            ++my_k;
                        }
                    }
                }
                e = warp_sum(e) & 3;
                if (lane == 0) {
                    if (e & 1) atomicOr(&ws->err, 1u);
                    a.outcomes[j] = uint8_t(e >> 1);
                    a.dets[j] = 1;
                }
            }
        }
        if (!grid_barrier(&ws->bar, epoch, &ws->err)) return;
        const u64 fkey = ldcg(&ws->first[wave % 3]);
        const int wend = min(a.count, pos + GW);
        const int f = (fkey == ~0ull) ? wend : int(fkey >> 32);
        if (my_det && j < f && lane == 0) {
            atomicAdd(&ws->n_det, 1ull); atomicAdd(&ws->k_det, (u64)my_k);
        }
        if (blockIdx.x == 0 && tid == 0) atomicAdd(&ws->waves, 1ull);
        ++wave;
        if (f >= wend) { pos = wend; continue; }

        // ------------------------------------------------ phase B: random at f --
        const u32 q = a.qubits[f];
        const int p = int(fkey & 0xffffffffu);          // pivot stabilizer row-bit
        const int pd = NS + p;                           // its destabilizer
        const u64* xcol = a.m.cols + (size_t)(2 * q) * RW;
        // stage mask, P, D with 1-D TMA
        if (tid == 0) {
            asm volatile("fence.proxy.async;" ::: "memory");
            const u32 bytes = u32(RW * 8 + 4 * Wp * 8);
            mbar_expect_tx(&s_mbar, bytes);
            tma_load_1d(s_mask, xcol, u32(RW * 8), &s_mbar);
            tma_load_1d(s_P, a.m.rows + (size_t)(2 * p) * Wp, u32(2 * Wp * 8), &s_mbar);
            tma_load_1d(s_D, a.m.rows + (size_t)(2 * pd) * Wp, u32(2 * Wp * 8), &s_mbar);
        }
        if (!mbar_wait(&s_mbar, tma_parity)) { if (tid == 0) atomicOr(&ws->err, 0x40000000u); }
        tma_parity ^= 1;
        const int sp = int((ldcg(a.m.sgn + (p >> 6)) >> (p & 63)) & 1ull);
        const int sd = int((ldcg(a.m.sgn + (pd >> 6)) >> (pd & 63)) & 1ull);
        __syncthreads();
        if (tid == 0) { s_mask[p >> 6] &= ~(1ull << (p & 63)); s_mask[pd >> 6] &= ~(1ull << (pd & 63)); }
        if (!grid_barrier(&ws->bar, epoch, &ws->err)) return;     // everyone has staged

        // B1: rowsum(i, p) on R for every i in the mask; unit = one byte of the mask
        for (int u = gw; u < RW * 8; u += GW) {
            u32 byte = u32((s_mask[u >> 3] >> ((u & 7) * 8)) & 0xffull);
            while (byte) {
                int b = __ffs(byte) - 1; byte &= byte - 1;
                const int i = u * 8 + b;
                u64* tx = a.m.rows + (size_t)(2 * i) * Wp;
                u64* tz = tx + Wp;
                int e = 0;
                for (int w = lane; w < W; w += 32) {
                    u64 x = ldcg(tx + w), z = ldcg(tz + w);
                    u64 px = s_P[w], pz = s_P[Wp + w];
                    e += g_word(px, pz, x, z);                     // left factor = pivot row
                    if (px) __stcg(tx + w, x ^ px);
                    if (pz) __stcg(tz + w, z ^ pz);
                }
                e = warp_sum(e) & 3;
                if (lane == 0) {
                    if (e & 1) atomicOr(&ws->err, 1u);
                    if (sp ^ (e >> 1)) atomicXor(a.m.sgn + (i >> 6), 1ull << (i & 63));
                }
            }
        }
        // B2: C form, column_j ^= mask for j in supp(P); unit = (half h, qubit word pw)
        for (int u = gw; u < 2 * W; u += GW) {
            const int h = u / W, pw = u % W;
            u64 bits = s_P[h * Wp + pw];
            while (bits) {
                int b = __ffsll((long long)bits) - 1; bits &= bits - 1;
                u64* col = a.m.cols + (size_t)(2 * (pw * 64 + b) + h) * RW;
                for (int w = lane; w < RW; w += 32) {
                    u64 mv = s_mask[w];
                    if (mv) atomicXor(col + w, mv);
                }
            }
        }
        // B3: C form, single-bit fixes for rows p (-> Z_q) and p+n (-> P); thread per (list, word)
        {
            const int gt = blockIdx.x * kMeasThreads + tid, GT = gridDim.x * kMeasThreads;
            const u64 pbit = 1ull << (p & 63), dbit = 1ull << (pd & 63);
            for (int u = gt; u < 4 * W; u += GT) {
                const int list = u / W, pw = u % W;
                const int h = list & 1;
                u64 bits; int word; u64 bit;
                if (list < 2) {          // row p: old P -> Z_q
                    bits = s_P[h * Wp + pw];
                    if (h == 1 && pw == int(q >> 6)) bits ^= 1ull << (q & 63);
                    word = p >> 6; bit = pbit;
                } else {                 // row p+n: old D -> P
                    bits = s_D[h * Wp + pw] ^ s_P[h * Wp + pw];
                    word = pd >> 6; bit = dbit;
                }
                while (bits) {
                    int b = __ffsll((long long)bits) - 1; bits &= bits - 1;
                    atomicXor(a.m.cols + (size_t)(2 * (pw * 64 + b) + h) * RW + word, bit);
                }
            }
        }
        // B4: R form, row p+n := P ; row p := Z_q   (block 1 if it exists)
        if (blockIdx.x == (gridDim.x > 1 ? 1 : 0)) {
            u64* rp = a.m.rows + (size_t)(2 * p) * Wp;
            u64* rd = a.m.rows + (size_t)(2 * pd) * Wp;
            for (int w = tid; w < 2 * Wp; w += kMeasThreads) {
                __stcg(rd + w, s_P[w]);
                u64 v = 0;
                if (w == Wp + int(q >> 6)) v = 1ull << (q & 63);
                __stcg(rp + w, v);
            }
        }
        // signs, record, counters (block 0)
        if (blockIdx.x == 0 && warp == 0) {
            int k = 0;
            for (int w = lane; w < RW; w += 32) k += __popcll(s_mask[w]);
            k = warp_sum(k);
            if (lane == 0) {
                const int out = counter_bit(a.seed, a.ordinal0 + (uint64_t)f);
                if (sp != out) atomicXor(a.m.sgn + (p >> 6), 1ull << (p & 63));
                if (sd != sp) atomicXor(a.m.sgn + (pd >> 6), 1ull << (pd & 63));
                a.outcomes[f] = uint8_t(out);
                a.dets[f] = 0;
                atomicAdd(&ws->n_rand, 1ull); atomicAdd(&ws->k_rand, (u64)k);
            }
        }
        if (!grid_barrier(&ws->bar, epoch, &ws->err)) return;
        pos = f + 1;
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
