// kernels_rows.cuh -- K5..K9: kernels over row-major (R form) sets of signed Pauli rows:
// commutation vectors / conflict bitmaps (popcount parity, ref: proj/src/pauli.cpp:117-140,
// 215-237), rowsum+i push-through (pauli.cpp:239-254), duplicate detection (same_axis,
// pauli.cpp:142-144), Pauli weight (pauli.cpp:100-106) and the first-fit resolver used by
// group_greedy and t_separate (Algorithm 3).
// R form: rows[(2*r + h) * Wp + w], h = 0 x / 1 z; signs are a bit-vector sgn[r>>6] bit r&63.
#pragma once
#include "common.cuh"

namespace skd {

// ---- predicates -------------------------------------------------------------
// mode 0 (GC): conflict = anticommute = parity of popc((ax&bz)^(bx&az))      (pauli.cpp:117-127)
// mode 1 (QWC): conflict = any word of (ax&bz)^(bx&az) non-zero               (pauli.cpp:129-140)
// mode: bits 0-7 = predicate (0 GC: anticommute, 1 QWC: any qubit-wise clash); bit 8 (kOrderedFit) only concerns the
// resolver below and is ignored here
constexpr int kOrderedFit = 0x100;
__device__ __forceinline__ bool conflict_words(const u64* ax, const u64* az, const u64* bx, const u64* bz, int W, int mode_) {
    const int mode = mode_ & 0xff;
    u64 acc = 0; int par = 0;
    for (int w = 0; w < W; ++w) {
        u64 v = (ax[w] & bz[w]) ^ (bx[w] & az[w]);
        acc |= v; par ^= __popcll(v);
    }
    return mode ? (acc != 0) : (par & 1);
}

// K5 vector form: bit i of out = p anticommutes with row i.  One warp per row.
__global__ void __launch_bounds__(256)
k_commutation_vector(const u64* __restrict__ rows, int Wp, int W, int nrows,
                     const u64* __restrict__ p /* x[Wp] z[Wp] */, u64* __restrict__ out_bits) {
    const int lane = threadIdx.x & 31;
    const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (row >= nrows) return;
    const u64* rx = rows + (size_t)(2 * row) * Wp; const u64* rz = rx + Wp;
    int par = 0;
    for (int w = lane; w < W; w += 32) par ^= __popcll((p[w] & rz[w]) ^ (rx[w] & p[Wp + w]));
    par = warp_sum(par) & 1;
    if (lane == 0 && par) atomicOr(&out_bits[row >> 6], 1ull << (row & 63));
}

// K7: rowsum_plus_i on every live row that anticommutes with the pushed rotations, applied IN ORDER.
// pushes: npush entries of (x[Wp] z[Wp]) ; psign[q] ; plevel[q] = source layer of push q (sorted
// descending).  Row r (layer lvl[r], or lvl == INT_MAX for M_tab rows) takes only pushes with
// plevel < lvl[r]; rows with lvl < 0 are dead.  One warp per row; row words stay in registers.
template <int WPL>   // words per lane: W <= 32*WPL
__global__ void __launch_bounds__(256)
k_push_through(u64* __restrict__ rows, u64* __restrict__ sgn, int Wp, int W, int row0, int nrows,
               const int* __restrict__ lvl, const u64* __restrict__ pushes, const uint8_t* __restrict__ psign,
               const int* __restrict__ plevel, int npush, u32* __restrict__ err, unsigned long long* __restrict__ n_updated) {
    const int lane = threadIdx.x & 31;
    const int r = row0 + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (r >= row0 + nrows) return;
    const int my = lvl ? lvl[r - row0] : 0x7fffffff;
    if (my < 0) return;
    u64* rx = rows + (size_t)(2 * r) * Wp; u64* rz = rx + Wp;
    u64 x[WPL], z[WPL];
#pragma unroll
    for (int k = 0; k < WPL; ++k) { int w = lane + 32 * k; x[k] = (w < W) ? rx[w] : 0; z[k] = (w < W) ? rz[w] : 0; }
    int sign = int((sgn[r >> 6] >> (r & 63)) & 1ull);
    const int sign0 = sign;
    bool dirty = false; unsigned long long upd = 0;
    for (int q = 0; q < npush; ++q) {
        if (plevel && plevel[q] >= my) continue;
        const u64* px = pushes + (size_t)q * 2 * Wp; const u64* pz = px + Wp;
        int par = 0, g = 0;
        u64 qx[WPL], qz[WPL];
#pragma unroll
        for (int k = 0; k < WPL; ++k) {
            int w = lane + 32 * k;
            qx[k] = (w < W) ? px[w] : 0; qz[k] = (w < W) ? pz[w] : 0;
            par ^= __popcll((qx[k] & z[k]) ^ (x[k] & qz[k]));
        }
        par = warp_sum(par) & 1;
        if (!par) continue;
#pragma unroll
        for (int k = 0; k < WPL; ++k) { g += g_word(qx[k], qz[k], x[k], z[k]); x[k] ^= qx[k]; z[k] ^= qz[k]; }
        g = warp_sum(g);
        const int sum = (2 * sign + 2 * int(psign[q]) + g + 1) & 3;     // pauli.cpp:240
        if (sum & 1) { if (lane == 0) atomicOr(err, 1u); }
        sign = sum >> 1;
        dirty = true; ++upd;
    }
    if (dirty) {
#pragma unroll
        for (int k = 0; k < WPL; ++k) { int w = lane + 32 * k; if (w < W) { rx[w] = x[k]; rz[w] = z[k]; } }
        if (lane == 0) {
            if (sign != sign0) atomicXor(&sgn[r >> 6], 1ull << (r & 63));
            if (n_updated) atomicAdd(n_updated, upd);
        }
    }
}

// K9: sum of popcount(x|z) over rows [0, nrows)
__global__ void __launch_bounds__(256)
k_weight_sum(const u64* __restrict__ rows, int Wp, int W, int nrows, const int* __restrict__ lvl, unsigned long long* __restrict__ out) {
    unsigned long long acc = 0;
    const size_t total = (size_t)nrows * W;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        int r = int(i / W), w = int(i % W);
        if (lvl && lvl[r] < 0) continue;
        acc += __popcll(rows[(size_t)(2 * r) * Wp + w] | rows[(size_t)(2 * r + 1) * Wp + w]);
    }
    int lo = warp_sum(int(acc & 0x7fffffff)), hi = warp_sum(int(acc >> 31));
    if ((threadIdx.x & 31) == 0) atomicAdd(out, (unsigned long long)lo + ((unsigned long long)hi << 31));
}

// K8a: 64-bit content hash of (x,z) per row; one warp per row.
__global__ void __launch_bounds__(256)
k_row_hash(const u64* __restrict__ rows, int Wp, int W, int nrows, u64* __restrict__ hash) {
    const int lane = threadIdx.x & 31;
    const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (r >= nrows) return;
    const u64* rx = rows + (size_t)(2 * r) * Wp; const u64* rz = rx + Wp;
    u64 h = 0;
    for (int w = lane; w < W; w += 32) h ^= splitmix64(rx[w] + 0x9e3779b97f4a7c15ULL * (2 * w + 1)) ^ splitmix64(~rz[w] + 0xc2b2ae3d27d4eb4fULL * (2 * w + 2));
#pragma unroll
    for (int o = 16; o; o >>= 1) h ^= __shfl_xor_sync(0xffffffffu, h, o);
    if (lane == 0) hash[r] = h;
}
// K8b: for row j: rank = number of earlier live rows in the same layer with identical (x,z);
// pred = the latest such row.  Odd rank => (pred, j) is a duplicate pair in scan order.
// Thread per row j; all lanes sweep the same i, so hash[i]/lvl[i] loads are broadcasts.
__global__ void __launch_bounds__(256)
k_dup_rank(const u64* __restrict__ rows, int Wp, int W, int nrows, const u64* __restrict__ hash,
           const int* __restrict__ lvl, int* __restrict__ pair_first /* [nrows], -1 if none */) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int jmax = min(nrows, (int)((blockIdx.x + 1) * blockDim.x));
    const bool live = j < nrows && (!lvl || lvl[j] >= 0);
    const u64 hj = live ? hash[j] : 0; const int lj = (live && lvl) ? lvl[j] : 0;
    int rank = 0, pred = -1;
    for (int i = 0; i < jmax; ++i) {
        if (!live || i >= j) continue;
        if (hash[i] != hj) continue;
        if (lvl && lvl[i] != lj) continue;
        const u64* a = rows + (size_t)(2 * i) * Wp; const u64* b = rows + (size_t)(2 * j) * Wp;
        bool eq = true;
        for (int w = 0; w < W && eq; ++w) eq = (a[w] == b[w]) && (a[Wp + w] == b[Wp + w]);
        if (eq) { ++rank; pred = i; }
    }
    if (j < nrows) pair_first[j] = (live && (rank & 1)) ? pred : -1;
}

// K5 matrix form for first-fit: block terms [t0, t0+B) against every earlier term m < t0.
// bitmap[(t - t0) * GW32 + (g >> 5)] bit (g & 31) = term t conflicts with a member of group g.
// Thread per earlier term m (coalesced load of its words + group id), block terms broadcast from smem.
__global__ void __launch_bounds__(256)
k_conflict_bitmap(const u64* __restrict__ rows, int Wp, int W, int t0, int B, int Bt, const u32* __restrict__ group_of,
                  int mode, u32* __restrict__ bitmap, int GW32) {
    extern __shared__ u64 s_blk[];          // [Bt][2*W]: x words then z words of each staged block term
    const int tb = t0 + blockIdx.y * Bt;    // first block term of this tile
    for (int i = threadIdx.x; i < Bt * 2 * W; i += blockDim.x) {
        const int k = i / (2 * W), w = i % (2 * W);
        const int t = tb + k;
        s_blk[i] = (t < t0 + B) ? rows[(size_t)(2 * t + (w >= W)) * Wp + (w % W)] : 0;
    }
    __syncthreads();
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = m < t0;                       // whole warps stay for the warp-level aggregation below
    const int mm = live ? m : 0;
    const u64* mx = rows + (size_t)(2 * mm) * Wp; const u64* mz = mx + Wp;
    const u32 g = live ? group_of[mm] : 0u;
    const u32 widx = g >> 5, gbit = 1u << (g & 31);
    // Do all lanes of this warp point into the same bitmap word?  (Neighbouring earlier terms sit in neighbouring groups
    // when nearly every term opens its own group -- QWC on random strings.)  Then the warp merges its bits with one REDUX.OR
    // and issues one atomic per block term instead of a load + atomic per conflicting pair; otherwise lanes go one by one.
    const u32 w_first = __shfl_sync(0xffffffffu, widx, 0);
    const bool one_word = __all_sync(0xffffffffu, !live || widx == w_first);
    for (int k = 0; k < Bt && tb + k < t0 + B; ++k) {
        const u64* bx = s_blk + (size_t)k * 2 * W; const u64* bz = bx + W;
        const bool c = live && conflict_words(bx, bz, mx, mz, W, mode);
        if (one_word) {
            const u32 bits = __reduce_or_sync(0xffffffffu, c ? gbit : 0u);
            if ((threadIdx.x & 31) == 0 && bits) {
                u32* word = bitmap + (size_t)(tb + k - t0) * GW32 + w_first;
                atomicOr(word, bits);                 // fire-and-forget reduction: no L2 round trip on the warp's path
            }
        } else if (c) {
            u32* word = bitmap + (size_t)(tb + k - t0) * GW32 + widx;
            atomicOr(word, gbit);
        }
    }
}

// ---- K5, group-major form (rows of at most 128 qubits: W <= 2) ------------------------------------------------------
// The terms placed so far are kept grouped (CSR: off[g] .. off[g+1] into gterms, 4 words x0 x1 z0 z1 per term), rebuilt
// per block by a counting sort.  The conflict kernel then runs ONE THREAD PER GROUP: a block term conflicts with the
// group as soon as one member conflicts, the first four members sit in registers, and 32 consecutive groups are exactly
// one bitmap word -> a warp ballot and one plain store per (block term, word): no atomics, and for GC ~10x fewer
// predicate evaluations than the term x term matrix (a random group is rejected after ~2 members).
// gmin = smallest group that received a term: the offsets of all groups in front of it do not change
__global__ void k_csr_count(const u32* __restrict__ group_of, int m0, int m1, u32* __restrict__ cnt, u32* __restrict__ gmin) {
    const int m = m0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (m < m1) { const u32 g = group_of[m]; atomicAdd(cnt + g, 1u); atomicMin(gmin, g); }
}
// exclusive scan of cnt[0, ng) by one CTA (a thread owns a contiguous chunk); off[ng] = total
__global__ void __launch_bounds__(1024)
k_csr_scan(const u32* __restrict__ cnt, const u32* __restrict__ ngroups, u32* __restrict__ off, const u32* __restrict__ gmin) {
    __shared__ u32 s_sum[1024];
    const int ng = int(*ngroups);
    const int g0 = int(min(*gmin, (u32)ng));                   // groups [0, g0) keep their offsets (off[g0] is still valid)
    const u32 base = g0 > 0 ? off[g0] : 0u;
    const int chunk = (ng - g0 + 1023) / 1024;
    const int lo = min(ng, g0 + int(threadIdx.x) * chunk), hi = min(ng, lo + chunk);
    __syncthreads();                                            // everybody has read off[g0] before it is rewritten
    u32 sum = 0;
    for (int i = lo; i < hi; ++i) sum += cnt[i];
    s_sum[threadIdx.x] = sum;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
        const u32 v = (int(threadIdx.x) >= o) ? s_sum[threadIdx.x - o] : 0u;
        __syncthreads();
        s_sum[threadIdx.x] += v;
        __syncthreads();
    }
    u32 run = base + s_sum[threadIdx.x] - sum;
    for (int i = lo; i < hi; ++i) { off[i] = run; run += cnt[i]; }
    if (threadIdx.x == 1023) off[ng] = base + s_sum[1023];
}
__global__ void k_csr_fill(const u64* __restrict__ rows, int Wp, int W, const u32* __restrict__ group_of, int t0,
                           const u32* __restrict__ off, u32* __restrict__ fillc, u64* __restrict__ gterms) {
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= t0) return;
    const u32 g = group_of[m];
    const u32 pos = off[g] + atomicAdd(fillc + g, 1u);
    const u64* x = rows + (size_t)(2 * m) * Wp; const u64* z = x + Wp;
    u64* o = gterms + (size_t)pos * 4;
    o[0] = x[0]; o[1] = W > 1 ? x[1] : 0ull; o[2] = z[0]; o[3] = W > 1 ? z[1] : 0ull;
}
__device__ __forceinline__ bool conflict4(u64 ax0, u64 ax1, u64 az0, u64 az1, u64 bx0, u64 bx1, u64 bz0, u64 bz1, int mode) {
    const u64 v0 = (ax0 & bz0) ^ (bx0 & az0), v1 = (ax1 & bz1) ^ (bx1 & az1);
    return mode == 0 ? (((__popcll(v0) + __popcll(v1)) & 1) != 0) : ((v0 | v1) != 0ull);
}
__global__ void __launch_bounds__(256)
k_conflict_groups(const u64* __restrict__ rows, int Wp, int W, int t0, int B, int Bt, const u32* __restrict__ ngroups,
                  const u32* __restrict__ off, const u64* __restrict__ gterms, int mode_, u32* __restrict__ bitmap, int GW32,
                  unsigned long long* __restrict__ npred, int shard = 0, int nshards = 1) {
    extern __shared__ u64 s_blk[];          // [Bt][4]: x0 x1 z0 z1 of each staged block term
    const int mode = mode_ & 0xff;
    const u32 ng = *ngroups;
    // Sharding by row blocks of the pair matrix: shard s of S owns the bitmap WORDS w with w % S == s, i.e. the groups
    // 32w .. 32w+31; its warps are dense over those words.  S == 1 is the plain kernel.
    if ((size_t)blockIdx.x * blockDim.x * nshards >= ng) return;                 // the grid is sized for the worst case (one group per term)
    const int tb = t0 + blockIdx.y * Bt;
    for (int i = threadIdx.x; i < Bt * 4; i += blockDim.x) {
        const int k = i >> 2, w = i & 3, t = tb + k;
        s_blk[i] = (t < t0 + B && (w & 1) < W) ? rows[(size_t)(2 * t + (w >> 1)) * Wp + (w & 1)] : 0ull;
    }
    __syncthreads();
    const u32 g = 32u * (((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * u32(nshards) + u32(shard)) + (threadIdx.x & 31u);
    const bool live = g < ng;
    const u32 start = live ? off[g] : 0u, cnt = live ? off[g + 1] - start : 0u;
    // first four members in registers; an all-zero (absent) member conflicts with nothing
    u64 m0[4] = {0, 0, 0, 0}, m1[4] = {0, 0, 0, 0}, m2[4] = {0, 0, 0, 0}, m3[4] = {0, 0, 0, 0};
    if (cnt > 0) { const u64* p = gterms + (size_t)start * 4; m0[0] = p[0]; m0[1] = p[1]; m0[2] = p[2]; m0[3] = p[3]; }
    if (cnt > 1) { const u64* p = gterms + (size_t)(start + 1) * 4; m1[0] = p[0]; m1[1] = p[1]; m1[2] = p[2]; m1[3] = p[3]; }
    if (cnt > 2) { const u64* p = gterms + (size_t)(start + 2) * 4; m2[0] = p[0]; m2[1] = p[1]; m2[2] = p[2]; m2[3] = p[3]; }
    if (cnt > 3) { const u64* p = gterms + (size_t)(start + 3) * 4; m3[0] = p[0]; m3[1] = p[1]; m3[2] = p[2]; m3[3] = p[3]; }
    const bool singles = __all_sync(0xffffffffu, cnt <= 1u);   // QWC on random strings: every group is a single term
    const int kend = min(Bt, t0 + B - tb);
    u32 evals = 0;                        // predicates this thread really evaluates (members that exist), for the C4 roofline
    for (int k = 0; k < kend; ++k) {
        const u64 bx0 = s_blk[4 * k], bx1 = s_blk[4 * k + 1], bz0 = s_blk[4 * k + 2], bz1 = s_blk[4 * k + 3];
        bool c = conflict4(m0[0], m0[1], m0[2], m0[3], bx0, bx1, bz0, bz1, mode);
        evals += min(cnt, 4u);
        if (!singles) {
            c |= conflict4(m1[0], m1[1], m1[2], m1[3], bx0, bx1, bz0, bz1, mode);
            c |= conflict4(m2[0], m2[1], m2[2], m2[3], bx0, bx1, bz0, bz1, mode);
            c |= conflict4(m3[0], m3[1], m3[2], m3[3], bx0, bx1, bz0, bz1, mode);
            if (!c && cnt > 4u) {
                for (u32 j = 4; j < cnt && !c; ++j) {
                    const u64* p = gterms + (size_t)(start + j) * 4;
                    c = conflict4(p[0], p[1], p[2], p[3], bx0, bx1, bz0, bz1, mode);
                    ++evals;
                }
            }
        }
        const u32 bits = __ballot_sync(0xffffffffu, c);
        if ((threadIdx.x & 31) == 0) bitmap[(size_t)(tb + k - t0) * GW32 + (g >> 5)] = bits;
    }
    if (npred) { evals = __reduce_add_sync(0xffffffffu, evals); if ((threadIdx.x & 31) == 0 && evals) atomicAdd(npred, (unsigned long long)evals); }
}

// K5 tile form (ref: proj/src/pauli.cpp:117-140): one bit per row pair of the tile [i0, i0+ni) x [j0, j0+nj).  A warp owns one
// output word (row i, 64 consecutive j): lane l evaluates pairs (i, j0 + 64*w + l) and (.., + 32 + l); the row i words are
// broadcast loads.  out[(i - i0) * words + w].
__global__ void __launch_bounds__(256)
k_commute_tile(const u64* __restrict__ rows, int Wp, int W, int mode, int i0, int ni, int j0, int nj, int words, u64* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const long long item = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (item >= (long long)ni * words) return;
    const int i = i0 + int(item / words), w = int(item % words);
    const u64* ax = rows + (size_t)(2 * i) * Wp; const u64* az = ax + Wp;
    u32 bits[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int jj = 64 * w + 32 * h + lane;
        bool c = false;
        if (jj < nj) {
            const u64* bx = rows + (size_t)(2 * (j0 + jj)) * Wp; const u64* bz = bx + Wp;
            int par = 0; u64 any = 0;
            for (int k = 0; k < W; ++k) { const u64 v = (ax[k] & bz[k]) ^ (bx[k] & az[k]); par ^= __popcll(v); any |= v; }
            c = mode == 0 ? (par & 1) : (any != 0);
        }
        bits[h] = __ballot_sync(0xffffffffu, c);
    }
    if (lane == 0) out[(size_t)(i - i0) * words + w] = (u64)bits[0] | ((u64)bits[1] << 32);
}

// EngineConfig.audit: symplectic form of a CHP tableau in the R form.  Row-bit a (stabilizer i = bit i,
// destabilizer i = bit NS + i) against row-bit b > a must anticommute iff b == a + NS.  Same warp-per-word layout as the tile.
__global__ void __launch_bounds__(256)
k_audit_tile(const u64* __restrict__ rows, int Wp, int W, int NS, int n, int a0, int na, unsigned long long* __restrict__ violations) {
    const int lane = threadIdx.x & 31;
    const int words = (2 * NS + 63) / 64;
    const long long item = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (item >= (long long)na * words) return;
    const int a = a0 + int(item / words), w = int(item % words);
    const bool alive = (a < NS) ? (a < n) : (a - NS < n);
    const u64* ax = rows + (size_t)(2 * a) * Wp; const u64* az = ax + Wp;
    int bad = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int b = 64 * w + 32 * h + lane;
        if (!alive || b <= a || b >= 2 * NS || ((b < NS) ? (b >= n) : (b - NS >= n))) continue;
        const u64* bx = rows + (size_t)(2 * b) * Wp; const u64* bz = bx + Wp;
        int par = 0;
        for (int k = 0; k < W; ++k) par ^= __popcll((ax[k] & bz[k]) ^ (bx[k] & az[k]));
        bad += ((par & 1) != (b == a + NS ? 1 : 0)) ? 1 : 0;
    }
    bad = __reduce_add_sync(0xffffffffu, bad);
    if (lane == 0 && bad) atomicAdd(violations, (unsigned long long)bad);
}

// First free group of every block term with respect to the groups that existed BEFORE the block (one CTA per bitmap row,
// all rows in parallel): the sequential resolver below starts its scan there instead of at word 0 -- bits only get added
// by the block-mates, so everything in front of that position stays occupied.
__global__ void __launch_bounds__(256)
k_first_free(const u32* __restrict__ bitmap, int GW32, const u32* __restrict__ ngroups, u32* __restrict__ first_free) {
    __shared__ u32 s_best;
    const u32* bm = bitmap + (size_t)blockIdx.x * GW32;
    const int words = int(*ngroups >> 5) + 1;
    if (threadIdx.x == 0) s_best = 0xffffffffu;
    __syncthreads();
    for (int w0 = 0; w0 < words; w0 += 4 * blockDim.x) {
        u32 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) { const int w = w0 + u * int(blockDim.x) + int(threadIdx.x); v[u] = (w < words) ? __ldcg(bm + w) : 0xffffffffu; }
        u32 best = 0xffffffffu;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const u32 freeb = ~v[u];
            if (freeb && best == 0xffffffffu) best = u32((w0 + u * int(blockDim.x) + int(threadIdx.x)) * 32 + __ffs(int(freeb)) - 1);
        }
        if (best != 0xffffffffu) atomicMin(&s_best, best);
        if (__syncthreads_or(best != 0xffffffffu)) break;
    }
    __syncthreads();
    if (threadIdx.x == 0) first_free[blockIdx.x] = s_best;
}

// First-fit resolver for one block (single CTA, sequential over the block's terms):
// term t takes the first group whose bit is clear; later block-mates that conflict with t get that bit set.
__global__ void __launch_bounds__(1024)
k_first_fit_block(const u64* __restrict__ rows, int Wp, int W, int t0, int B, int mode,
                  u32* __restrict__ bitmap, int GW32, u32* __restrict__ group_of, u32* __restrict__ ngroups_io,
                  const u32* __restrict__ first_free) {
    __shared__ u32 s_first;
    __shared__ u32 s_ng;
    if (threadIdx.x == 0) s_ng = *ngroups_io;
    __syncthreads();
    for (int k = 0; k < B; ++k) {
        const int t = t0 + k;
        if (threadIdx.x == 0) s_first = 0xffffffffu;
        __syncthreads();
        const u32 ng = s_ng;
        const u32* bm = bitmap + (size_t)k * GW32;
        // groups >= ng are free by construction; scan words covering [0, ng]
        const int words = int(ng >> 5) + 1;
        u32 g;
        if (mode & kOrderedFit) {
            // order-preserving variant (exact T-layer separation): the group right after the LAST conflicting one
            if (threadIdx.x == 0) s_first = 0u;
            __syncthreads();
            for (int w = threadIdx.x; w < words; w += blockDim.x) {
                const u32 b = __ldcg(bm + w);
                if (b) atomicMax(&s_first, u32(w * 32 + 32 - __clz(int(b))));
            }
            __syncthreads();
            g = min(s_first, ng);
        } else {
        {
            // 8 independent loads per thread and round (the words of a thread ascend, so its first hit is its minimum): the
            // scan of a long row costs words / (8 * 1024) L2 round trips instead of words / 1024
            u32 best = 0xffffffffu;
            const int wstart = min(words - 1, int(first_free[k] >> 5));      // nothing is free in front of it
            for (int w0 = wstart + int(threadIdx.x); w0 < words && best == 0xffffffffu; w0 += 8 * blockDim.x) {
                u32 v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) { const int w = w0 + u * int(blockDim.x); v[u] = (w < words) ? __ldcg(bm + w) : 0xffffffffu; }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const u32 freeb = ~v[u];
                    if (freeb && best == 0xffffffffu) best = u32((w0 + u * int(blockDim.x)) * 32 + __ffs(int(freeb)) - 1);
                }
            }
            if (best != 0xffffffffu) atomicMin(&s_first, best);
        }
        __syncthreads();
        g = min(s_first, ng);                       // first free existing group, else a new one
        }
        if (threadIdx.x == 0) { group_of[t] = g; if (g == ng) s_ng = ng + 1; }
        // propagate to later block-mates
        const u64* tx = rows + (size_t)(2 * t) * Wp; const u64* tz = tx + Wp;
        for (int k2 = k + 1 + threadIdx.x; k2 < B; k2 += blockDim.x) {
            const u64* ox = rows + (size_t)(2 * (t0 + k2)) * Wp; const u64* oz = ox + Wp;
            // fire-and-forget reduction (no load on this thread's path); the scan above reads with ld.cg after the barrier
            if (conflict_words(ox, oz, tx, tz, W, mode)) atomicOr(bitmap + (size_t)k2 * GW32 + (g >> 5), 1u << (g & 31));
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *ngroups_io = s_ng;
}

// First-fit resolver, thread-per-term form (plain first fit only; the order-preserving variant keeps the kernel above).
// Thread k owns block term t0+k and its running candidate `cand` = first group that is free for it given the groups
// that existed before the block (k_first_free) and the groups taken so far by conflicting block-mates.  Per term ONE
// broadcast (the term that is being placed publishes its group) and one predicate evaluation per later thread; a
// candidate only has to move when a conflicting block-mate takes exactly that group -- then the next free bit of that
// thread's bitmap row is searched by the whole CTA (rare for GC; for QWC on random strings the next candidate is always
// the next new group and no memory is touched).  Row k of the bitmap is only ever modified by thread k (fire-and-forget
// reductions), and only read by others after a barrier.
__global__ void __launch_bounds__(1024)
k_first_fit_threads(const u64* __restrict__ rows, int Wp, int W, int t0, int B, int mode,
                    u32* __restrict__ bitmap, int GW32, u32* __restrict__ group_of, u32* __restrict__ ngroups_io,
                    const u32* __restrict__ first_free) {
    __shared__ u32 s_g, s_ngprev, s_ng, s_who, s_best, s_from;
    const int tid = threadIdx.x;
    const bool mine = tid < B;
    const u64* mx = rows + (size_t)(2 * (t0 + (mine ? tid : 0))) * Wp; const u64* mz = mx + Wp;
    u32* myrow = bitmap + (size_t)(mine ? tid : 0) * GW32;
    u32 cand = mine ? first_free[tid] : 0xffffffffu;
    u32 from = 0;                                              // where a handed-over search continues (bit index, word aligned)
    if (tid == 0) s_ng = *ngroups_io;
    __syncthreads();
    for (int k = 0; k < B; ++k) {
        if (tid == k) {
            const u32 ng = s_ng, g = min(cand, ng);
            group_of[t0 + k] = g; s_g = g; s_ngprev = ng;
            if (g == ng) s_ng = ng + 1;
            s_who = 0xffffffffu;
        }
        __syncthreads();
        const u32 g = s_g, ng = s_ng;
        bool need = false;
        if (mine && tid > k) {
            const u64* tx = rows + (size_t)(2 * (t0 + k)) * Wp; const u64* tz = tx + Wp;
            if (conflict_words(mx, mz, tx, tz, W, mode)) {
                // cand <= group count before this placement, so cand is my effective candidate.  A group below it is occupied
                // for me already; one above it has to be remembered for later searches; the candidate itself has to move.
                if (g > cand) atomicOr(myrow + (g >> 5), 1u << (g & 31));
                else if (g == cand) {
                    u32 c = g + 1;
                    for (int steps = 0; c < ng; ++steps) {             // own row: pre-block bits + my own reductions
                        if (steps == 16) { need = true; from = c; break; }
                        const u32 w = c >> 5;
                        u32 freeb = ~__ldcg(myrow + w);
                        if (c & 31u) freeb &= ~((1u << (c & 31u)) - 1u);
                        if (freeb) { c = w * 32 + u32(__ffs(int(freeb)) - 1); break; }
                        c = (w + 1) * 32;
                    }
                    if (!need) cand = min(c, ng);                      // everything from ng on is a new group: free by construction
                    else atomicMin(&s_who, (u32)tid);
                }
            }
        }
        // rare: a search longer than 16 words is finished by the whole CTA, one row at a time
        while (__syncthreads_or(need)) {
            const u32 who = s_who;
            if ((u32)tid == who) s_from = from;
            if (tid == 0) s_best = 0xffffffffu;
            __syncthreads();
            const u32* bm = bitmap + (size_t)who * GW32;
            const int w_lo = int(s_from >> 5), w_hi = int(ng >> 5);          // bits >= ng are free
            u32 best = 0xffffffffu;
            for (int w = w_lo + tid; w <= w_hi && best == 0xffffffffu; w += blockDim.x) {
                const u32 freeb = ~__ldcg(bm + w);
                if (freeb) best = u32(w * 32 + __ffs(int(freeb)) - 1);
            }
            if (best != 0xffffffffu) atomicMin(&s_best, best);
            __syncthreads();
            if ((u32)tid == who) { cand = min(s_best, ng); need = false; s_who = 0xffffffffu; }
            __syncthreads();
            if (need) atomicMin(&s_who, (u32)tid);
        }
    }
    if (tid == 0) *ngroups_io = s_ng;
}

// ---- first fit by free lists (rows of at most 128 qubits; the default resolver of config C4) --------------------------------
// A term of a GC instance fits very few of the groups that exist when its block starts (two on average at N = 10^6: a group of k
// random members accepts a term with probability 2^-k), so instead of walking bitmap rows the resolver works on
//   * the term's FREE LIST: its first kFreeList free pre-block groups in ascending order (k_free_lists, all rows in parallel), and
//   * a per-term bit mask over the groups created inside the block (at most one per term: 1024 bits, in shared memory).
// The sequential part: the term whose turn it is takes the first live entry of its list, else the first in-block group without a
// conflicting member, else a new group; every later term that conflicts with it strikes that group from its own list / mask --
// inside a warp of 32 consecutive terms by shuffles, across warps once per 32 terms (one block barrier).  Identical groups to the scanning resolvers (same first-fit rule).
constexpr int kFreeList = 12;
// free pre-block groups of every block term, ascending; fcnt = how many there are (kFreeList + 1 stands for "more than the list holds").
// Coalesced sweep in chunks of 256 words: a chunk without a free bit costs one barrier (GC rows are almost all ones), one with
// free bits is compacted in word order (warp scan + one shared-memory hop), and the sweep stops once the list is full.
__global__ void __launch_bounds__(256)
k_free_lists(const u32* __restrict__ bitmap, int GW32, const u32* __restrict__ ngroups, u32* __restrict__ fl, u32* __restrict__ fcnt) {
    __shared__ u32 s_w[8];
    const u32* bm = bitmap + (size_t)blockIdx.x * GW32;
    const u32 ng = *ngroups;
    const int words = int((ng + 31) >> 5);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    u32 found = 0;                                    // entries written so far (CTA-uniform)
    for (int w0 = 0; w0 < words && found <= (u32)kFreeList; w0 += 256) {
        const int w = w0 + int(threadIdx.x);
        u32 freeb = (w < words) ? ~__ldcg(bm + w) : 0u;
        if (w == words - 1 && (ng & 31u)) freeb &= (1u << (ng & 31u)) - 1u;      // groups >= ng do not exist yet
        if (!__syncthreads_or(freeb != 0u)) continue;
        const u32 cnt = __popc(freeb);
        u32 incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) { const u32 v = __shfl_up_sync(0xffffffffu, incl, o); if (lane >= o) incl += v; }
        if (lane == 31) s_w[warp] = incl;
        __syncthreads();
        u32 at = found + incl - cnt, tot = 0;
#pragma unroll
        for (int t = 0; t < 8; ++t) { if (t < warp) at += s_w[t]; tot += s_w[t]; }
        while (freeb && at < (u32)kFreeList) { const int b = __ffs(int(freeb)) - 1; freeb &= freeb - 1; fl[(size_t)blockIdx.x * kFreeList + at] = u32(w * 32 + b); ++at; }
        found += tot;
        __syncthreads();                               // s_w is reused by the next chunk
    }
    if (threadIdx.x == 0) fcnt[blockIdx.x] = min(found, (u32)kFreeList + 1u);
}

__device__ __forceinline__ void load_term4(const u64* __restrict__ rows, int Wp, int W, int m, u64* o) {
    const u64* x = rows + (size_t)(2 * m) * Wp; const u64* z = x + Wp;
    o[0] = x[0]; o[1] = W > 1 ? x[1] : 0ull; o[2] = z[0]; o[3] = W > 1 ? z[1] : 0ull;
}
// In-block conflict matrix for the free-list resolver: cb[i][w] bit k = term t0+i conflicts with term t0+32w+k (i, 32w+k < B).
// A thread per (term, word): the 1024 x 1024 pair checks of a block on the whole machine instead of on the resolver's one SM.
__global__ void __launch_bounds__(256)
k_conflict_block(const u64* __restrict__ rows, int Wp, int W, int t0, int B, int mode, u32* __restrict__ cb) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = idx >> 5, w = idx & 31;
    if (i >= B) return;
    u32 bits = 0;
    if (32 * w < i) {                                   // only earlier terms matter to term i
        u64 a[4]; load_term4(rows, Wp, W, t0 + i, a);
        const int kend = min(32, i - 32 * w);
        for (int k = 0; k < kend; ++k) {
            u64 b[4]; load_term4(rows, Wp, W, t0 + 32 * w + k, b);
            if (conflict4(a[0], a[1], a[2], a[3], b[0], b[1], b[2], b[3], mode)) bits |= 1u << k;
        }
    }
    cb[(size_t)i * 32 + w] = bits;
}
// Pipelined grouping: the group-major conflict kernel of block n runs on a side stream, beside the resolver of block n-1, over
// the groups as they were after block n-2.  This kernel adds what it could not know: the conflicts of block n's terms with the
// terms block n-1 has placed meanwhile (into old groups or new ones).  A thread per (term, 32 previous terms); GC bitmap rows
// are almost all ones already, so the bit is read first and few atomics are issued.
__global__ void __launch_bounds__(256)
k_conflict_prev(const u64* __restrict__ rows, int Wp, int W, int t0, int B, int tp0, int Bp, int mode, const u32* __restrict__ group_of,
                u32* __restrict__ bitmap, int GW32, unsigned long long* __restrict__ npred) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = idx >> 5, w = idx & 31;
    u32 evals = 0;
    if (i < B && 32 * w < Bp) {
        u64 a[4]; load_term4(rows, Wp, W, t0 + i, a);
        u32* row = bitmap + (size_t)i * GW32;
        const int kend = min(32, Bp - 32 * w);
        for (int k = 0; k < kend; ++k) {
            u64 b[4]; load_term4(rows, Wp, W, tp0 + 32 * w + k, b);
            if (conflict4(a[0], a[1], a[2], a[3], b[0], b[1], b[2], b[3], mode)) {
                const u32 g = group_of[tp0 + 32 * w + k], bit = 1u << (g & 31u);
                if (!(__ldcg(row + (g >> 5)) & bit)) atomicOr(row + (g >> 5), bit);
            }
        }
        evals = (u32)kend;
    }
    if (npred) { evals = __reduce_add_sync(0xffffffffu, evals); if ((threadIdx.x & 31) == 0 && evals) atomicAdd(npred, (unsigned long long)evals); }
}
__device__ __forceinline__ u32 lst_last(const u32* fl, int tid, int have) { return fl[(size_t)tid * kFreeList + have - 1]; }
// dynamic shared memory: in-block masks [32][1024] u32
__global__ void __launch_bounds__(1024)
k_first_fit_lists(int t0, int B, u32* __restrict__ bitmap, int GW32, u32* __restrict__ group_of, u32* __restrict__ ngroups_io,
                  const u32* __restrict__ fl, const u32* __restrict__ fcnt, const u32* __restrict__ cb) {
    extern __shared__ u64 s_dyn[];
    u32* s_nb = reinterpret_cast<u32*>(s_dyn);                      // [32][1024]: in-block groups struck for thread tid, bit (g - ng0)
    __shared__ u32 s_gl[1024], s_ng;                                // groups of the block's terms placed so far ; groups that exist now
    const int tid = threadIdx.x;
    const bool mine = tid < B;
    const u32 ng0 = *ngroups_io;                                    // groups that exist when the block starts
#pragma unroll
    for (int w = 0; w < 32; ++w) s_nb[w * 1024 + tid] = 0u;
    u32 lst[16];                                                    // my free pre-block groups, ascending (constant; `live` says which are still free)
    const u32 total = mine ? fcnt[tid] : 0u;
    const int have = int(min(total, (u32)kFreeList));
    unsigned long long hmask = 0;                                   // bit (g & 63) of every listed group: most strikes miss the list and stop here
#pragma unroll
    for (int i = 0; i < 16; ++i) { lst[i] = (mine && i < have) ? fl[(size_t)tid * kFreeList + i] : 0xffffffffu; if (lst[i] != 0xffffffffu) hmask |= 1ull << (lst[i] & 63u); }
    u32 live = (1u << have) - 1u;
    const u32 last_listed = have ? lst_last(fl, tid, have) : 0u;
    u32 nbfull = 0, nb0 = 0, nb1 = 0;                               // in-block groups struck for me: words 0 and 1 here, the rest in s_nb
    const bool ovf = total > (u32)kFreeList;                        // more free pre-block groups than the list holds: strikes also go to the bitmap row
    u32* myrow = bitmap + (size_t)(mine ? tid : 0) * GW32;
    const u32* mycb = cb + (size_t)(mine ? tid : 0) * 32;           // my conflicts with the earlier terms of the block, a word per sub-batch
    if (tid == 0) s_ng = ng0;
    __syncthreads();
    // a conflicting earlier term placed in group g: g leaves my list / my in-block mask
    auto strike = [&](u32 g) {
        if (g >= ng0) {
            const u32 w = (g - ng0) >> 5, bit = 1u << ((g - ng0) & 31u);
            u32 v;
            if (w == 0) v = (nb0 |= bit);                        // the first 64 in-block groups live in registers: no shared-memory
            else if (w == 1) v = (nb1 |= bit);                   // round trip on the chain from one term's decision to the next
            else { v = s_nb[w * 1024 + tid] | bit; s_nb[w * 1024 + tid] = v; }
            if (v == 0xffffffffu && w == nbfull) ++nbfull;       // leading words that are full (a lower bound is enough: the search starts there)
        } else {
            if ((hmask >> (g & 63u)) & 1ull) {
                u32 hit = 0;                                        // independent compares: nothing here lengthens the chain from one term's decision to the next
#pragma unroll
                for (int i = 0; i < kFreeList; ++i) hit |= (lst[i] == g) ? (1u << i) : 0u;
                live &= ~hit;
            }
            if (ovf) atomicOr(myrow + (g >> 5), 1u << (g & 31));
        }
    };
    // The terms are placed in order, 32 at a time: the warp that owns sub-batch j places its terms one after the other with warp
    // shuffles only, publishes the 32 groups, and after ONE block barrier every later warp strikes them from its own terms' lists
    // (conflicts come precomputed from k_conflict_block: the loop visits the set bits of one word).  32 barriers per block of 1024
    // terms instead of 1024.  Same order of decisions, same information at each decision: identical groups.
    const int lane = tid & 31, warp = tid >> 5;
    const int nsub = (B + 31) >> 5;
    u32 cw_next = (mine && warp >= 0) ? __ldg(mycb) : 0u;
    for (int j = 0; j < nsub; ++j) {
        const int base = 32 * j, cntk = min(32, B - base);
        u32 cw = cw_next;                                           // my conflicts with sub-batch j (for my own sub-batch: with the lanes before me),
        cw_next = (mine && warp >= j + 1 && j + 1 < nsub) ? __ldg(mycb + j + 1) : 0u;      // fetched one sub-batch ahead: the load is never on the chain
        if (warp == j) {
            u32 ng = s_ng, myg = 0;
            const u32 cmask = cw;
            // Every lane keeps its CANDIDATE -- the group it would take if its turn were now: first live list entry, else (list
            // truncated) the rest of its bitmap row, else the first in-block group without a conflicting member, else the next new
            // group, written as the number that group would get.  A turn is then one shuffle; only the lanes that conflict with
            // the placed term AND had exactly its group as candidate look for the next one.  (A lane whose candidate was "new" and
            // does not conflict with the lane that just opened that group keeps the same number: it now means "join it".)
            auto candidate = [&](u32 ngc) -> u32 {
                u32 g = 0xffffffffu;
                if (live) {
                    const int idx = __ffs(int(live)) - 1;          // four select levels instead of a chain of twelve
                    const u32 a0 = (idx & 1) ? lst[1] : lst[0], a1 = (idx & 1) ? lst[3] : lst[2], a2 = (idx & 1) ? lst[5] : lst[4], a3 = (idx & 1) ? lst[7] : lst[6];
                    const u32 a4 = (idx & 1) ? lst[9] : lst[8], a5 = (idx & 1) ? lst[11] : lst[10], a6 = (idx & 1) ? lst[13] : lst[12], a7 = (idx & 1) ? lst[15] : lst[14];
                    const u32 b0 = (idx & 2) ? a1 : a0, b1 = (idx & 2) ? a3 : a2, b2 = (idx & 2) ? a5 : a4, b3 = (idx & 2) ? a7 : a6;
                    const u32 c0 = (idx & 4) ? b1 : b0, c1 = (idx & 4) ? b3 : b2;
                    g = (idx & 8) ? c1 : c0;
                }
                if (g == 0xffffffffu && ovf) {
                    for (u32 c = last_listed + 1; c < ng0;) {                      // behind the last listed group
                        const u32 w = c >> 5;
                        u32 freeb = ~__ldcg(myrow + w);
                        if (c & 31u) freeb &= ~((1u << (c & 31u)) - 1u);
                        if (freeb) { const u32 f = w * 32 + u32(__ffs(int(freeb)) - 1); if (f < ng0) g = f; break; }
                        c = (w + 1) * 32;
                    }
                }
                if (g == 0xffffffffu) {
                    const u32 nnew = ngc - ng0;
                    for (u32 w = nbfull; w * 32 < nnew; ++w) {
                        u32 freeb = ~(w == 0 ? nb0 : (w == 1 ? nb1 : s_nb[w * 1024 + tid]));
                        if ((w + 1) * 32 > nnew) freeb &= (1u << (nnew & 31u)) - 1u;
                        if (freeb) { g = ng0 + w * 32 + u32(__ffs(int(freeb)) - 1); break; }
                    }
                }
                return g == 0xffffffffu ? ngc : g;
            };
            u32 cand = mine ? candidate(ng) : 0xffffffffu;
            for (int k = 0; k < cntk; ++k) {
                const u32 g = __shfl_sync(0xffffffffu, cand, k);
                if (lane == k) { group_of[t0 + base + k] = g; myg = g; }
                if (g == ng) ++ng;
                if ((cmask >> k) & 1u) {
                    strike(g);
                    if (cand == g) cand = candidate(ng);
                }
            }
            s_gl[tid] = myg;
            if (lane == 0) s_ng = ng;
        }
        __syncthreads();
        if (warp > j) {
            while (cw) { const int k = __ffs(int(cw)) - 1; cw &= cw - 1; strike(s_gl[base + k]); }
        }
    }
    __syncthreads();
    if (tid == 0) *ngroups_io = s_ng;
}

// verify_grouping: number of intra-group pairs violating the predicate.
// Thread per row j sweeps all i < j (broadcast loads of group ids).
__global__ void __launch_bounds__(256)
k_verify_grouping(const u64* __restrict__ rows, int Wp, int W, int nrows, const u32* __restrict__ group_of,
                  int mode, unsigned long long* __restrict__ nviol) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int jmax = min(nrows, (int)((blockIdx.x + 1) * blockDim.x));
    const u32 gj = j < nrows ? group_of[j] : 0xffffffffu;
    unsigned long long bad = 0;
    for (int i = 0; i < jmax; ++i) {
        if (j >= nrows || i >= j || group_of[i] != gj) continue;
        const u64* a = rows + (size_t)(2 * i) * Wp; const u64* b = rows + (size_t)(2 * j) * Wp;
        bad += conflict_words(a, a + Wp, b, b + Wp, W, mode);
    }
    if (bad) atomicAdd(nviol, bad);
}

// copy rows idx[k] (x and z halves) into a dense push list  out[k][2*Wp]
__global__ void k_gather_rows(const u64* __restrict__ rows, int Wp, const int* __restrict__ idx, int count, u64* __restrict__ out) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (size_t)count * 2 * Wp) return;
    const int k = int(i / (2 * Wp)), w = int(i % (2 * Wp));
    out[i] = rows[(size_t)(2 * idx[k]) * Wp + w];
}
// min over j of (pair_first[j] << 32 | j) for pair_first[j] >= 0
__global__ void k_min_pair(const int* __restrict__ pair_first, int nrows, unsigned long long* __restrict__ out) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < nrows && pair_first[j] >= 0) atomicMin(out, ((unsigned long long)(u32)pair_first[j] << 32) | (u32)j);
}

}  // namespace skd
