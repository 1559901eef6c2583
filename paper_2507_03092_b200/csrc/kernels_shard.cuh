// kernels_shard.cuh -- device side of a ROW SHARD of a CHP tableau.
//
// A shard owns the slots [lo, lo + nloc): stabilizer i and destabilizer i for every i in the range
// (co-located so that the deterministic branch "destabilizer i selects stabilizer i" stays local).
// Local row-bit space: stabilizer i -> bit i - lo, destabilizer i -> bit NS + i - lo, NS = 64*ceil(nloc/64);
// the qubit (column) space is the global one.  Both forms of common.cuh are kept, with RW = 2*NS/64 row words:
// gate layers run the ordinary k_layer on the C form (no communication: rows are independent);
// a measurement block keeps C and R valid together (the random branch updates both), so the pivot search and
// the partner search always read contiguous C columns and the Pauli products always read contiguous R rows.
//
// What crosses shards is produced / consumed here as plain device buffers; the exchange itself (allreduce-min
// of the pivot candidates, broadcast of the pivot row, allgather of the partial products) is done by the host
// driver over NCCL (paper_2507_03092_b200/sharded.py).
#pragma once
#include "common.cuh"

namespace skd {

constexpr u32 kShardNone = 0x7f7f7f7fu;     // "no stabilizer of this shard has an x here" (memset-able, > any row index)

// SPEC:125-133 restricted to the shard's slots
__global__ void k_shard_identity(u64* __restrict__ cols, u64* __restrict__ rows, int lo, int nloc, int RW, int Wp, int NS) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nloc) return;
    const int q = lo + i;
    const u64 qb = 1ull << (q & 63);
    cols[(size_t)(2 * q + 1) * RW + (i >> 6)] = 1ull << (i & 63);
    cols[(size_t)(2 * q) * RW + ((NS + i) >> 6)] = 1ull << ((NS + i) & 63);
    rows[(size_t)(2 * i + 1) * Wp + (q >> 6)] = qb;
    rows[(size_t)(2 * (NS + i)) * Wp + (q >> 6)] = qb;
}

// Pivot search (smallest stabilizer index with x_{i,q} = 1) over the shard's stabilizers: one warp per
// measurement, contiguous column words, cand[j] = GLOBAL index or kShardNone.  The shards' candidates are then
// min-reduced by the driver.
__global__ void __launch_bounds__(256)
k_shard_pivot(const u64* __restrict__ cols, const u32* __restrict__ qubits, int m, int RW, int NSW, int lo, int* __restrict__ cand) {
    const int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (j >= m) return;
    const u64* col = cols + (size_t)(2 * qubits[j]) * RW;
    u32 best = kShardNone;
    for (int w0 = 0; w0 < NSW; w0 += 32) {
        const int w = w0 + lane;
        const u64 v = w < NSW ? __ldcg(col + w) : 0ull;
        if (v) best = u32(lo + 64 * w + __ffsll((long long)v) - 1);
        if (__any_sync(0xffffffffu, v != 0ull)) break;       // words ascend: the first non-empty group holds the minimum
    }
    best = warp_min(best);
    if (lane == 0) cand[j] = int(best);
}

// Rows of this shard that the random branch multiplies by the pivot row: the x column of q over all local row bits,
// without the pivot itself and its destabilizer partner (overwritten afterwards; SURVEY section 7 hazard).
__global__ void k_shard_mask(const u64* __restrict__ cols, u32 q, int RW, int NS, int pb, u64* __restrict__ mask) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= RW) return;
    u64 v = __ldcg(cols + (size_t)(2 * q) * RW + w);
    if (pb >= 0) {
        if ((pb >> 6) == w) v &= ~(1ull << (pb & 63));
        const int d = NS + pb;
        if ((d >> 6) == w) v &= ~(1ull << (d & 63));
    }
    mask[w] = v;
}

// pivot row -> exchange buffer  prow = [x: Wp][z: Wp][sign][pad]
__global__ void k_shard_get_row(DMat m, int rb, u64* __restrict__ prow) {
    const int Wp = int(m.Wp);
    for (int w = threadIdx.x; w < 2 * Wp; w += blockDim.x) prow[w] = __ldcg(m.rows + (size_t)(2 * rb) * Wp + w);
    if (threadIdx.x == 0) { prow[2 * Wp] = (__ldcg(m.sgn + (rb >> 6)) >> (rb & 63)) & 1ull; prow[2 * Wp + 1] = 0; }
}

// rowsum(h, pivot) for every masked local row h, R form: one warp per row.
__global__ void __launch_bounds__(256)
k_shard_rowsum(DMat m, const u64* __restrict__ mask, const u64* __restrict__ prow, u32* __restrict__ err, u64* __restrict__ k_rand) {
    const int h = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (h >= 64 * int(m.RW)) return;
    if (!((mask[h >> 6] >> (h & 63)) & 1ull)) return;
    const int Wp = int(m.Wp), W = int(m.W);
    u64* hx = m.rows + (size_t)(2 * h) * Wp; u64* hz = hx + Wp;
    const u64* px = prow; const u64* pz = prow + Wp;
    int e = 0;
    for (int w = lane; w < W; w += 32) {
        const u64 ax = px[w], az = pz[w], bx = hx[w], bz = hz[w];
        e += g_word(ax, az, bx, bz);
        hx[w] = bx ^ ax; hz[w] = bz ^ az;
    }
    e = warp_sum(e);
    if (lane == 0) {
        const int rh = int((__ldcg(m.sgn + (h >> 6)) >> (h & 63)) & 1ull), rp = int(prow[2 * Wp] & 1ull);
        const int sum = (2 * rh + 2 * rp + e) & 3;
        if (sum & 1) atomicOr(err, 1u);
        else if ((sum >> 1) != rh) atomicXor(m.sgn + (h >> 6), 1ull << (h & 63));
        atomicAdd(k_rand, 1ull);
    }
}
// the same update on the C form: column j ^= mask for every j in the pivot row's support (one warp per qubit)
__global__ void __launch_bounds__(256)
k_shard_colxor(DMat m, const u64* __restrict__ mask, const u64* __restrict__ prow) {
    const int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (j >= int(m.n)) return;
    const int Wp = int(m.Wp), RW = int(m.RW);
    const bool bx = (prow[j >> 6] >> (j & 63)) & 1ull, bz = (prow[Wp + (j >> 6)] >> (j & 63)) & 1ull;
    if (!bx && !bz) return;
    u64* cx = m.cols + (size_t)(2 * j) * RW; u64* cz = cx + RW;
    for (int w = lane; w < RW; w += 32) {
        const u64 mk = mask[w];
        if (!mk) continue;
        if (bx) cx[w] ^= mk;
        if (bz) cz[w] ^= mk;
    }
}
// Owner of the pivot, after the rowsums: destabilizer p := old pivot row, stabilizer p := (-1)^outcome Z_q,
// in both forms.  Single CTA; a thread owns whole 64-qubit words, so no two threads touch one column.
__global__ void __launch_bounds__(256)
k_shard_fix(DMat m, int NS, int pb, u32 q, const u64* __restrict__ prow, int outcome) {
    const int Wp = int(m.Wp), W = int(m.W), RW = int(m.RW), db = NS + pb;
    const u64 pbit = 1ull << (pb & 63), dbit = 1ull << (db & 63);
    // bit flips in the C form are fire-and-forget reductions (no load on the thread's path); a column is only touched by
    // the thread that owns its 64-qubit word, and one thread's atomics to one address keep program order
    for (int w = threadIdx.x; w < W; w += blockDim.x) {
        u64* dx = m.rows + (size_t)(2 * db) * Wp + w; u64* dz = dx + Wp;
        const u64 nx = prow[w], nz = prow[Wp + w];
        u64 tx = *dx ^ nx, tz = *dz ^ nz;                       // C form, bit db: toggle where the old row differs from the new one
        while (tx) { const int b = __ffsll((long long)tx) - 1; tx &= tx - 1; atomicXor(m.cols + (size_t)(2 * (64 * w + b)) * RW + (db >> 6), dbit); }
        while (tz) { const int b = __ffsll((long long)tz) - 1; tz &= tz - 1; atomicXor(m.cols + (size_t)(2 * (64 * w + b) + 1) * RW + (db >> 6), dbit); }
        u64 cx = nx, cz = nz;                                   // C form, bit pb: the row still equals the pivot row -> clear it
        while (cx) { const int b = __ffsll((long long)cx) - 1; cx &= cx - 1; atomicXor(m.cols + (size_t)(2 * (64 * w + b)) * RW + (pb >> 6), pbit); }
        while (cz) { const int b = __ffsll((long long)cz) - 1; cz &= cz - 1; atomicXor(m.cols + (size_t)(2 * (64 * w + b) + 1) * RW + (pb >> 6), pbit); }
        *dx = nx; *dz = nz;
        m.rows[(size_t)(2 * pb) * Wp + w] = 0;
        u64 zrow = 0;
        if (w == int(q >> 6)) {                                 // stabilizer p := Z_q (after this thread's own clearing of that column)
            zrow = 1ull << (q & 63);
            atomicOr(m.cols + (size_t)(2 * q + 1) * RW + (pb >> 6), pbit);
        }
        m.rows[(size_t)(2 * pb + 1) * Wp + w] = zrow;
    }
    if (threadIdx.x == 0) {
        u64 s = m.sgn[db >> 6]; s = (s & ~dbit) | ((prow[2 * Wp] & 1ull) ? dbit : 0ull); m.sgn[db >> 6] = s;
        s = m.sgn[pb >> 6]; s = (s & ~pbit) | (outcome ? pbit : 0ull); m.sgn[pb >> 6] = s;
    }
}

// Deterministic branch, this shard's share: the product of the stabilizers i whose destabilizer has
// x_{n+i,q} = 1, as a signed Pauli  part[j] = [x: Wp][z: Wp][i-exponent mod 4][pad].  One warp per measurement; the
// partner search reads the contiguous destabilizer half of the C column.  Stabilizers commute, so the product does
// not depend on the order of the factors (Pauli multiplication is associative).
__global__ void __launch_bounds__(256)
k_shard_det_partial(DMat m, const u32* __restrict__ qubits, int cnt, int NS, u64* __restrict__ part, int PW, u64* __restrict__ k_det) {
    const int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (j >= cnt) return;
    const int Wp = int(m.Wp), W = int(m.W), RW = int(m.RW);
    const u32* col32 = reinterpret_cast<const u32*>(m.cols + (size_t)(2 * qubits[j]) * RW + NS / 64);
    u64* ax = part + (size_t)j * PW; u64* az = ax + Wp;
    for (int w = lane; w < 2 * Wp + 2; w += 32) ax[w] = 0;
    __syncwarp();
    int e = 0, k = 0;
    const int G32 = NS / 32;
    for (int g0 = 0; g0 < G32; g0 += 32) {
        const u32 mw = (g0 + lane < G32) ? __ldcg(col32 + g0 + lane) : 0u;
        u32 any = __ballot_sync(0xffffffffu, mw != 0u);
        while (any) {
            const int src = __ffs(int(any)) - 1; any &= any - 1;
            u32 bits = __shfl_sync(0xffffffffu, mw, src);
            while (bits) {
                const int b = __ffs(int(bits)) - 1; bits &= bits - 1;
                const int i = (g0 + src) * 32 + b;              // local slot = stabilizer row bit
                const u64* rx = m.rows + (size_t)(2 * i) * Wp; const u64* rz = rx + Wp;
                for (int w = lane; w < W; w += 32) {
                    const u64 sx = __ldcg(rx + w), sz = __ldcg(rz + w), cx = ax[w], cz = az[w];
                    e += g_word(sx, sz, cx, cz);
                    ax[w] = cx ^ sx; az[w] = cz ^ sz;
                }
                if (lane == 0) e += 2 * int((__ldcg(m.sgn + (i >> 6)) >> (i & 63)) & 1ull);
                ++k;
            }
        }
    }
    e = warp_sum(e);
    if (lane == 0) { ax[2 * Wp] = u64(e & 3); if (k) atomicAdd(k_det, (u64)k); }
}
// The shards' partial products multiplied in shard order -> outcome = sign of the product.
// gathered = [nshards][cnt][PW].  One warp per measurement.
__global__ void __launch_bounds__(256)
k_shard_det_combine(const u64* __restrict__ gathered, int nshards, int cnt, int W, int Wp, int PW, uint8_t* __restrict__ outcomes, u32* __restrict__ err) {
    const int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (j >= cnt) return;
    int e = 0;
    for (int w = lane; w < W; w += 32) {
        u64 cx = 0, cz = 0;
        for (int g = 0; g < nshards; ++g) {
            const u64* p = gathered + ((size_t)g * cnt + j) * PW;
            const u64 sx = p[w], sz = p[Wp + w];
            e += g_word(sx, sz, cx, cz);
            cx ^= sx; cz ^= sz;
        }
    }
    e = warp_sum(e);
    if (lane == 0) {
        for (int g = 0; g < nshards; ++g) e += int(gathered[((size_t)g * cnt + j) * PW + 2 * Wp] & 3ull);
        if (e & 1) atomicOr(err, 1u);
        outcomes[j] = uint8_t((e & 3) >> 1);
    }
}

}  // namespace skd
