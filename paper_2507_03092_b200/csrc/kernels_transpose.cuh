// kernels_transpose.cuh -- bit-matrix transposition between the qubit-major (C)
// and row-major (R) forms.   dst[r][c] = src[c][r].
//
// One CTA moves a 256 x 256-bit tile through shared memory so that both the
// global loads and the global stores are 32-byte contiguous per matrix row;
// each warp transposes 32x32-bit blocks in registers with a 5-stage shuffle butterfly.
// Roofline: HBM/L2 streaming, reads + writes the matrix once (2 * bits/8 bytes).
#pragma once
#include "common.cuh"

namespace skd {

__device__ __forceinline__ void bfly(u32& v, int j, u32 m, int lane) {
    const u32 p = __shfl_xor_sync(0xffffffffu, v, j);
    v = (lane & j) ? (((p >> j) & m) | (v & ~m)) : ((v & m) | ((p & m) << j));
}
// 32x32-bit transpose across a warp (lane = row).  The two coarse stages exchange whole bytes: one byte permute each instead
// of shift/mask/merge (the kernel is instruction bound: ncu, 58 % SM throughput at 86 % active warps).
__device__ __forceinline__ u32 transpose32(u32 v, int lane) {
    u32 p = __shfl_xor_sync(0xffffffffu, v, 16);
    v = __byte_perm(v, p, (lane & 16) ? 0x3276u : 0x5410u);      // halves:  low lanes keep v.lo | p.lo << 16, high lanes p.hi >> 16 | v.hi
    p = __shfl_xor_sync(0xffffffffu, v, 8);
    v = __byte_perm(v, p, (lane & 8) ? 0x3715u : 0x6240u);       // bytes of each half
    bfly(v, 4, 0x0f0f0f0fu, lane); bfly(v, 2, 0x33333333u, lane); bfly(v, 1, 0x55555555u, lane);
    return v;
}

// All sizes in 32-bit words.  Loads outside [src_rows) x [src_words) read 0;
// stores outside [dst_rows) x [dst_words) are dropped.  blockIdx.z selects one of gridDim.z
// independent matrices (src + z*src_zoff -> dst + z*dst_zoff: the x and z halves of a store).
// If `flag` is given the kernel is a no-op unless *flag != 0 (device-side "C form is stale").
// VEC: every row start and width is a multiple of four 32-bit words (true for tableaux): 16-byte loads and stores, two per
// thread instead of eight 4-byte ones (the kernel is instruction bound, see transpose32).
template <bool VEC>
__device__ __forceinline__ void transpose_bits_body(const u32* __restrict__ src, size_t src_stride, int src_rows, int src_words,
                                                    u32* __restrict__ dst, size_t dst_stride, int dst_rows, int dst_words,
                                                    u32 (*tin)[9], u32 (*tout)[9]) {
    const int c0 = blockIdx.x * 256;          // first src row of the tile  (= dst bit offset)
    const int w0 = blockIdx.y * 8;            // first src word of the tile (= dst row offset / 32)
    const int t = threadIdx.x;
    if (VEC) {
        // two threads read the 32 contiguous bytes a src row has in the tile
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int rr = k * 128 + (t >> 1), ww = (t & 1) * 4;
            const int gr = c0 + rr, gw = w0 + ww;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (gr < src_rows && gw < src_words) v = __ldcg(reinterpret_cast<const uint4*>(src + (size_t)gr * src_stride + gw));
            tin[rr][ww] = v.x; tin[rr][ww + 1] = v.y; tin[rr][ww + 2] = v.z; tin[rr][ww + 3] = v.w;
        }
    } else {
        // load: 8 consecutive threads read 32 contiguous bytes of one src row
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            int rr = k * 32 + (t >> 3), ww = t & 7;
            int gr = c0 + rr, gw = w0 + ww;
            u32 v = 0;
            if (gr < src_rows && gw < src_words) v = __ldcg(src + (size_t)gr * src_stride + gw);
            tin[rr][ww] = v;
        }
    }
    __syncthreads();
    const int warp = t >> 5, lane = t & 31;
    // 8 x 8 blocks of 32x32 bits; warp handles block-row `warp` (src rows 32*warp ..)
#pragma unroll
    for (int bj = 0; bj < 8; ++bj) {
        // src row (c0 + 32*warp + lane), bits 32*(w0+bj) .. : 32x32 bit transpose across the warp
        const u32 mine = transpose32(tin[warp * 32 + lane][bj], lane);
        // lane b holds dst row (32*(w0+bj) + b), word (c0/32 + warp)
        tout[bj * 32 + lane][warp] = mine;
    }
    __syncthreads();
    if (VEC) {
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int rr = k * 128 + (t >> 1), ww = (t & 1) * 4;
            const int gr = w0 * 32 + rr, gw = (c0 >> 5) + ww;
            if (gr < dst_rows && gw < dst_words)
                __stcg(reinterpret_cast<uint4*>(dst + (size_t)gr * dst_stride + gw), make_uint4(tout[rr][ww], tout[rr][ww + 1], tout[rr][ww + 2], tout[rr][ww + 3]));
        }
    } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            int rr = k * 32 + (t >> 3), ww = t & 7;
            int gr = w0 * 32 + rr, gw = (c0 >> 5) + ww;
            if (gr < dst_rows && gw < dst_words) __stcg(dst + (size_t)gr * dst_stride + gw, tout[rr][ww]);
        }
    }
}
__global__ void __launch_bounds__(256)
k_transpose_bits(const u32* __restrict__ src, size_t src_stride, int src_rows, int src_words,
                 u32* __restrict__ dst, size_t dst_stride, int dst_rows, int dst_words,
                 size_t src_zoff, size_t dst_zoff, const u32* __restrict__ flag) {
    __shared__ u32 tin[256][9];    // [src row in tile][word], +1 pad: conflict-free column reads
    __shared__ u32 tout[256][9];   // [dst row in tile][word]
    pdl_trigger();
    pdl_wait();
    if (flag && __ldcg(flag) == 0u) return;
    src += (size_t)blockIdx.z * src_zoff; dst += (size_t)blockIdx.z * dst_zoff;
    const bool vec = ((src_stride | dst_stride | src_zoff | dst_zoff | (size_t)src_words | (size_t)dst_words) & 3) == 0 &&
                     ((reinterpret_cast<size_t>(src) | reinterpret_cast<size_t>(dst)) & 15) == 0;
    if (vec) transpose_bits_body<true>(src, src_stride, src_rows, src_words, dst, dst_stride, dst_rows, dst_words, tin, tout);
    else transpose_bits_body<false>(src, src_stride, src_rows, src_words, dst, dst_stride, dst_rows, dst_words, tin, tout);
}

// ---- register-block variant -------------------------------------------------------------------------------------------
// The shuffle version above is bound by the shared-memory / shuffle pipe (ncu round 2: short-scoreboard stalls 13 of 30 cycles per
// issue, L1 pipe 77 % busy, 8.4 M warp instructions for the stabilizer half at d=71): seven such operations per 32x32 block.  Here
// ONE THREAD owns a 32x32-bit block in 32 registers and transposes it with the five swap stages as plain ALU work (two byte
// permutes per pair for the 16- and 8-bit stages), so a block costs one conflict-free shared load and one global store per word:
// about a quarter of the instructions and a seventh of the shared-memory traffic.
//   tile = 512 src rows x 16 src words (64 contiguous bytes per src row: two full sectors per load);
//   thread (warp wv, lane l): row-block l & 15, src word 2*wv + (l >> 4)  ->  a half-warp stores 16 consecutive words (64 bytes)
//   of each of its 32 dst rows straight from registers.
// Requires every stride / width / offset to be a multiple of four 32-bit words (checked by the host).
constexpr int kTrRows = 512, kTrWords = 16, kTrBlkStride = 32 * kTrWords + 2;     // +2 words: the 16 row-blocks x 2 words of a warp hit 32 distinct banks
constexpr int kTrSmemWords = (kTrRows / 32) * kTrBlkStride;
__device__ __forceinline__ void transpose_tile_regs(const u32* __restrict__ src, size_t src_stride, int src_rows, int src_words,
                                                    u32* __restrict__ dst, size_t dst_stride, int dst_rows, int dst_words,
                                                    int bx, int by, u32* tin) {
    const int c0 = bx * kTrRows, w0 = by * kTrWords;
    const int t = threadIdx.x;
    {
        // thread t loads 16 bytes of src rows (t >> 2) + 64 k: one pointer, advanced by 64 rows (the kernel is issue bound --
        // ncu round 2: 56 % issue active at 50 % occupancy -- so the address arithmetic is kept out of the unrolled bodies)
        const int part = t & 3, r0 = t >> 2;
        const int gw = w0 + 4 * part;
        const uint4* sp = reinterpret_cast<const uint4*>(src + (size_t)(c0 + r0) * src_stride + gw);
        const size_t sstep = (size_t)16 * src_stride;           // 64 rows, in uint4
        u32* p = tin + (r0 >> 5) * kTrBlkStride + (r0 & 31) * kTrWords + 4 * part;      // 8-byte aligned (kTrBlkStride is even)
        const bool wok = gw < src_words;
        const int rleft = src_rows - c0 - r0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            uint4 v = make_uint4(0, 0, 0, 0);
            if (wok && 64 * k < rleft) v = __ldcg(sp);
            sp += sstep;
            *reinterpret_cast<uint2*>(p + 2 * k * kTrBlkStride) = make_uint2(v.x, v.y);
            *reinterpret_cast<uint2*>(p + 2 * k * kTrBlkStride + 2) = make_uint2(v.z, v.w);
        }
    }
    __syncthreads();
    const int lane = t & 31, blk = lane & 15, word = 2 * (t >> 5) + (lane >> 4);
    u32 a[32];
    const u32* q = tin + blk * kTrBlkStride + word;
#pragma unroll
    for (int i = 0; i < 32; ++i) a[i] = q[i * kTrWords];
    // a[i] bit b  ->  a[b] bit i ; skipped by a warp whose 32 blocks are all zero (tableaux of local codes are mostly zero blocks
    // away from a band around the diagonal, and the kernel is issue bound)
    u32 any = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) any |= a[i];
    if (__any_sync(0xffffffffu, any != 0)) {
#pragma unroll
        for (int k = 0; k < 16; ++k) { const u32 lo = a[k], hi = a[k + 16]; a[k] = __byte_perm(lo, hi, 0x5410u); a[k + 16] = __byte_perm(lo, hi, 0x7632u); }
#pragma unroll
        for (int k = 0; k < 32; ++k) if (!(k & 8)) { const u32 lo = a[k], hi = a[k + 8]; a[k] = __byte_perm(lo, hi, 0x6240u); a[k + 8] = __byte_perm(lo, hi, 0x7351u); }
#pragma unroll
        for (int k = 0; k < 32; ++k) if (!(k & 4)) { const u32 x = ((a[k] >> 4) ^ a[k + 4]) & 0x0f0f0f0fu; a[k + 4] ^= x; a[k] ^= x << 4; }
#pragma unroll
        for (int k = 0; k < 32; ++k) if (!(k & 2)) { const u32 x = ((a[k] >> 2) ^ a[k + 2]) & 0x33333333u; a[k + 2] ^= x; a[k] ^= x << 2; }
#pragma unroll
        for (int k = 0; k < 32; ++k) if (!(k & 1)) { const u32 x = ((a[k] >> 1) ^ a[k + 1]) & 0x55555555u; a[k + 1] ^= x; a[k] ^= x << 1; }
    }
    const int gw = (c0 >> 5) + blk;
    if (gw < dst_words) {
        u32* d = dst + (size_t)(32 * (w0 + word)) * dst_stride + gw;
        const int left = dst_rows - 32 * (w0 + word);
        if (left >= 32) {
#pragma unroll
            for (int b = 0; b < 32; ++b) { __stcg(d, a[b]); d += dst_stride; }
        } else {
#pragma unroll
            for (int b = 0; b < 32; ++b) { if (b < left) __stcg(d, a[b]); d += dst_stride; }
        }
    }
}
__global__ void __launch_bounds__(256, 4)
k_transpose_regs(const u32* __restrict__ src, size_t src_stride, int src_rows, int src_words,
                 u32* __restrict__ dst, size_t dst_stride, int dst_rows, int dst_words,
                 size_t src_zoff, size_t dst_zoff, const u32* __restrict__ flag) {
    __shared__ __align__(16) u32 tin[kTrSmemWords];
    pdl_trigger();
    pdl_wait();
    if (flag && __ldcg(flag) == 0u) return;
    transpose_tile_regs(src + (size_t)blockIdx.z * src_zoff, src_stride, src_rows, src_words, dst + (size_t)blockIdx.z * dst_zoff, dst_stride, dst_rows, dst_words,
                        blockIdx.x, blockIdx.y, tin);
}

// The same tile move as a device function for use inside a persistent kernel: `nthr` = 256 threads of one half-CTA
// (thread index t in [0,256)), synchronised with the named barrier `bar_id`; tin/tout = 2 x 256 x 9 words of shared memory.
__device__ __forceinline__ void transpose_tile_256(const u32* __restrict__ src, size_t src_stride, int src_rows, int src_words,
                                                   u32* __restrict__ dst, size_t dst_stride, int dst_rows, int dst_words,
                                                   int c0, int w0, int t, int bar_id, u32 (*tin)[9], u32 (*tout)[9]) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        int rr = k * 32 + (t >> 3), ww = t & 7;
        int gr = c0 + rr, gw = w0 + ww;
        u32 v = 0;
        if (gr < src_rows && gw < src_words) v = __ldcg(src + (size_t)gr * src_stride + gw);
        tin[rr][ww] = v;
    }
    asm volatile("bar.sync %0, 256;" ::"r"(bar_id) : "memory");
    const int warp = t >> 5, lane = t & 31;
#pragma unroll
    for (int bj = 0; bj < 8; ++bj) {
        tout[bj * 32 + lane][warp] = transpose32(tin[warp * 32 + lane][bj], lane);
    }
    asm volatile("bar.sync %0, 256;" ::"r"(bar_id) : "memory");
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        int rr = k * 32 + (t >> 3), ww = t & 7;
        int gr = w0 * 32 + rr, gw = (c0 >> 5) + ww;
        if (gr < dst_rows && gw < dst_words) __stcg(dst + (size_t)gr * dst_stride + gw, tout[rr][ww]);
    }
    asm volatile("bar.sync %0, 256;" ::"r"(bar_id) : "memory");      // tin/tout are reused by the next tile
}

// sign bit-vector <-> one byte per row (host ABI); rowbit = map of tableau row index
__global__ void k_signs_to_bytes(const u64* __restrict__ sgn, uint8_t* __restrict__ out, int nrows, int split, int NS) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nrows) return;
    int rb = (i < split) ? i : NS + (i - split);
    out[i] = uint8_t((__ldcg(sgn + (rb >> 6)) >> (rb & 63)) & 1ull);
}
__global__ void k_bytes_to_signs(const uint8_t* __restrict__ in, u64* __restrict__ sgn, int nrows, int split, int NS) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nrows) return;
    int rb = (i < split) ? i : NS + (i - split);
    if (in[i]) atomicOr(&sgn[rb >> 6], 1ull << (rb & 63));
}

// sign bytes of rows [first, first + nrows) of a plain row set (no stabilizer / destabilizer split): set or clear each bit
__global__ void k_bytes_to_signs_at(const uint8_t* __restrict__ in, u64* __restrict__ sgn, int nrows, int first) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nrows) return;
    const int rb = first + i;
    if (in[i]) atomicOr(&sgn[rb >> 6], 1ull << (rb & 63)); else atomicAnd(&sgn[rb >> 6], ~(1ull << (rb & 63)));
}

// host row-major (nrows x W, separate x / z arrays) <-> device R form (stride 2*Wp, row-bit mapped)
__global__ void k_pack_rows(const u64* __restrict__ hx, const u64* __restrict__ hz, u64* __restrict__ rows,
                            int nrows, int W, int Wp, int split, int NS) {
    size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)nrows * W) return;
    int i = int(idx / W), w = int(idx % W);
    int rb = (i < split) ? i : NS + (i - split);
    rows[(size_t)(2 * rb) * Wp + w] = hx[idx];
    rows[(size_t)(2 * rb + 1) * Wp + w] = hz[idx];
}
__global__ void k_unpack_rows(const u64* __restrict__ rows, u64* __restrict__ hx, u64* __restrict__ hz,
                              int nrows, int W, int Wp, int split, int NS) {
    size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)nrows * W) return;
    int i = int(idx / W), w = int(idx % W);
    int rb = (i < split) ? i : NS + (i - split);
    hx[idx] = __ldcg(rows + (size_t)(2 * rb) * Wp + w);
    hz[idx] = __ldcg(rows + (size_t)(2 * rb + 1) * Wp + w);
}

// identity tableau in both forms: stabilizer q = Z_q, destabilizer q = X_q
__global__ void k_identity(u64* __restrict__ cols, u64* __restrict__ rows, int n, int RW, int Wp, int NS) {
    int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const u64 qb = 1ull << (q & 63);
    // C: z column of qubit q has bit (row q); x column has bit (row NS+q)
    cols[(size_t)(2 * q + 1) * RW + (q >> 6)] = qb;
    cols[(size_t)(2 * q) * RW + ((NS + q) >> 6)] = 1ull << ((NS + q) & 63);
    // R: row q has z bit q ; row NS+q has x bit q
    rows[(size_t)(2 * q + 1) * Wp + (q >> 6)] = qb;
    rows[(size_t)(2 * (NS + q)) * Wp + (q >> 6)] = qb;
}

}  // namespace skd
