// kernels_layer.cuh -- K1: one fused layer of Clifford gates on disjoint qubits,
// applied to the qubit-major (C) form.  Every touched column word is loaded once
// and stored once per layer; the sign column is updated once per layer.
//
// Row rules (per row, pre-update bits; ref: proj/src/pauli.cpp:146-187, SPEC:135-163,
// derived gates SPEC:190 collapsed to their closed forms -- same tableau result):
//   H    r ^= x&z        ; swap(x,z)
//   S    r ^= x&z        ; z ^= x
//   SDG  r ^= x&~z       ; z ^= x
//   X    r ^= z          Y   r ^= x^z          Z   r ^= x
//   CX   r ^= xc&zt&~(xt^zc) ; xt ^= xc ; zc ^= zt
//   CZ   r ^= xa&xb&(za^zb)  ; za ^= xb ; zb ^= xa
//   SWAP exchange columns
//   XCX  r ^= zc&zt&(xc^xt)     ; xc ^= zt ; xt ^= zc        (= H_c CX_{c->t} H_c, the three rules above composed)
// Here one "bit" is a 64-bit word = 64 rows, processed as 128-bit vectors.
//
// Roofline: HBM/L2 streaming.  Algorithmic bytes per gate (fused form):
// H 4 columns, S/SDG 3, X/Z 1, Y 2, CX/CZ 6, SWAP 8, times RW*8 bytes, plus 2*RW*8 per layer.
#pragma once
#include "common.cuh"

namespace skd {

// internal op kinds of the Clifford+T pass (never cross the C ABI): append a T / T-dagger row
constexpr uint8_t SK_APPEND_T = 12, SK_APPEND_TDG = 13;
// internal kind made by the host's H-window pass (compile_segment): H_c ; CX c->t ; H_c as one gate, "X-controlled X"
constexpr uint8_t SK_XCX = 14;

__device__ __forceinline__ ulonglong2 ld2(const ulonglong2* p) { return __ldcg(p); }
__device__ __forceinline__ void st2(ulonglong2* p, ulonglong2 v) { __stcg(p, v); }
__device__ __forceinline__ bool nz2(ulonglong2 v) { return (v.x | v.y) != 0; }
__device__ __forceinline__ ulonglong2 operator^(ulonglong2 a, ulonglong2 b) { return make_ulonglong2(a.x ^ b.x, a.y ^ b.y); }
__device__ __forceinline__ ulonglong2 operator&(ulonglong2 a, ulonglong2 b) { return make_ulonglong2(a.x & b.x, a.y & b.y); }
__device__ __forceinline__ ulonglong2 operator~(ulonglong2 a) { return make_ulonglong2(~a.x, ~a.y); }

// (Measured, round 2: batching the first loads of up to four independent gates per thread -- 2 dependent round trips per batch
// instead of 2 per gate -- is SLOWER, 17-23 us against 10-12 us per d=71 layer: 114 registers cut the resident warps 4x and the
// kernel is L2-bandwidth bound (about 44 MB of sector traffic per CX layer), not latency bound.  Kept as is.)
// (Measured, round 2 as well: a NONZERO MAP of the gate form -- one bit per 128-row vector of a column, kept exact by every store,
// consulted by this kernel, by the C -> R transpose and rebuilt by the in-kernel R -> C -- cuts the DRAM reads of a d=71 layer from
// 8.7 MB to 0.8 MB and those of the stabilizer-half transpose from 22.7 MB to 5 MB, and makes both SLOWER: layers 13-20 us against
// 10-12 us (map words prefetched one gate ahead, warp-owned words without atomics, grid sized to one resident wave: all tried),
// the transpose 28 us against 20 us.  Neither kernel is DRAM bound: each is bound by its chain of dependent accesses, and the
// map lookup lengthens that chain.  Reverted; bit-exact while it existed.)
// (Measured, round 2, third attempt at the chain: TWO row-vectors per thread, the loads of a gate issued for both before either
// is used, CTAs of half the threads and chunks of half the gates -- 64 registers with the two-qubit kinds folded into one body;
// d=71 whole program 8.66 ms against 8.42 ms, and the folded body alone with one vector per thread 8.82 ms.  The per-kind bodies
// below at 40 registers stay.  A cap of 32 registers -- 12 CTAs per SM instead of 9, chunks of 6 gates -- spills 40 bytes: 8.61 ms.)
// gates: ngates entries; CTA b handles gates [b*gpb, (b+1)*gpb), or [block_off[b], block_off[b+1]) when the host
// supplies chunk boundaries; thread v owns 128-bit row-vector v of every column it visits.
// Merged layers: a launch may hold several consecutive layers provided every set of gates that share qubits (a
// "cluster", e.g. H a ; CX a d) sits inside ONE chunk in program order -- the same thread then applies them in order to
// its row-vector (its own store is visible to its own later load), and no other CTA touches those columns.
__global__ void __launch_bounds__(256)
k_layer(u64* __restrict__ cols, u64* __restrict__ sgn, const sk_gate* __restrict__ gates,
        int ngates, int RW, int gpb, const u32* __restrict__ block_off) {
    pdl_trigger();
    pdl_wait();
    const int g0 = block_off ? int(block_off[blockIdx.x]) : blockIdx.x * gpb;
    const int g1 = block_off ? int(block_off[blockIdx.x + 1]) : min(ngates, g0 + gpb);
    const int RW2 = RW >> 1;
    for (int v = threadIdx.x; v < RW2; v += blockDim.x) {
        ulonglong2 s = make_ulonglong2(0, 0);
        for (int g = g0; g < g1; ++g) {
            const sk_gate G = gates[g];
            ulonglong2* xa = reinterpret_cast<ulonglong2*>(cols + (size_t)(2 * G.q0) * RW) + v;
            ulonglong2* za = xa + RW2;
            switch (G.kind) {
                case SK_H: {
                    ulonglong2 x = ld2(xa), z = ld2(za);
                    s = s ^ (x & z);
                    if (nz2(x ^ z)) { st2(xa, z); st2(za, x); }
                } break;
                case SK_S: {
                    ulonglong2 x = ld2(xa);
                    if (nz2(x)) { ulonglong2 z = ld2(za); s = s ^ (x & z); st2(za, z ^ x); }
                } break;
                case SK_SDG: {
                    ulonglong2 x = ld2(xa);
                    if (nz2(x)) { ulonglong2 z = ld2(za); s = s ^ (x & ~z); st2(za, z ^ x); }
                } break;
                case SK_X: s = s ^ ld2(za); break;
                case SK_Z: s = s ^ ld2(xa); break;
                case SK_Y: s = s ^ ld2(xa) ^ ld2(za); break;
                case SK_CX: {
                    ulonglong2* xt = reinterpret_cast<ulonglong2*>(cols + (size_t)(2 * G.q1) * RW) + v;
                    ulonglong2* zt = xt + RW2;
                    ulonglong2 xc = ld2(xa), ztv = ld2(zt);
                    bool hx = nz2(xc), hz = nz2(ztv);
                    if (hx | hz) {                       // all-zero source words: nothing moves
                        ulonglong2 xtv = ld2(xt), zc = ld2(za);
                        s = s ^ (xc & ztv & ~(xtv ^ zc));
                        if (hx) st2(xt, xtv ^ xc);
                        if (hz) st2(za, zc ^ ztv);
                    }
                } break;
                case SK_XCX: {
                    ulonglong2* xt = reinterpret_cast<ulonglong2*>(cols + (size_t)(2 * G.q1) * RW) + v;
                    ulonglong2* zt = xt + RW2;
                    ulonglong2 zc = ld2(za), ztv = ld2(zt);
                    bool hc = nz2(zc), ht = nz2(ztv);
                    if (hc | ht) {
                        ulonglong2 xc = ld2(xa), xtv = ld2(xt);
                        s = s ^ (zc & ztv & (xc ^ xtv));
                        if (ht) st2(xa, xc ^ ztv);
                        if (hc) st2(xt, xtv ^ zc);
                    }
                } break;
                case SK_CZ: {
                    ulonglong2* xb = reinterpret_cast<ulonglong2*>(cols + (size_t)(2 * G.q1) * RW) + v;
                    ulonglong2* zb = xb + RW2;
                    ulonglong2 x0 = ld2(xa), x1 = ld2(xb);
                    bool h0 = nz2(x0), h1 = nz2(x1);
                    if (h0 | h1) {
                        ulonglong2 z0 = ld2(za), z1 = ld2(zb);
                        s = s ^ (x0 & x1 & (z0 ^ z1));
                        if (h1) st2(za, z0 ^ x1);
                        if (h0) st2(zb, z1 ^ x0);
                    }
                } break;
                case SK_SWAP: {
                    ulonglong2* xb = reinterpret_cast<ulonglong2*>(cols + (size_t)(2 * G.q1) * RW) + v;
                    ulonglong2* zb = xb + RW2;
                    ulonglong2 x0 = ld2(xa), x1 = ld2(xb), z0 = ld2(za), z1 = ld2(zb);
                    if (nz2(x0 ^ x1)) { st2(xa, x1); st2(xb, x0); }
                    if (nz2(z0 ^ z1)) { st2(za, z1); st2(zb, z0); }
                } break;
                case SK_APPEND_T: case SK_APPEND_TDG: {      // Algorithm 2: new row q1 := (+|-) Z_q0 (row was all-zero)
                    if (int(G.q1 >> 7) == v) {
                        ulonglong2 z = ld2(za);
                        const unsigned long long bit = 1ull << (G.q1 & 63);
                        if (G.q1 & 64) { z.y |= bit; if (G.kind == SK_APPEND_TDG) s.y ^= bit; }
                        else { z.x |= bit; if (G.kind == SK_APPEND_TDG) s.x ^= bit; }
                        st2(za, z);
                    }
                } break;
                default: break;
            }
        }
        if (s.x) atomicXor(&sgn[2 * v], s.x);
        if (s.y) atomicXor(&sgn[2 * v + 1], s.y);
    }
}

// Row-major twin used for short gate runs while the R form is live: one thread
// per row-bit applies the whole (ordered) gate list to its row.  Keeps R valid
// without a full re-transposition.  Signs are NOT touched here (k_layer owns them).
__global__ void __launch_bounds__(256)
k_gates_rowmajor(u64* __restrict__ rows, const sk_gate* __restrict__ gates, int ngates, int Wp, int nrowbits) {
    int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nrowbits) return;
    u64* x = rows + (size_t)(2 * r) * Wp;
    u64* z = x + Wp;
    for (int g = 0; g < ngates; ++g) {
        const sk_gate G = gates[g];
        const u32 wa = G.q0 >> 6; const u64 ma = 1ull << (G.q0 & 63);
        switch (G.kind) {
            case SK_H: { u64 xv = x[wa], zv = z[wa]; u64 d = (xv ^ zv) & ma; if (d) { x[wa] = xv ^ d; z[wa] = zv ^ d; } } break;
            case SK_S: case SK_SDG: { u64 xv = x[wa] & ma; if (xv) z[wa] ^= xv; } break;
            case SK_CX: {
                const u32 wb = G.q1 >> 6; const u64 mb = 1ull << (G.q1 & 63);
                if (x[wa] & ma) x[wb] ^= mb;
                if (z[wb] & mb) z[wa] ^= ma;
            } break;
            case SK_CZ: {
                const u32 wb = G.q1 >> 6; const u64 mb = 1ull << (G.q1 & 63);
                bool xa_ = x[wa] & ma, xb_ = x[wb] & mb;
                if (xb_) z[wa] ^= ma;
                if (xa_) z[wb] ^= mb;
            } break;
            case SK_SWAP: {
                const u32 wb = G.q1 >> 6; const u64 mb = 1ull << (G.q1 & 63);
                bool xa_ = x[wa] & ma, xb_ = x[wb] & mb, za_ = z[wa] & ma, zb_ = z[wb] & mb;
                if (xa_ != xb_) { x[wa] ^= ma; x[wb] ^= mb; }
                if (za_ != zb_) { z[wa] ^= ma; z[wb] ^= mb; }
            } break;
            default: break;   // X, Y, Z: signs only
        }
    }
}

}  // namespace skd
