// common.cuh -- device helpers shared by all stabkit-b200 kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "stabkit_b200.h"

namespace skd {

using u64 = unsigned long long;
using u32 = unsigned int;

// ---- data layout -----------------------------------------------------------
// A set of signed n-qubit Pauli rows lives on the device in up to two forms:
//
//  C ("qubit-major", the gate form): for every qubit j two bit-columns over the
//    rows, x then z, RW 64-bit words each:   cols[(2*j + h) * RW + w]
//    bit b of word w is row 64*w + b.  Signs: sgn[w], same row-bit space.
//    A gate on qubit j touches 2 contiguous columns -> exactly the algorithmic
//    bytes of SURVEY.md section 8d, coalesced, 64 rows per ALU op.
//
//  R ("row-major", the measurement form): for every row-bit r the x words then
//    the z words, Wp words each:            rows[(2*r + h) * Wp + w]
//    Rowsum reads/writes whole rows: one contiguous 16*Wp-byte block per row.
//
// For a CHP tableau stabilizer i is row-bit i and destabilizer i is
// row-bit NS + i with NS = 64*W, W = ceil(n/64): both halves are word aligned
// (RW = 2*W).  Padding rows/bits are all-zero and stay zero under every rule.
struct DMat {
    uint64_t n = 0;     // qubits
    uint32_t W = 0;     // ceil(n/64)
    uint32_t Wp = 0;    // W rounded up to even (16-byte aligned half rows)
    uint32_t RW = 0;    // row words (even)
    u64* cols = nullptr;
    u64* sgn = nullptr;
    u64* rows = nullptr;
};

// ---- memory ----------------------------------------------------------------
// Loads of data another CTA may have written during this launch bypass L1.
__device__ __forceinline__ u64 ldcg(const u64* p) { return __ldcg(p); }
__device__ __forceinline__ u32 ld_acquire(const u32* p) {
    u32 v; asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}

// ---- programmatic dependent launch (sm_90+): a kernel launched with cudaLaunchAttributeProgrammaticStreamSerialization may be
// scheduled while its predecessor in the stream still runs; pdl_wait() blocks until the predecessor has completed and its writes
// are visible (a no-op for a normal launch), pdl_trigger() lets the successor start being scheduled.  Hides the launch latency
// between the small dependent kernels of a Clifford run.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---- rng (ref: proj/include/stabkit/rng.hpp:23-39) ---------------------------
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
__host__ __device__ __forceinline__ int counter_bit(uint64_t seed, uint64_t ordinal) {
    return int(splitmix64(seed ^ splitmix64(ordinal ^ 0xd1b54a32d192ed03ULL)) & 1);
}

// ---- Pauli phase arithmetic (ref: proj/src/pauli.cpp:189-205) -
// i-exponent of the product a*b (a = LEFT factor) over one word: +1 for
// (X,Y),(Y,Z),(Z,X), -1 for the reversed pairs.  Only the value mod 4 is used.
__device__ __forceinline__ int g_word(u64 ax, u64 az, u64 bx, u64 bz) {
    u64 anti = (ax & bz) ^ (bx & az);
    // +i positions: a=X,b=Y | a=Y,b=Z | a=Z,b=X
    u64 plus = anti & ((ax & ~az & bx) | (ax & az & ~bx) | (~ax & az & ~bz));
    return __popcll(plus) - __popcll(anti & ~plus);
}

// (one REDUX instruction each instead of five shuffle + op steps)
__device__ __forceinline__ int warp_sum(int v) { return __reduce_add_sync(0xffffffffu, v); }
__device__ __forceinline__ u32 warp_min(u32 v) { return __reduce_min_sync(0xffffffffu, v); }

// ---- grid-wide barrier for cooperative (co-resident) launches ---------------
// Monotone counter; `epoch` is the per-thread running target.  Bounded spin:
// on timeout the error flag is raised and the caller bails out (never hangs).
__device__ __forceinline__ bool grid_barrier(u32* bar, u32& epoch, u32* err) {
    __shared__ u32 s_ok;
    epoch += gridDim.x;
    __syncthreads();
    if (threadIdx.x == 0) {
        // arrive: one release reduction (orders this CTA's writes -- bar.sync above made them cumulative -- before the count);
        // wait: acquire loads (the bar.sync below hands the acquired view to the other threads).  Measured against
        // fence + atomicAdd ... fence: 0.09 ms of 8.6 ms at d=71 (316 barriers).
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        u32 ok = 1;
        unsigned long long spins = 0;
        while (int(ld_acquire(bar) - epoch) < 0) {
            if (++spins > (1ull << 24)) { ok = 0; atomicExch(err, 0x80000000u); break; }
        }
        s_ok = ok;
    }
    __syncthreads();
    return s_ok != 0;
}

// ---- 1-D TMA (cp.async.bulk) global -> shared with an mbarrier --------------
__device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(u64* bar, u32 count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(u64* bar, u32 bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst_smem, const void* src_gmem, u32 bytes, u64* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst_smem)), "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// returns false on timeout
__device__ __forceinline__ bool mbar_wait(u64* bar, u32 parity) {
    u32 done = 0;
    for (u32 it = 0; it < (1u << 20); ++it) {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
        if (done) return true;
    }
    return false;
}

}  // namespace skd
