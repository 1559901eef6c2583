// microbench: cost of one "factorise step" skeleton (REDUX + STS + named barrier + LDS ...) in one CTA,
// alone vs while the other CTAs of a cooperative grid spin on a global barrier word.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64; typedef unsigned int u32;
__device__ __forceinline__ u32 ld_acq(const u32* p) { u32 v; asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ u32 ld_rlx(const u32* p) { u32 v; asm volatile("ld.relaxed.gpu.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
// mode: 0 = other CTAs exit at once; 1 = spin with ld.acquire; 2 = spin with ld.relaxed + nanosleep
__global__ void step(u32* flag, int iters, int Tact, int mode, u64* out, u32 seed) {
    __shared__ u32 wmin[2][16]; __shared__ u64 bp[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (blockIdx.x != 0) {
        if (mode == 0) return;
        if (threadIdx.x == 0) {
            if (mode == 1) while (ld_acq(flag) == 0) {}
            else while (ld_rlx(flag) == 0) { __nanosleep(200); }
        }
        __syncthreads();
        return;
    }
    u64 b = seed * 0x9e3779b97f4a7c15ull + tid; u32 h = tid * 7 + 1;
    long long c0 = clock64();
    if (tid < Tact) {
        for (int j = 0; j < iters; ++j) {
            u32 m = ((b >> (j & 63)) & 1) ? h : 0xffffffffu;
            m = __reduce_min_sync(0xffffffffu, m);
            if (lane == 0) wmin[j & 1][warp] = m;
            named_bar(1, Tact);
            u32 p = 0xffffffffu;
            for (int t = 0; t < (Tact >> 5); ++t) p = min(p, wmin[j & 1][t]);
            if (h == p) bp[j & 1] = b;
            named_bar(1, Tact);
            const u64 x = bp[j & 1];
            if ((b >> (j & 63)) & 1) b ^= x * 3 + j;
            h += (u32)(x & 1);
        }
    }
    long long c1 = clock64();
    __syncthreads();
    if (tid == 0) { out[0] = c1 - c0; out[1] = b + h; atomicExch(flag, 1u); }
}
int main() {
    u64* out; cudaMallocManaged(&out, 64);
    u32* flag; cudaMalloc(&flag, 4);
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int mode = 0; mode < 3; ++mode)
        for (int Tact : {32, 64, 192, 512}) {
            int iters = 20000; u32 seed = 12345;
            void* args[] = {&flag, &iters, &Tact, &mode, &out, &seed};
            for (int rep = 0; rep < 2; ++rep) {
                cudaMemset(flag, 0, 4);
                cudaLaunchCooperativeKernel((void*)step, dim3(sms), dim3(512), args, 0, 0);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
            }
            printf("mode %d (0 alone, 1 others spin ld.acquire, 2 others spin relaxed+nanosleep)  Tact %3d : %.0f cycles/step\n", mode, Tact, double(out[0]) / iters);
        }
    return 0;
}
