// microbench: dependent-load latency (ld.cg / ld.ca) for various footprints, grid barrier latency.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
typedef unsigned long long u64; typedef unsigned int u32;
__device__ __forceinline__ u64 gtime() { u64 t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__global__ void chase(const u32* p, int iters, int mode, u64* out) {
    u32 i = 0; u64 t0 = gtime(); long long c0 = clock64();
    for (int k = 0; k < iters; ++k) i = mode ? __ldcg(p + i) : p[i];
    long long c1 = clock64(); u64 t1 = gtime();
    out[0] = t1 - t0; out[1] = c1 - c0; out[2] = i;
}
__device__ __forceinline__ u32 ld_acq(const u32* p) { u32 v; asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__global__ void bar_mine(u32* bar, int iters, u64* out) {
    u32 epoch = 0; u64 t0 = gtime();
    for (int k = 0; k < iters; ++k) {
        epoch += gridDim.x; __syncthreads();
        if (threadIdx.x == 0) { __threadfence(); atomicAdd(bar, 1u); while (int(ld_acq(bar) - epoch) < 0) {} __threadfence(); }
        __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = gtime() - t0;
}
__global__ void bar_cg(int iters, u64* out) {
    cg::grid_group g = cg::this_grid(); u64 t0 = gtime();
    for (int k = 0; k < iters; ++k) g.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = gtime() - t0;
}
// lighter barrier: no trailing fence, relaxed polling with nanosleep
__global__ void bar_light(u32* bar, int iters, u64* out) {
    u32 epoch = 0; u64 t0 = gtime();
    for (int k = 0; k < iters; ++k) {
        epoch += gridDim.x; __syncthreads();
        if (threadIdx.x == 0) { asm volatile("red.release.gpu.global.add.u32 [%0], 1;" :: "l"(bar) : "memory"); while (int(ld_acq(bar) - epoch) < 0) {} }
        __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = gtime() - t0;
}
int main() {
    u64* out; cudaMallocManaged(&out, 64);
    for (size_t mb : {1, 32, 100, 400}) {
        size_t n = mb * (1 << 20) / 4; std::vector<u32> h(n);
        // random cyclic permutation with stride >= 128B
        size_t lines = n / 32; std::vector<u32> perm(lines); for (size_t i = 0; i < lines; ++i) perm[i] = i;
        srand(1); for (size_t i = lines - 1; i > 0; --i) { size_t j = rand() % (i + 1); std::swap(perm[i], perm[j]); }
        for (size_t i = 0; i < lines; ++i) h[perm[i] * 32] = perm[(i + 1) % lines] * 32;
        u32* d; cudaMalloc(&d, n * 4); cudaMemcpy(d, h.data(), n * 4, cudaMemcpyHostToDevice);
        for (int mode = 0; mode < 2; ++mode) {
            chase<<<1, 1>>>(d, 20000, mode, out); cudaDeviceSynchronize();   // warm
            chase<<<1, 1>>>(d, 20000, mode, out); cudaDeviceSynchronize();
            printf("chase %4zu MB %s: %.1f ns/load (%.0f cycles)\n", mb, mode ? "ld.cg" : "ld.ca", out[0] / 20000.0, out[1] / 20000.0);
        }
        cudaFree(d);
    }
    u32* bar; cudaMalloc(&bar, 4);
    int dev = 0, sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    for (int threads : {64, 512}) {
        int iters = 2000; void* args1[] = {&bar, &iters, &out};
        cudaMemset(bar, 0, 4); cudaLaunchCooperativeKernel((void*)bar_mine, dim3(sms), dim3(threads), args1, 0, 0); cudaDeviceSynchronize();
        printf("barrier mine   %d thr: %.2f us\n", threads, out[0] / 1e3 / iters);
        cudaMemset(bar, 0, 4); cudaLaunchCooperativeKernel((void*)bar_light, dim3(sms), dim3(threads), args1, 0, 0); cudaDeviceSynchronize();
        printf("barrier light  %d thr: %.2f us\n", threads, out[0] / 1e3 / iters);
        void* args2[] = {&iters, &out};
        cudaLaunchCooperativeKernel((void*)bar_cg, dim3(sms), dim3(threads), args2, 0, 0); cudaDeviceSynchronize();
        printf("barrier cg     %d thr: %.2f us   (%s)\n", threads, out[0] / 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
