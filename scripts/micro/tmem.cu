// Microbenchmark: tcgen05.ld / tcgen05.st throughput per SM on sm_100a.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2410_02367_b200/csrc/sab_ptx.cuh"
using namespace sab;
template <int MODE>  // 0: ld 32x32b.x32, 1: ld 16x32bx2.x32, 2: st 32x32b.x32, 3: ld x32 without per-ld wait (4 in flight)
__global__ void k(uint32_t* out, int iters, long long* cyc) {
    __shared__ uint32_t tb;
    const int warp = threadIdx.x / 32;
    if (warp == 0) tmem_alloc<512>(smem_u32(&tb));
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t base = tb + ((uint32_t)((warp % 4) * 32) << 16) + (warp / 4) * 32 % 512;
    uint32_t acc = 0;
    uint32_t r[32];
    for (int i = 0; i < 32; ++i) r[i] = i;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) { tmem_ld32(base, r); tmem_wait_ld(); for (int q = 0; q < 32; ++q) acc ^= r[q]; }
        if (MODE == 1) { tmem_ld16x2_32(base, r); tmem_wait_ld(); for (int q = 0; q < 32; ++q) acc ^= r[q]; }
        if (MODE == 2) { r[0] = it; r[1] ^= acc; tmem_st32(base, r); tmem_wait_st(); }
        if (MODE == 3) {
            uint32_t a[32], b[32], c[32], d[32];
            tmem_ld32(base, a); tmem_ld32(base + 32, b); tmem_ld32(base + 64, c); tmem_ld32(base + 96, d);
            tmem_wait_ld(); for (int q = 0; q < 32; ++q) acc ^= a[q] ^ b[q] ^ c[q] ^ d[q];
        }
    }
    __syncthreads();
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    tc_fence_before(); __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tb); }
}
template <int MODE> void run(const char* name, int warps, uint32_t* out, long long* cyc) {
    int iters = 2048;
    k<MODE><<<148, warps * 32>>>(out, iters, cyc);
    k<MODE><<<148, warps * 32>>>(out, iters, cyc);
    long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    double bytes = double(iters) * warps * 4096 * (MODE == 3 ? 4 : 1);
    printf("%-28s warps %2d: %.1f B/clk/SM  (%.0f cyc per op per warp)\n", name, warps, bytes / h, double(h) / iters);
}
int main() {
    uint32_t* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
    for (int w : {1, 4, 8, 16}) run<0>("ld 32x32b.x32 + wait", w, out, cyc);
    for (int w : {4, 16}) run<1>("ld 16x32bx2.x32 + wait", w, out, cyc);
    for (int w : {4, 16}) run<3>("4x ld 32x32b.x32, one wait", w, out, cyc);
    for (int w : {1, 4, 16}) run<2>("st 32x32b.x32 + wait", w, out, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
