// Microbenchmark: MUFU.EX2 and FFMA2 throughput per SM on sm_100a (warps per SM varied).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
template <int ILP>
__global__ void k_ex2(float* out, int iters, long long* cyc) {
    float v[ILP];
    for (int i = 0; i < ILP; ++i) v[i] = -0.001f * (threadIdx.x + i);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < ILP; ++i) v[i] = ex2(v[i]) - 1.0f;
    long long t1 = clock64();
    float s = 0; for (int i = 0; i < ILP; ++i) s += v[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    float* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
    long long h[148];
    for (int warps : {1, 2, 4, 8, 16}) {
        int iters = 4096;
        k_ex2<16><<<148, warps * 32>>>(out, iters, cyc);
        cudaDeviceSynchronize();
        k_ex2<16><<<148, warps * 32>>>(out, iters, cyc);
        cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
        double ops = double(iters) * 16 * warps * 32;
        printf("warps/SM %2d: ex2 lanes/clk/SM = %.2f (cycles %lld)\n", warps, ops / h[0], h[0]);
    }
    return 0;
}
