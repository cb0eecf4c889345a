// sab_peak.cu -- measured tcgen05 tensor-pipe peaks for bench.py's roofline (bench
// infrastructure, not part of the SageAttn library).
//
// One CTA per SM, one elected thread issues back-to-back dense MMAs of shape
// M=128, N=256 (the largest cta_group::1 tile) from SMEM operands filled with
// pseudo-random data into a TMEM accumulator:
//   kind::i8  (K=32 per instruction, int32 accumulate) -> INT8 ops / clk / SM
//   kind::f16 (K=16 per instruction, fp32 accumulate)  -> FP16 flops / clk / SM
// The result is a per-cycle rate (SM clock64), so bench.py can turn it into the
// peak at the clock its own kernel actually ran at (sampled through NVML).
//
//   extern "C" int sab_peak_probe(int kind, int iters, double* ops_per_clk_per_sm,
//                                 double* ops_per_s, double* mhz)
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_2410_02367_b200/csrc/sab_ptx.cuh"

using namespace sab;

namespace {

constexpr int kM = 128, kN = 256;

template <bool I8>
__global__ void __launch_bounds__(128, 1) peak_kernel(int iters, long long* cycles) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tbase;
    __shared__ uint64_t bar;
    // A: 128 x 128 bytes, B: 256 x 128 bytes (K = 128 int8 or 64 fp16 per stage), SW128.
    constexpr int kBytes = (kM + kN) * 128;
    uint32_t x = 0x9E3779B9u * (blockIdx.x + 1);
    for (int i = threadIdx.x; i < kBytes / 4; i += blockDim.x) {
        uint32_t h = (x ^ (i * 0x85EBCA6Bu)) * 0xC2B2AE35u;
        h ^= h >> 13;
        // int8: random codes in [-64, 63]; fp16: random values in [0.5, 1) with random sign
        reinterpret_cast<uint32_t*>(sm)[i] = I8 ? (h & 0x7F7F7F7Fu) - 0x40404040u : ((h & 0x83FF83FFu) | 0x38003800u);
    }
    fence_proxy_async_smem();
    if (threadIdx.x < 32) tmem_alloc<256>(smem_u32(&tbase));
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&bar), 1);
        fence_barrier_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x == 0) {
        const uint32_t sa = smem_u32(sm), sb = sa + kM * 128;
        const uint64_t da = make_smem_desc(sa, 16, 1024, kSwizzle128B);
        const uint64_t db = make_smem_desc(sb, 16, 1024, kSwizzle128B);
        constexpr uint32_t idesc = I8 ? make_idesc(2, 1, 1, 0, 0, kM, kN) : make_idesc(1, 0, 0, 0, 0, kM, kN);
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {  // 4 x 32 bytes of K per row = one 128-byte swizzle atom
                if (I8)
                    umma_i8_ss(tbase, da + kk * 2, db + kk * 2, idesc, (it | kk) != 0);
                else
                    umma_f16_ss(tbase, da + kk * 2, db + kk * 2, idesc, (it | kk) != 0);
            }
        }
        umma_commit(smem_u32(&bar));
        mbar_wait_spin(smem_u32(&bar), 0);
        cycles[blockIdx.x] = clock64() - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tc_fence_after();
        tmem_dealloc<256>(tbase);
    }
}

}  // namespace

extern "C" int sab_peak_probe(int kind, int iters, double* ops_per_clk_per_sm, double* ops_per_s, double* mhz) {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
        return 1;
    const bool i8 = kind == 0;
    auto kern = i8 ? peak_kernel<true> : peak_kernel<false>;
    const int smem = (kM + kN) * 128 + 1024;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return 2;
    long long* cyc = nullptr;
    if (cudaMalloc(&cyc, sizeof(long long) * sms) != cudaSuccess) return 3;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    kern<<<sms, 128, smem>>>(iters / 4 + 1, cyc);  // warm-up
    cudaEventRecord(a);
    kern<<<sms, 128, smem>>>(iters, cyc);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    long long host[1024];
    if (e == cudaSuccess) e = cudaMemcpy(host, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    cudaFree(cyc);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    if (e != cudaSuccess) return 4;
    double mean_cyc = 0;
    for (int i = 0; i < sms; ++i) mean_cyc += double(host[i]) / sms;
    // ops per instruction: 2 * M * N * K, K = 32 (i8) or 16 (f16)
    const double ops = 2.0 * kM * kN * (i8 ? 32 : 16) * 4.0 * iters;
    *ops_per_clk_per_sm = ops / mean_cyc;
    *ops_per_s = ops * sms / (ms * 1e-3);
    *mhz = mean_cyc / (ms * 1e-3) / 1e6;
    return 0;
}
