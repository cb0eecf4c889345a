// Microbenchmark: issue cost of the K2 MMA shapes on sm_100a (one CTA per SM, one
// issuing thread, back-to-back MMAs into TMEM, then commit + wait).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2410_02367_b200/csrc/sab_ptx.cuh"
using namespace sab;

template <int MODE>
__global__ void k(int iters, long long* cyc) {
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tb;
    __shared__ uint64_t bar;
    for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
    if (threadIdx.x < 32) tmem_alloc<512>(smem_u32(&tb));
    if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); fence_barrier_init(); }
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t t = tb;
    const uint32_t sa = smem_u32(sm), sb = smem_u32(sm + 32768), sv = smem_u32(sm + 65536);
    if (threadIdx.x == 0) {
        // QK: A = 128x128 int8 (SW128, SBO 1024), B = 64x128 int8; PV: V 64x128 fp16 MN-major SW128 panels.
        const uint64_t da = make_smem_desc(sa, 16, 1024, kSwizzle128B);
        const uint64_t db = make_smem_desc(sb, 16, 1024, kSwizzle128B);
        const uint64_t dv = make_smem_desc(sv, 64 * 64 * 2, 1024, kSwizzle128B);
        const uint64_t dbias = make_smem_desc(sa, 128, 256, kSwizzleNone);
        constexpr uint32_t i_qk64 = make_idesc(2, 1, 1, 0, 0, 128, 64);
        constexpr uint32_t i_qk128 = make_idesc(2, 1, 1, 0, 0, 128, 128);
        constexpr uint32_t i_qk256 = make_idesc(2, 1, 1, 0, 0, 128, 256);
        constexpr uint32_t i_bias = make_idesc(1, 0, 0, 0, 0, 128, 64);
        constexpr uint32_t i_pv128 = make_idesc(1, 0, 0, 0, 1, 128, 128);
        constexpr uint32_t i_pv64 = make_idesc(1, 0, 0, 0, 1, 128, 64);
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                if (MODE == 0) umma_i8_ss(t, da + kk * 2, db + kk * 2, i_qk64, 1);
                if (MODE == 1) umma_i8_ss(t, da + kk * 2, db + kk * 2, i_qk128, 1);
                if (MODE == 2) umma_i8_ss(t, da + kk * 2, db + kk * 2, i_qk256, 1);
                if (MODE == 3) umma_f16_ss(t, dbias, dbias, i_bias, 1);
                if (MODE == 4) umma_f16_ts(t + 256, t + kk * 8, dv + kk * 128, i_pv128, 1);
                if (MODE == 5) umma_f16_ts(t + 256, t + kk * 8, dv + kk * 128, i_pv64, 1);
                if (MODE == 6) {  // one K2 step for one query tile (d=128): bias + 4 QK + 4 PV
                    if (kk == 0) umma_f16_ss(t, dbias, dbias, i_bias, 0);
                    umma_i8_ss(t, da + kk * 2, db + kk * 2, i_qk64, 1);
                }
                if (MODE == 6) umma_f16_ts(t + 256, t + 64 + kk * 8, dv + kk * 128, i_pv128, 1);
                if (MODE == 7) umma_i8_ts(t, t + 384 + kk * 8, db + kk * 2, i_qk64, 1);
                if (MODE == 8) umma_f16_ts(t, t + 384, dbias, i_bias, 1);
                if (MODE == 9) {  // one K2 step for one query tile (d=64), SS QK + SS bias
                    if (kk == 0) umma_f16_ss(t, dbias, dbias, i_bias, 0);
                    if (kk < 2) umma_i8_ss(t, da + kk * 2, db + kk * 2, i_qk64, 1);
                    umma_f16_ts(t + 256, t + 64 + kk * 8, dv + kk * 128, i_pv64, 1);
                }
                if (MODE == 10) {  // same with Q^ and the bias A operand in TMEM
                    if (kk == 0) umma_f16_ts(t, t + 416, dbias, i_bias, 0);
                    if (kk < 2) umma_i8_ts(t, t + 384 + kk * 8, db + kk * 2, i_qk64, 1);
                    umma_f16_ts(t + 256, t + 64 + kk * 8, dv + kk * 128, i_pv64, 1);
                }
            }
        }
        umma_commit(smem_u32(&bar));
        mbar_wait_spin(smem_u32(&bar), 0);
        long long t1 = clock64();
        cyc[blockIdx.x] = t1 - t0;
    }
    tc_fence_before(); __syncthreads();
    if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc<512>(t); }
}
template <int MODE> void run(const char* name, long long* cyc, double floor_per) {
    const int iters = 4096;
    cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    k<MODE><<<148, 128, 100 * 1024>>>(iters, cyc);
    k<MODE><<<148, 128, 100 * 1024>>>(iters, cyc);
    long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-34s %.1f cycles per group of 4 (ideal %.0f)\n", name, double(h) / iters, floor_per);
}
int main() {
    long long* cyc; cudaMalloc(&cyc, 148 * 8);
    run<0>("i8 SS 128x64x32 (QK)", cyc, 4 * 32);
    run<1>("i8 SS 128x128x32", cyc, 4 * 64);
    run<2>("i8 SS 128x256x32", cyc, 4 * 128);
    run<3>("f16 SS 128x64x16 (bias)", cyc, 4 * 32);
    run<4>("f16 TS 128x128x16 (PV d128)", cyc, 4 * 64);
    run<5>("f16 TS 128x64x16 (PV d64)", cyc, 4 * 32);
    run<6>("K2 tile step d128 (bias+QK+PV)", cyc, 32 + 128 + 256);
    run<7>("i8 TS 128x64x32 (QK, Q in TMEM)", cyc, 4 * 32);
    run<8>("f16 TS 128x64x16 (bias, A in TMEM)", cyc, 4 * 32);
    run<9>("K2 tile step d64 SS", cyc, 32 + 64 + 128);
    run<10>("K2 tile step d64 TS (Q, bias in TMEM)", cyc, 32 + 64 + 128);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
