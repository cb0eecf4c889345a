// Probe: how a tcgen05.mma kind::f16 with an F16 accumulator (c_format 0) stores D in TMEM
// (one value per 32-bit column, low or high half, or two per column) and how it reads the
// accumulator back when accumulate = 1.  A = B = 1.0, M=128, N=64, K=16 -> D = 16 (+ C).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2410_02367_b200/csrc/sab_ptx.cuh"
using namespace sab;
__global__ void k(uint32_t fill, int acc, uint32_t* out) {
    __shared__ __align__(1024) uint16_t ab[8192];
    __shared__ uint32_t tb;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) ab[i] = 0x3C00;
    if (warp == 0) tmem_alloc<128>(smem_u32(&tb));
    if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); fence_barrier_init(); }
    fence_proxy_async_smem();
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t t = tb + ((uint32_t)(warp * 32) << 16);
    tmem_fill32(t, fill); tmem_fill32(t + 32, fill); tmem_fill32(t + 64, fill); tmem_fill32(t + 96, fill);
    tmem_wait_st();
    tc_fence_before(); __syncthreads(); tc_fence_after();
    if (threadIdx.x == 0) {
        const uint64_t da = make_smem_desc(smem_u32(ab), 128, 256, kSwizzleNone);
        const uint64_t db = make_smem_desc(smem_u32(ab + 4096), 128, 256, kSwizzleNone);
        umma_f16_ss(tb, da, db, make_idesc(0 /*F16*/, 0, 0, 0, 0, 128, 64), acc);
        umma_commit(smem_u32(&bar));
    }
    mbar_wait(smem_u32(&bar), 0);
    tc_fence_after();
    uint32_t r[32];
    for (int c = 0; c < 128; c += 32) {
        tmem_ld32(t + c, r); tmem_wait_ld();
        for (int i = 0; i < 32; ++i) out[threadIdx.x * 128 + c + i] = r[i];
    }
    tc_fence_before(); __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc<128>(tb); }
}
int main() {
    uint32_t* d; cudaMalloc(&d, 128 * 128 * 4);
    static uint32_t h[128 * 128];
    const uint32_t fills[3] = {0xDEADBEEFu, 0x00003C00u, 0x3C000000u};
    const int accs[3] = {0, 1, 1};
    for (int t = 0; t < 3; ++t) {
        k<<<1, 128>>>(fills[t], accs[t], d);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        printf("fill=%08x acc=%d err=%s\n", fills[t], accs[t], cudaGetErrorString(e));
        for (int row : {0, 77}) {
            printf(" row %d:", row);
            for (int c : {0, 1, 2, 31, 32, 33, 63, 64, 65, 127}) printf(" [%d]%08x", c, h[row * 128 + c]);
            printf("\n");
        }
    }
    return 0;
}
