// Microbenchmark: the MMA issue sequence of one K2 CTA, without softmax or TMA,
// to locate the gap between the summed per-MMA costs (umma.cu) and the
// free-running MMA skeleton of the real kernel.  One CTA per SM, one issuing
// thread, cycles per 64-key step (two 128-row query tiles).
//
// Modes (d = 128 unless noted):
//   0  K2 order: PV_A(j), bias+QK_A(j+2) into the buffer PV_A(j) read, PV_B(j), bias+QK_B(j+2);
//      commits as in K2 (pv_done, s_full per tile, kv_empty per step)
//   1  as 0, QK writes the other S buffer (no WAR on the P columns PV just read)
//   2  as 0, order PV_A, PV_B, QK_A, QK_B
//   3  as 0, no commits
//   4  as 0, no bias MMA
//   5  3-slot S ring shared by A and B (seq s = 2j + x, slot s % 3), SS QK
//   6  as 5, Q^ from TMEM (TS QK)
//   7  as 6, no bias MMA (bound)
//   8  as 0, K/V SMEM address fixed (no 6-stage rotation)
//   9  as 0 but QK N=128 over two S buffers (one 128-key QK per two steps; S TMEM layout ignored)
//  10  as 0 plus K/V staged by bulk copies (24 KB per step from an L2-resident global buffer)
//      through the 6-stage full/empty mbarrier ring, as K2's TMA producer does
//  11  as 10 with the 3-slot ring and Q^ in TMEM (mode 6)
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../../paper_2410_02367_b200/csrc/sab_ptx.cuh"
using namespace sab;

template <int MODE>
__global__ void k(int iters, long long* cyc, const uint8_t* gkv) {
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tb;
    __shared__ uint64_t bar[8];
    __shared__ uint64_t kvf[8], kve[8];
    for (int i = threadIdx.x; i < 200 * 1024 / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(sm)[i] = make_uint4(0x01020304u * (i & 7), 0x05060708u, 0x3c003c00u, 0x11223344u);
    fence_proxy_async_smem();
    if (threadIdx.x < 32) tmem_alloc<512>(smem_u32(&tb));
    if (threadIdx.x == 0) {
        for (int i = 0; i < 8; ++i) {
            mbar_init(smem_u32(&bar[i]), 1);
            mbar_init(smem_u32(&kvf[i]), 1);
            mbar_init(smem_u32(&kve[i]), 1);
        }
        fence_barrier_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t t = tb;
    constexpr int D = 128, S = 6;
    constexpr int kQBytes = 128 * D, kKBytes = 64 * D, kVBytes = 64 * D * 2;
    const uint32_t sQ = smem_u32(sm), sK = sQ + 2 * kQBytes, sV = sK + S * kKBytes, sBias = sV + S * kVBytes;
    constexpr bool kTma = MODE >= 10;
    if (kTma && threadIdx.x == 32) {  // producer: K^ (8 KB) + V (16 KB) per step
        const uint8_t* src = gkv + static_cast<size_t>(blockIdx.x % 16) * (1 << 20);
        for (int j = 0; j < iters + 2; ++j) {
            const int s = j % S;
            mbar_wait(smem_u32(&kve[s]), ((j / S) & 1) ^ 1);
            mbar_arrive_expect_tx(smem_u32(&kvf[s]), kKBytes + kVBytes);
            const size_t off = static_cast<size_t>(j % 32) * (kKBytes + kVBytes);
            bulk_load(sK + s * kKBytes, src + off, kKBytes, smem_u32(&kvf[s]));
            bulk_load(sV + s * kVBytes, src + off + kKBytes, kVBytes, smem_u32(&kvf[s]));
        }
    }
    if (threadIdx.x == 0) {
        const uint64_t dq0 = make_smem_desc(sQ, 16, 8 * D, kSwizzle128B);
        const uint64_t dk0 = make_smem_desc(sK, 16, 8 * D, kSwizzle128B);
        const uint64_t dv0 = make_smem_desc(sV, 64 * 64 * 2, 1024, kSwizzle128B);
        const uint64_t dba = make_smem_desc(sBias, 128, 256, kSwizzleNone);
        const uint64_t dbb = make_smem_desc(sBias + 8192, 128, 256, kSwizzleNone);
        constexpr uint32_t i_qk = make_idesc(2, 1, 1, 0, 0, 128, 64);
        constexpr uint32_t i_qk128 = make_idesc(2, 1, 1, 0, 0, 128, 128);
        constexpr uint32_t i_bias = make_idesc(1, 0, 0, 0, 0, 128, 64);
        constexpr uint32_t i_bias128 = make_idesc(1, 0, 0, 0, 0, 128, 128);
        constexpr uint32_t i_pv = make_idesc(1, 0, 0, 0, 1, 128, D);
        auto s_col = [&](int x, int j) -> uint32_t {
            if ((MODE >= 5 && MODE <= 7) || MODE == 11) return ((2 * j + x) % 3) * 64;
            return x * 128 + (j & 1) * 64;
        };
        auto qk = [&](int x, int j, int s) {
            uint32_t ts = t + s_col(x, j);
            if (MODE == 1) ts = t + x * 128 + ((j + 1) & 1) * 64;
            const uint64_t dq = dq0 + ((x * kQBytes) >> 4);
            const uint64_t dk = dk0 + (MODE == 8 ? 0 : ((s * kKBytes) >> 4));
            if (MODE != 4 && MODE != 7) umma_f16_ss(ts, dba, dbb, i_bias, 0);
#pragma unroll
            for (int kk = 0; kk < D / 32; ++kk) {
                if (MODE == 6 || MODE == 7 || MODE == 11)
                    umma_i8_ts(ts, t + 192 + x * 32 + kk * 8, dk + kk * 2, i_qk, 1);
                else
                    umma_i8_ss(ts, dq + kk * 2, dk + kk * 2, i_qk, 1);
            }
            if (MODE != 3) umma_commit(smem_u32(&bar[x]));
        };
        auto qk128 = [&](int x, int j, int s) {  // 128 keys at once, every other step
            const uint32_t ts = t + x * 128;
            const uint64_t dq = dq0 + ((x * kQBytes) >> 4);
            const uint64_t dk = dk0 + ((s * kKBytes) >> 4);
            umma_f16_ss(ts, dba, dbb, i_bias128, 0);
#pragma unroll
            for (int kk = 0; kk < D / 32; ++kk) umma_i8_ss(ts, dq + kk * 2, dk + kk * 2, i_qk128, 1);
            umma_commit(smem_u32(&bar[x]));
        };
        auto pv = [&](int x, int j, int s) {
            const uint32_t tp = t + s_col(x, j);
            const uint32_t to = t + 256 + x * D;
            const uint64_t dv = dv0 + (MODE == 8 ? 0 : ((s * kVBytes) >> 4));
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) umma_f16_ts(to, tp + kk * 8, dv + kk * 128, i_pv, 1);
            if (MODE != 3) umma_commit(smem_u32(&bar[2 + x]));
        };
        if (kTma) {
            mbar_wait(smem_u32(&kvf[0]), 0);
            mbar_wait(smem_u32(&kvf[1]), 0);
            tc_fence_after();
        }
        long long t0 = clock64();
        for (int j = 0; j < iters; ++j) {
            const int s = j % S;
            if (kTma) {  // K/V of step j+2 (used by QK(j+2)) must have landed
                mbar_wait(smem_u32(&kvf[(j + 2) % S]), ((j + 2) / S) & 1);
                tc_fence_after();
            }
            if (MODE == 2) {
                pv(0, j, s);
                pv(1, j, s);
                qk(0, j + 2, (j + 2) % S);
                qk(1, j + 2, (j + 2) % S);
            } else if (MODE == 9) {
                pv(0, j, s);
                if ((j & 1) == 0) qk128(0, j + 2, (j + 2) % S);
                pv(1, j, s);
                if ((j & 1) == 0) qk128(1, j + 2, (j + 2) % S);
            } else if ((MODE >= 5 && MODE <= 7) || MODE == 11) {
                pv(0, j, s);
                qk(1, j + 1, (j + 1) % S);  // slot of PV_A(j) is reused by QK_B(j+1) (seq 2j -> 2j+3)
                pv(1, j, s);
                qk(0, j + 2, (j + 2) % S);  // seq 2j+1 -> 2j+4
            } else {
                pv(0, j, s);
                qk(0, j + 2, (j + 2) % S);
                pv(1, j, s);
                qk(1, j + 2, (j + 2) % S);
            }
            if (MODE != 3) umma_commit(smem_u32(kTma ? &kve[s] : &bar[4]));
        }
        umma_commit(smem_u32(&bar[5]));
        mbar_wait_spin(smem_u32(&bar[5]), 0);
        long long t1 = clock64();
        cyc[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tc_fence_after();
        tmem_dealloc<512>(t);
    }
}

template <int MODE>
void run(const char* name, long long* cyc) {
    const int iters = 4096;
    const int smem = 210 * 1024;
    cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    static uint8_t* g = nullptr;
    if (!g) {
        cudaMalloc(&g, 16u << 20);
        cudaMemset(g, 1, 16u << 20);
    }
    k<MODE><<<148, 128, smem>>>(iters, cyc, g);
    k<MODE><<<148, 128, smem>>>(iters, cyc, g);
    long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double mx = 0, mean = 0;
    for (int i = 0; i < 148; ++i) {
        mean += double(h[i]) / 148;
        mx = h[i] > mx ? double(h[i]) : mx;
    }
    printf("%-62s %7.1f cycles/step (max SM %7.1f)\n", name, mean / iters, mx / iters);
}

int main() {
    long long* cyc;
    cudaMalloc(&cyc, 148 * 8);
    run<0>("0 K2 order (PV_x(j), bias+QK_x(j+2) same buffer)", cyc);
    run<1>("1 QK into the other S buffer (no adjacent WAR)", cyc);
    run<2>("2 order PV_A PV_B QK_A QK_B", cyc);
    run<3>("3 K2 order, no commits", cyc);
    run<4>("4 K2 order, no bias MMA", cyc);
    run<5>("5 3-slot shared S ring, SS QK", cyc);
    run<6>("6 3-slot shared S ring, Q^ in TMEM (TS QK)", cyc);
    run<7>("7 as 6 without bias", cyc);
    run<8>("8 K2 order, fixed K/V stage address", cyc);
    run<9>("9 QK N=128 every other step", cyc);
    run<10>("10 K2 order + bulk-copied K/V ring (24 KB/step)", cyc);
    run<11>("11 3-slot ring, Q^ in TMEM, bulk-copied K/V ring", cyc);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
