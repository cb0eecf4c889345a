// Microbenchmark: the K2 softmax_row compute phase alone (registers only), cycles per
// 64-key row step at 1, 2 and 4 warps per SM sub-partition.
#include <cstdio>
#include "../../paper_2410_02367_b200/csrc/sab_attention.cu"
namespace sab { namespace {
__device__ __forceinline__ void consume(const uint32_t (&pk)[32]) {
    asm volatile("" ::"r"(pk[0]), "r"(pk[1]), "r"(pk[2]), "r"(pk[3]), "r"(pk[4]), "r"(pk[5]), "r"(pk[6]), "r"(pk[7]),
                 "r"(pk[8]), "r"(pk[9]), "r"(pk[10]), "r"(pk[11]), "r"(pk[12]), "r"(pk[13]), "r"(pk[14]), "r"(pk[15]),
                 "r"(pk[16]), "r"(pk[17]), "r"(pk[18]), "r"(pk[19]), "r"(pk[20]), "r"(pk[21]), "r"(pk[22]),
                 "r"(pk[23]), "r"(pk[24]), "r"(pk[25]), "r"(pk[26]), "r"(pk[27]), "r"(pk[28]), "r"(pk[29]),
                 "r"(pk[30]), "r"(pk[31]));
}
__global__ void kbench(float* out, int iters, long long* cyc, float cgv) {
    uint32_t r[64];
#pragma unroll
    for (int c = 0; c < 64; ++c) r[c] = 0x4B400000u + ((threadIdx.x * 7 + c * 13) % 2000) - 1000;
    float m = -INFINITY, l = 0.0f;
    bool rescale;
    uint32_t pk[32];
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const float alpha = softmax_row<false, false>(r, pk, cgv, 0, 0, 1 << 30, m, l, rescale, nullptr);
        consume(pk);
        r[0] += 1;
        l += alpha;
    }
    __syncthreads();
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = l + m;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
}}
int main() {
    float* out; long long* cyc;
    cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
    for (int warps : {4, 8, 16}) {
        int iters = 2000;
        sab::kbench<<<148, warps * 32>>>(out, iters, cyc, 0.01f);
        sab::kbench<<<148, warps * 32>>>(out, iters, cyc, 0.01f);
        long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("warps/SMSP %d: %.0f cycles per row-step per SMSP (%.0f per warp-step); MUFU floor %d\n", warps / 4,
               double(h) / iters, double(h) / iters, (warps / 4) * 56 * 8);
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
