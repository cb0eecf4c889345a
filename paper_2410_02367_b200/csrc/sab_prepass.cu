// sab_prepass.cu -- K1, the fused SageAttn-B pre-pass (HBM-bound).
//
// Replaces, bit-exactly, the reference pre-processing of attention.hpp:336-360:
//   smooth_k            quant.hpp:220-242 (pairwise_column_sum, quant.hpp:203-213)
//   fold_scale_into_q   quant.hpp:246-252
//   quantize(per_block(128 | 64), Int8)   quant.hpp:95-173
//   V -> binary16 grid  attention.hpp:371-375 (fp32 inputs only; F9: hardware
//                       cvt.rn.f16.f32 == round_to_half for finite floats)
//
// Two launches per call:
//   fp16 inputs, per-block scales (the SAGEAttn-B bench and fp16 drop-in path):
//     k1_mean_and_q   grid (n_partials + ceil(N/128), units): mean-tree partials of
//                     K (the last CTA of each unit, found by a per-unit counter,
//                     sums the top of the tree -> mean_k) next to Q fold+quantize
//                     chunks, which do not need mean_k;
//     k1_k_fast       grid (ceil(N/128), units): smooth + quantize K.
//   otherwise (fp32 inputs, per-token scales, smoothing off):
//     k1_mean_partials  grid (n_partials, units): the same mean tree;
//   k1_quantize       grid (ceil(N/128), units): reads mean_k, then quantizes
//                     one 128-token Q group and the two 64-token K groups of
//                     that chunk.
//
// Tree equivalence: with depth = the smallest k such that
// floor(N/2^k) < 9, every node at that depth holds 4..9 tokens and every node
// above it splits in two, so the reference recursion is a perfect binary tree
// over 2^depth leaf nodes.  A leaf of <= 8 tokens is a sequential sum from
// 0.0f; a 9-token leaf is (4 sequential) + (5 sequential).
//
// No fast-math anywhere: explicit __fmul_rn / __fsub_rn / __fdiv_rn /
// __float2int_rn reproduce the reference's binary32 operations one for one.
#include <cuda_fp16.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <type_traits>

#include "sab_internal.h"
#include "sab_ptx.cuh"

namespace sab {

int tree_depth(int n) {
    int depth = 0;
    while ((n >> depth) >= 9) ++depth;
    return depth;
}

// Leaves of the mean tree summed per mean-partial CTA: any power of two keeps the tree
// (the CTA sums an aligned perfect subtree, mean_top the perfect tree above).  32 by default;
// SAB_K1_NODES (4, 8, 16, 32 or 64) overrides it for tuning.
int nodes_per_cta(int depth) {
    static const int cap = [] {
        const char* e = std::getenv("SAB_K1_NODES");
        const int v = e ? std::atoi(e) : 32;
        return (v == 4 || v == 8 || v == 16 || v == 64) ? v : 32;
    }();
    const int nodes = 1 << depth;
    return nodes < cap ? nodes : cap;
}

namespace {

constexpr int kThreads = 256;

template <typename T>
__device__ __forceinline__ void load8(const T* src, float (&x)[8]);

template <>
__device__ __forceinline__ void load8<__half>(const __half* src, float (&x)[8]) {
    const uint4 u = *reinterpret_cast<const uint4*>(src);
    const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 f = __half22float2(h[i]);
        x[2 * i] = f.x;
        x[2 * i + 1] = f.y;
    }
}

template <>
__device__ __forceinline__ void load8<float>(const float* src, float (&x)[8]) {
    const float4 a = *reinterpret_cast<const float4*>(src);
    const float4 b = *(reinterpret_cast<const float4*>(src) + 1);
    x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
    x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
}

// RoPE of the 8 channels [col, col + 8) of token t (sab_prepass_rope), binary32 with
// every product and sum rounded (no contraction):
//   interleaved (pairs 2i, 2i+1):  x0' = x0 c - x1 s,   x1' = x0 s + x1 c
//   half split  (pairs i, i+d/2):  x_i' = x_i c - x_{i+d/2} s,   x_{i+d/2}' = x_{i+d/2} c + x_i s
// with c = cos[t][i], s = sin[t][i]; `pr` holds channels col ^ (d/2) (half split only).
template <int D>
__device__ __forceinline__ void rope8(const PrepassParams& p, int t, int col, float (&x)[8], const float (&pr)[8]) {
    const float* cs = p.rope_cos + static_cast<size_t>(t) * (D / 2);
    const float* sn = p.rope_sin + static_cast<size_t>(t) * (D / 2);
    if (p.rope == SAB_ROPE_INTERLEAVED) {
        const float4 c = __ldg(reinterpret_cast<const float4*>(cs + col / 2));
        const float4 s = __ldg(reinterpret_cast<const float4*>(sn + col / 2));
        const float cc[4] = {c.x, c.y, c.z, c.w}, ss[4] = {s.x, s.y, s.z, s.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float x0 = x[2 * e], x1 = x[2 * e + 1];
            x[2 * e] = __fsub_rn(__fmul_rn(x0, cc[e]), __fmul_rn(x1, ss[e]));
            x[2 * e + 1] = __fadd_rn(__fmul_rn(x0, ss[e]), __fmul_rn(x1, cc[e]));
        }
    } else {
        const bool lo = col < D / 2;
        const int i0 = lo ? col : col - D / 2;
        float cc[8], ss[8];
        *reinterpret_cast<float4*>(cc) = __ldg(reinterpret_cast<const float4*>(cs + i0));
        *reinterpret_cast<float4*>(cc + 4) = __ldg(reinterpret_cast<const float4*>(cs + i0) + 1);
        *reinterpret_cast<float4*>(ss) = __ldg(reinterpret_cast<const float4*>(sn + i0));
        *reinterpret_cast<float4*>(ss + 4) = __ldg(reinterpret_cast<const float4*>(sn + i0) + 1);
#pragma unroll
        for (int e = 0; e < 8; ++e)
            x[e] = lo ? __fsub_rn(__fmul_rn(x[e], cc[e]), __fmul_rn(pr[e], ss[e]))
                      : __fadd_rn(__fmul_rn(x[e], cc[e]), __fmul_rn(pr[e], ss[e]));
    }
}

// load8 of row `row` (token t), rotated when RoPE is on.
template <typename T, int D>
__device__ __forceinline__ void load8_rope(const PrepassParams& p, const T* rowp, int t, int col, float (&x)[8]) {
    load8<T>(rowp + col, x);
    if (p.rope) {
        float pr[8];
        if (p.rope == SAB_ROPE_HALF) load8<T>(rowp + (col ^ (D / 2)), pr);
        rope8<D>(p, t, col, x, pr);
    }
}

// Raw 8-element vector as loaded (fp16: 16 B, fp32: 32 B), kept in registers
// in its input format so K1 keeps Q and K of a 128-token chunk on chip.
template <typename T>
struct Raw8;
template <>
struct Raw8<__half> {
    uint4 u;
    __device__ __forceinline__ void load(const __half* src) { u = __ldg(reinterpret_cast<const uint4*>(src)); }
    __device__ __forceinline__ void zero() { u = make_uint4(0, 0, 0, 0); }
    __device__ __forceinline__ void get(float (&x)[8]) const {
        const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 f = __half22float2(h[i]);
            x[2 * i] = f.x;
            x[2 * i + 1] = f.y;
        }
    }
};
template <>
struct Raw8<float> {
    float4 a, b;
    __device__ __forceinline__ void load(const float* src) {
        a = __ldg(reinterpret_cast<const float4*>(src));
        b = __ldg(reinterpret_cast<const float4*>(src) + 1);
    }
    __device__ __forceinline__ void zero() { a = b = make_float4(0.f, 0.f, 0.f, 0.f); }
    __device__ __forceinline__ void get(float (&x)[8]) const {
        x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
        x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
    }
};

__device__ __forceinline__ bool all_finite8(const float (&x)[8]) {
    bool ok = true;
#pragma unroll
    for (int i = 0; i < 8; ++i) ok &= isfinite(x[i]);
    return ok;
}

// Token range [a, b) of leaf node `node` of the pairwise tree over [0, n):
// descend `depth` levels, splitting [a, b) at a + (b - a) / 2 (quant.hpp:210).
__device__ __forceinline__ void leaf_range(int node, int depth, int n, int& a, int& b) {
    a = 0;
    b = n;
    for (int lv = depth - 1; lv >= 0; --lv) {
        const int mid = a + (b - a) / 2;
        if ((node >> lv) & 1) a = mid; else b = mid;
    }
}

// Sequential binary32 sum from 0.0f of rows [t0, t1), t1 - t0 <= 9
// (quant.hpp:205-208).  All row loads are issued before the dependent adds.
template <typename T, int D>
__device__ __forceinline__ void seq_sum(const T* base, int t0, int t1, int col, float (&s)[8]) {
    Raw8<T> v[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) {
        if (t0 + i < t1) v[i].load(base + static_cast<size_t>(t0 + i) * D + col);
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) s[e] = 0.0f;
#pragma unroll
    for (int i = 0; i < 9; ++i) {
        if (t0 + i < t1) {
            float x[8];
            v[i].get(x);
#pragma unroll
            for (int e = 0; e < 8; ++e) s[e] = __fadd_rn(s[e], x[e]);
        }
    }
}

// Top of the pairwise tree: combines the n_partials (power of two) CTA partial
// sums of one unit as a perfect binary tree (binary-counter evaluation, left +
// right), then mean = sum * (1.0f / N)  (quant.hpp:228, 235).  Channel c; the
// partials of the other CTAs are read through L2 (__ldcg).
// seq_sum of rotated rows (RoPE on): one row at a time.
template <typename T, int D>
__device__ __forceinline__ void seq_sum_rope(const PrepassParams& p, const T* base, int t0, int t1, int col,
                                             float (&s)[8]) {
#pragma unroll
    for (int e = 0; e < 8; ++e) s[e] = 0.0f;
    for (int t = t0; t < t1; ++t) {
        float x[8];
        load8_rope<T, D>(p, base + static_cast<size_t>(t) * D, t, col, x);
#pragma unroll
        for (int e = 0; e < 8; ++e) s[e] = __fadd_rn(s[e], x[e]);
    }
}

template <int D>
__device__ __forceinline__ void mean_top(const PrepassParams& p, int unit, int c) {
    const float* part = p.partials + static_cast<size_t>(unit) * p.n_partials * D + c;
    float stk[24];
    int top = 0;
    for (int i0 = 0; i0 < p.n_partials; i0 += 8) {  // n_partials is 1, 2, 4 or a multiple of 8
        float xs[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) xs[u] = (i0 + u < p.n_partials) ? __ldcg(part + static_cast<size_t>(i0 + u) * D) : 0.0f;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = i0 + u;
            if (i < p.n_partials) {
                float x = xs[u];
                for (int t = i; t & 1; t >>= 1) x = __fadd_rn(stk[--top], x);
                stk[top++] = x;
            }
        }
    }
    p.mean[static_cast<size_t>(unit) * D + c] = __fmul_rn(stk[0], p.inv_n);
}

// k1_fused's per-unit "mean(K) written" flag: release by the CTA that wrote mean_k,
// acquire by the K chunks of the unit.
__device__ __forceinline__ void flag_release(int* f) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(f), "r"(1) : "memory");
}
__device__ __forceinline__ void flag_wait(const int* f) {
    for (;;) {
        int v;
        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
        if (v) return;
        __nanosleep(128);
    }
}

template <typename T, int D, int G, bool FLAG = false>
__device__ __forceinline__ void mean_partial(const PrepassParams& p, int unit, int chunk) {
    constexpr int CV = D / 8;           // 8-channel vectors per row
    constexpr int NG = kThreads / CV;   // node groups per CTA
    __shared__ float red[NG][D];

    const int cv = threadIdx.x % CV;
    const int grp = threadIdx.x / CV;
    const int active = p.nodes_per_cta / G;  // groups holding G nodes each
    const T* base = static_cast<const T*>(p.k) + static_cast<size_t>(unit) * p.n * D;

    if (grp < active) {
        float ns[G][8];
        const int node0 = chunk * p.nodes_per_cta + grp * G;
#pragma unroll
        for (int g = 0; g < G; ++g) {
            int a, b;
            leaf_range(node0 + g, p.depth, p.n, a, b);
            if (b - a <= 8) {
                if (p.rope) seq_sum_rope<T, D>(p, base, a, b, cv * 8, ns[g]);
                else seq_sum<T, D>(base, a, b, cv * 8, ns[g]);
            } else {  // 9-token leaf: (4) + (5)
                float lo[8], hi[8];
                const int mid = a + (b - a) / 2;
                if (p.rope) {
                    seq_sum_rope<T, D>(p, base, a, mid, cv * 8, lo);
                    seq_sum_rope<T, D>(p, base, mid, b, cv * 8, hi);
                } else {
                    seq_sum<T, D>(base, a, mid, cv * 8, lo);
                    seq_sum<T, D>(base, mid, b, cv * 8, hi);
                }
#pragma unroll
                for (int i = 0; i < 8; ++i) ns[g][i] = __fadd_rn(lo[i], hi[i]);
            }
        }
        // Perfect binary tree over the G nodes of this group (left + right).
#pragma unroll
        for (int step = 1; step < G; step *= 2)
#pragma unroll
            for (int g = 0; g < G; g += 2 * step)
#pragma unroll
                for (int i = 0; i < 8; ++i) ns[g][i] = __fadd_rn(ns[g][i], ns[g + step][i]);
#pragma unroll
        for (int i = 0; i < 8; ++i) red[grp][cv * 8 + i] = ns[0][i];
    }
    __syncthreads();
    // Perfect binary tree over the active groups.
    for (int stride = 1; stride < active; stride *= 2) {
        if (grp < active && (grp % (2 * stride)) == 0) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
                red[grp][cv * 8 + i] = __fadd_rn(red[grp][cv * 8 + i], red[grp + stride][cv * 8 + i]);
        }
        __syncthreads();
    }
    if (grp == 0) {
        float* dst = p.partials + (static_cast<size_t>(unit) * p.n_partials + chunk) * D + cv * 8;
#pragma unroll
        for (int i = 0; i < 8; ++i) dst[i] = red[0][cv * 8 + i];
        __threadfence();  // the writers publish the partial before the CTA's counter increment
    }
    // The last CTA of the unit to finish sums the top of the tree (no second launch).
    __shared__ int s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        s_last = atomicAdd(p.counters + unit, 1) == p.n_partials - 1;
        if (s_last) p.counters[unit] = 0;  // ready for the next call
    }
    __syncthreads();
    if (s_last) {
        __threadfence();
        if (threadIdx.x < D) mean_top<D>(p, unit, threadIdx.x);
        if constexpr (FLAG) {  // s_last is CTA-uniform
            __threadfence();
            __syncthreads();
            if (threadIdx.x == 0) flag_release(p.ready + unit);
        }
    }
}

#ifndef SAB_K1_PART_MINB
#define SAB_K1_PART_MINB 1  // CTAs per SM bound of k1_mean_partials (tuning)
#endif
template <typename T, int D, int G>
__global__ void __launch_bounds__(kThreads, SAB_K1_PART_MINB) k1_mean_partials(PrepassParams p) {
    griddep_launch_dependents();  // k1_quantize's input loads may start behind this grid
    mean_partial<T, D, G>(p, blockIdx.y, blockIdx.x);
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// quant.hpp:141-152: delta = amax / 127, inv = 1 / delta; zero group -> (1, 0).
__device__ __forceinline__ void int8_scale(float amax, float& delta, float& inv) {
    if (amax == 0.0f) {
        delta = 1.0f;
        inv = 0.0f;
    } else {
        delta = __fdiv_rn(amax, 127.0f);
        inv = __fdiv_rn(1.0f, delta);
    }
}

// quant.hpp:95-101 on a pair: clamp(nearbyint(x * inv), -127, 127).  The product
// is rounded first (mul.rn, exactly the reference's `x * inv_scale`), clamped in
// float (identical to clamping the integer for |v| <= 127.5, and maps +-inf like
// the reference), and rounded to nearest-even by adding 2^23 + 2^22: the low
// byte of the biased float's bits is then the two's-complement INT8 code.
template <bool CLAMP>
__device__ __forceinline__ uint2 code_pair(float x0, float x1, float inv) {
    float t0 = __fmul_rn(x0, inv), t1 = __fmul_rn(x1, inv);
    if (CLAMP) {  // only reachable when 1/delta overflowed (amax < ~127 * 2^-128)
        t0 = fminf(fmaxf(t0, -127.0f), 127.0f);
        t1 = fminf(fmaxf(t1, -127.0f), 127.0f);
    }
    return make_uint2(__float_as_uint(__fadd_rn(t0, 12582912.0f)), __float_as_uint(__fadd_rn(t1, 12582912.0f)));
}

// Eight codes packed little-endian into two words (low bytes of the biased floats).
// Without CLAMP the reference's clamp is a no-op: |x| <= amax gives
// |x * inv| <= 127 * (1 + 3 ulp) < 127.5 whenever inv = 1/(amax/127) is finite.
template <bool CLAMP>
__device__ __forceinline__ uint2 codes8_fast(const float (&x)[8], float inv) {
    const uint2 a = code_pair<CLAMP>(x[0], x[1], inv), b = code_pair<CLAMP>(x[2], x[3], inv);
    const uint2 c = code_pair<CLAMP>(x[4], x[5], inv), d = code_pair<CLAMP>(x[6], x[7], inv);
    const uint32_t lo = __byte_perm(__byte_perm(a.x, a.y, 0x0040), __byte_perm(b.x, b.y, 0x0040), 0x5410);
    const uint32_t hi = __byte_perm(__byte_perm(c.x, c.y, 0x0040), __byte_perm(d.x, d.y, 0x0040), 0x5410);
    return make_uint2(lo, hi);
}

// ---- packed helpers for the fp16 fast path (two binary32 lanes per instruction)
struct f2 {
    float x, y;
};
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
    f2 d;
    asm("{\n\t.reg .b64 a, b, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
        "mul.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
    f2 d;
    asm("{\n\t.reg .b64 a, b, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
        "add.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}
__device__ __forceinline__ f2 h2f(uint32_t w) {
    const float2 v = __half22float2(*reinterpret_cast<const __half2*>(&w));
    return f2{v.x, v.y};
}
// Codes of eight already-scaled values t = x * inv (binary32, rounded): clamp to
// +-127 (CLAMP only), round to nearest-even by adding 2^23 + 2^22, and pack the
// low bytes of the biased floats little-endian into two words.
template <bool CLAMP>
__device__ __forceinline__ uint2 pack_codes8(const f2 (&t)[4]) {
    uint32_t b[8];
#pragma unroll
    for (int w = 0; w < 4; ++w) {
        f2 v = t[w];
        if (CLAMP) {
            v.x = fminf(fmaxf(v.x, -127.0f), 127.0f);
            v.y = fminf(fmaxf(v.y, -127.0f), 127.0f);
        }
        v = add2(v, f2{12582912.0f, 12582912.0f});
        b[2 * w] = __float_as_uint(v.x);
        b[2 * w + 1] = __float_as_uint(v.y);
    }
    const uint32_t lo = __byte_perm(__byte_perm(b[0], b[1], 0x0040), __byte_perm(b[2], b[3], 0x0040), 0x5410);
    const uint32_t hi = __byte_perm(__byte_perm(b[4], b[5], 0x0040), __byte_perm(b[6], b[7], 0x0040), 0x5410);
    return make_uint2(lo, hi);
}

constexpr int kQThreads = 256;

// One CTA quantizes one 128-token chunk of one unit: the Q and K rows of the
// chunk (contiguous in HBM) arrive by two bulk copies into shared memory, so
// the CTA needs few registers and three CTAs share an SM (one's copies overlap
// another's arithmetic).
template <typename T, int D>
__global__ void __launch_bounds__(kQThreads) k1_quantize(PrepassParams p) {
    constexpr int CV = D / 8;
    constexpr int VPT = kBlockQ * CV / kQThreads;  // 8-element vectors per thread per tensor
    constexpr int kChunkBytes = kBlockQ * D * static_cast<int>(sizeof(T));
    extern __shared__ __align__(128) uint8_t smem[];
    T* sq = reinterpret_cast<T*>(smem);
    T* sk = reinterpret_cast<T*>(smem + kChunkBytes);
    __shared__ uint64_t bar;
    __shared__ float s_mean[D];
    __shared__ float s_red[kQThreads / 32][3];
    __shared__ float s_inv[3];

    const int unit = blockIdx.y;
    const int chunk = blockIdx.x;
    const int tid = threadIdx.x;
    const int r0 = chunk * kBlockQ;
    const int rows = min(kBlockQ, p.n - r0);
    const size_t ubase = static_cast<size_t>(unit) * p.n * D;
    const uint32_t bytes = static_cast<uint32_t>(rows) * D * sizeof(T);

    if (tid == 0) {
        mbar_init(smem_u32(&bar), 1);
        fence_barrier_init();
    }
    __syncthreads();
    if (tid == 0) {
        mbar_arrive_expect_tx(smem_u32(&bar), 2 * bytes);
        bulk_load(smem_u32(sq), static_cast<const T*>(p.q) + ubase + static_cast<size_t>(r0) * D, bytes, smem_u32(&bar));
        bulk_load(smem_u32(sk), static_cast<const T*>(p.k) + ubase + static_cast<size_t>(r0) * D, bytes, smem_u32(&bar));
    }
    // mean_k (computed by k1_mean_partials; zero when smoothing is off).  The chunk's Q and K
    // loads (inputs) are in flight before the wait for the producer grid (PDL launch).
    griddep_wait();
    griddep_launch_dependents();  // K2 may be scheduled behind this grid's last wave
    if (tid < D) s_mean[tid] = p.smooth ? p.mean[static_cast<size_t>(unit) * D + tid] : 0.0f;
    __syncthreads();
    mbar_wait(smem_u32(&bar), 0);

    if (p.per_token) {
        // SAGEAttn-T: Granularity::per_token (quant.hpp:37-63) -- one scale per row of
        // folded Q and of smoothed K.  A row's 8-channel vectors sit on CV consecutive
        // lanes, which reduce its two maxima by shuffles; then each lane writes its codes.
        const int ngq = (p.n + kBlockKV - 1) / kBlockKV * kBlockKV;  // scale rows [units][npad], npad = 64*ceil(n/64)
        bool finite = true;
#pragma unroll 1
        for (int i = 0; i < VPT; ++i) {
            const int v = tid + i * kQThreads;
            const int row = v / CV, col = (v % CV) * 8;
            const bool valid = row < rows;
            float q[8], k[8];
            float aq = 0.0f, ak = 0.0f;
            if (valid) {
                load8_rope<T, D>(p, sq + row * D, r0 + row, col, q);
                load8_rope<T, D>(p, sk + row * D, r0 + row, col, k);
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    finite &= isfinite(q[e]) && isfinite(k[e]);
                    q[e] = __fmul_rn(q[e], p.fold);
                    k[e] = __fsub_rn(k[e], s_mean[col + e]);
                    aq = fmaxf(aq, fabsf(q[e]));
                    ak = fmaxf(ak, fabsf(k[e]));
                }
            }
#pragma unroll
            for (int o = CV / 2; o > 0; o >>= 1) {
                aq = fmaxf(aq, __shfl_xor_sync(0xffffffffu, aq, o));
                ak = fmaxf(ak, __shfl_xor_sync(0xffffffffu, ak, o));
            }
            if (valid) {
                float dq, iq, dk, ik;
                int8_scale(aq, dq, iq);
                int8_scale(ak, dk, ik);
                const size_t off = ubase + static_cast<size_t>(r0 + row) * D + col;
                *reinterpret_cast<uint2*>(p.qcodes + off) = isinf(iq) ? codes8_fast<true>(q, iq) : codes8_fast<false>(q, iq);
                *reinterpret_cast<uint2*>(p.kcodes + off) = isinf(ik) ? codes8_fast<true>(k, ik) : codes8_fast<false>(k, ik);
                if (col == 0) {
                    p.qscales[static_cast<size_t>(unit) * ngq + r0 + row] = dq;
                    p.kscales[static_cast<size_t>(unit) * ngq + r0 + row] = dk;
                }
            }
        }
        if (!finite) atomicOr(p.status, kStatusNonFinite);
        if (p.v16 || p.check_v) {
            bool vfin = true;
            for (int v = tid; v < rows * CV; v += kQThreads) {
                const int row = v / CV, c8 = (v % CV) * 8;
                const size_t off = ubase + static_cast<size_t>(r0 + row) * D + c8;
                float x[8];
                load8<T>(static_cast<const T*>(p.v) + off, x);
                vfin &= all_finite8(x);
                if (p.v16) {
                    uint4 h;
                    h.x = pack_half2(x[0], x[1]);
                    h.y = pack_half2(x[2], x[3]);
                    h.z = pack_half2(x[4], x[5]);
                    h.w = pack_half2(x[6], x[7]);
                    *reinterpret_cast<uint4*>(p.v16 + off) = h;
                }
            }
            if (!vfin) atomicOr(p.status, kStatusNonFinite);
        }
        return;
    }

    if constexpr (std::is_same<T, __half>::value) if (!p.rope) {
        // fp16 fast path.  Every thread keeps one 8-channel column block (CV divides
        // the thread count), so its eight K means live in registers.
        const int col = (tid % CV) * 8;
        f2 mc[4];
#pragma unroll
        for (int w = 0; w < 4; ++w) mc[w] = f2{-s_mean[col + 2 * w], -s_mean[col + 2 * w + 1]};
        // Pass 1.  Q: the group max of |fl(q * fold)| is fl(max|q| * fold) (rounding
        // is monotone and sign-symmetric), and max|q| is an unsigned 16-bit max over
        // the fp16 bit patterns with the sign cleared -- which also flags inf / NaN
        // (>= 0x7C00).  K: the binary32 smooth fl(k - mean) and its group maxima.
        uint32_t qbits = 0, kbits = 0;
        float amax_k0 = 0.0f, amax_k1 = 0.0f;
#pragma unroll
        for (int i = 0; i < VPT; ++i) {
            const int row = (tid + i * kQThreads) / CV;
            if (row < rows) {
                const uint4 uq = *reinterpret_cast<const uint4*>(sq + row * D + col);
                const uint4 uk = *reinterpret_cast<const uint4*>(sk + row * D + col);
                const uint32_t wq[4] = {uq.x, uq.y, uq.z, uq.w}, wk[4] = {uk.x, uk.y, uk.z, uk.w};
                float a = 0.0f;
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                    qbits = __vmaxu2(qbits, wq[w] & 0x7FFF7FFFu);
                    kbits = __vmaxu2(kbits, wk[w] & 0x7FFF7FFFu);
                    const f2 d = add2(h2f(wk[w]), mc[w]);
                    a = fmaxf(a, fmaxf(fabsf(d.x), fabsf(d.y)));
                }
                if (i < VPT / 2) amax_k0 = fmaxf(amax_k0, a);
                else amax_k1 = fmaxf(amax_k1, a);
            }
        }
        const uint32_t qb = max(qbits & 0xFFFFu, qbits >> 16), kb = max(kbits & 0xFFFFu, kbits >> 16);
        if (qb >= 0x7C00u || kb >= 0x7C00u) atomicOr(p.status, kStatusNonFinite);
        const __half qh = __ushort_as_half(static_cast<unsigned short>(qb));
        float amax_q = __fmul_rn(__half2float(qh), p.fold);
        amax_q = warp_max(amax_q);
        amax_k0 = warp_max(amax_k0);
        amax_k1 = warp_max(amax_k1);
        if ((tid & 31) == 0) {
            s_red[tid >> 5][0] = amax_q;
            s_red[tid >> 5][1] = amax_k0;
            s_red[tid >> 5][2] = amax_k1;
        }
        __syncthreads();
        if (tid < 3) {
            float m = 0.0f;
            for (int w = 0; w < kQThreads / 32; ++w) m = fmaxf(m, s_red[w][tid]);
            float delta, inv;
            int8_scale(m, delta, inv);
            s_inv[tid] = inv;
            const int ngk = (p.n + kBlockKV - 1) / kBlockKV;
            if (tid == 0) {
                p.qscales[static_cast<size_t>(unit) * ((p.n + kBlockQ - 1) / kBlockQ) + chunk] = delta;
            } else {
                const int g = 2 * chunk + (tid - 1);
                if (g < ngk) p.kscales[static_cast<size_t>(unit) * ngk + g] = delta;
            }
        }
        __syncthreads();
        // Pass 2: codes, recomputing the binary32 fold / smooth from shared memory.
        const float inv_q = s_inv[0], inv_k0 = s_inv[1], inv_k1 = s_inv[2];
        const bool clamp = isinf(inv_q) || isinf(inv_k0) || isinf(inv_k1);  // 1/delta overflowed
        const f2 fold2{p.fold, p.fold}, iq2{inv_q, inv_q};
#pragma unroll
        for (int i = 0; i < VPT; ++i) {
            const int row = (tid + i * kQThreads) / CV;
            if (row < rows) {
                const uint4 uq = *reinterpret_cast<const uint4*>(sq + row * D + col);
                const uint4 uk = *reinterpret_cast<const uint4*>(sk + row * D + col);
                const uint32_t wq[4] = {uq.x, uq.y, uq.z, uq.w}, wk[4] = {uk.x, uk.y, uk.z, uk.w};
                const float ik = i < VPT / 2 ? inv_k0 : inv_k1;
                const f2 ik2{ik, ik};
                f2 tq[4], tk[4];
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                    tq[w] = mul2(mul2(h2f(wq[w]), fold2), iq2);
                    tk[w] = mul2(add2(h2f(wk[w]), mc[w]), ik2);
                }
                const size_t off = ubase + static_cast<size_t>(r0 + row) * D + col;
                *reinterpret_cast<uint2*>(p.qcodes + off) = clamp ? pack_codes8<true>(tq) : pack_codes8<false>(tq);
                *reinterpret_cast<uint2*>(p.kcodes + off) = clamp ? pack_codes8<true>(tk) : pack_codes8<false>(tk);
            }
        }
        if (p.check_v) {
            bool vfin = true;
            for (int v = tid; v < rows * CV; v += kQThreads) {
                const int row = v / CV, c8 = (v % CV) * 8;
                float x[8];
                load8<T>(static_cast<const T*>(p.v) + ubase + static_cast<size_t>(r0 + row) * D + c8, x);
                vfin &= all_finite8(x);
            }
            if (!vfin) atomicOr(p.status, kStatusNonFinite);
        }
        return;
    }

    // Pass 1: fold (Q) / smooth (K) in binary32 and the group maxima.
    float amax_q = 0.0f, amax_k0 = 0.0f, amax_k1 = 0.0f, nan_probe = 0.0f;
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
        const int v = tid + i * kQThreads;
        const int row = v / CV, col = (v % CV) * 8;
        if (row < rows) {
            float q[8], k[8];
            load8_rope<T, D>(p, sq + row * D, r0 + row, col, q);
            load8_rope<T, D>(p, sk + row * D, r0 + row, col, k);
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                nan_probe = fmaf(q[e], 0.0f, nan_probe);  // NaN iff some input is inf or NaN
                nan_probe = fmaf(k[e], 0.0f, nan_probe);
                amax_q = fmaxf(amax_q, fabsf(__fmul_rn(q[e], p.fold)));
                const float ks = fabsf(__fsub_rn(k[e], s_mean[col + e]));
                if (i < VPT / 2) amax_k0 = fmaxf(amax_k0, ks);
                else amax_k1 = fmaxf(amax_k1, ks);
            }
        }
    }
    amax_q = warp_max(amax_q);
    amax_k0 = warp_max(amax_k0);
    amax_k1 = warp_max(amax_k1);
    if ((tid & 31) == 0) {
        s_red[tid >> 5][0] = amax_q;
        s_red[tid >> 5][1] = amax_k0;
        s_red[tid >> 5][2] = amax_k1;
    }
    if (nan_probe != nan_probe) atomicOr(p.status, kStatusNonFinite);
    __syncthreads();
    if (tid < 3) {
        float m = 0.0f;
        for (int w = 0; w < kQThreads / 32; ++w) m = fmaxf(m, s_red[w][tid]);
        float delta, inv;
        int8_scale(m, delta, inv);
        s_inv[tid] = inv;
        const int ngk = (p.n + kBlockKV - 1) / kBlockKV;
        if (tid == 0) {
            p.qscales[static_cast<size_t>(unit) * ((p.n + kBlockQ - 1) / kBlockQ) + chunk] = delta;
        } else {
            const int g = 2 * chunk + (tid - 1);
            if (g < ngk) p.kscales[static_cast<size_t>(unit) * ngk + g] = delta;
        }
    }
    __syncthreads();

    // Pass 2: codes (the binary32 fold / smooth is recomputed from shared memory).
    const float inv_q = s_inv[0], inv_k0 = s_inv[1], inv_k1 = s_inv[2];
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
        const int v = tid + i * kQThreads;
        const int row = v / CV, col = (v % CV) * 8;
        if (row < rows) {
            float q[8], k[8];
            load8_rope<T, D>(p, sq + row * D, r0 + row, col, q);
            load8_rope<T, D>(p, sk + row * D, r0 + row, col, k);
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                q[e] = __fmul_rn(q[e], p.fold);
                k[e] = __fsub_rn(k[e], s_mean[col + e]);
            }
            const size_t off = ubase + static_cast<size_t>(r0 + row) * D + col;
            const float ik = i < VPT / 2 ? inv_k0 : inv_k1;
            *reinterpret_cast<uint2*>(p.qcodes + off) =
                isinf(inv_q) ? codes8_fast<true>(q, inv_q) : codes8_fast<false>(q, inv_q);
            *reinterpret_cast<uint2*>(p.kcodes + off) = isinf(ik) ? codes8_fast<true>(k, ik) : codes8_fast<false>(k, ik);
        }
    }

    // V: fp32 inputs -> fp16 grid (with the finiteness check); fp16 inputs
    // are only scanned when asked (validate_input, attention.hpp:101).
    if (p.v16 || p.check_v) {
        bool vfin = true;
        for (int v = tid; v < rows * CV; v += kQThreads) {
            const int row = v / CV, col = (v % CV) * 8;
            const size_t off = ubase + static_cast<size_t>(r0 + row) * D + col;
            float x[8];
            load8<T>(static_cast<const T*>(p.v) + off, x);
            vfin &= all_finite8(x);
            if (p.v16) {
                uint4 h;
                h.x = pack_half2(x[0], x[1]);
                h.y = pack_half2(x[2], x[3]);
                h.z = pack_half2(x[4], x[5]);
                h.w = pack_half2(x[6], x[7]);
                *reinterpret_cast<uint4*>(p.v16 + off) = h;
            }
        }
        if (!vfin) atomicOr(p.status, kStatusNonFinite);
    }
}

// ---- fp16, per-block fast path in two launches (SAGEAttn-B bench / drop-in fp16 path):
//   k1_mean_and_q  grid (n_partials + ceil(N/128), units): CTAs [0, n_partials) are the
//                  mean-tree partials of K (last CTA sums the top), the others fold and
//                  quantize one 128-token Q chunk -- Q does not need mean(K), so K's
//                  reduction and Q's quantization share one pass over HBM;
//   k1_k_fast      grid (ceil(N/128), units): smooth + quantize the two 64-token K groups
//                  of a chunk once mean(K) is known (K is re-read, mostly from L2).
template <int D>
__device__ __forceinline__ void q_chunk_fast(const PrepassParams& p, int unit, int chunk, uint8_t* smem) {
    constexpr int CV = D / 8;
    constexpr int VPT = kBlockQ * CV / kQThreads;
    const __half* sq = reinterpret_cast<const __half*>(smem);
    __shared__ uint64_t bar;
    __shared__ float s_red[kQThreads / 32];
    __shared__ float s_inv;
    const int tid = threadIdx.x;
    const int r0 = chunk * kBlockQ;
    const int rows = min(kBlockQ, p.n - r0);
    const size_t ubase = static_cast<size_t>(unit) * p.n * D;
    const uint32_t bytes = static_cast<uint32_t>(rows) * D * 2;
    if (tid == 0) {
        mbar_init(smem_u32(&bar), 1);
        fence_barrier_init();
        mbar_arrive_expect_tx(smem_u32(&bar), bytes);
        bulk_load(smem_u32(smem), static_cast<const __half*>(p.q) + ubase + static_cast<size_t>(r0) * D, bytes,
                  smem_u32(&bar));
    }
    __syncthreads();
    mbar_wait(smem_u32(&bar), 0);
    const int col = (tid % CV) * 8;
    // max|fl(q * fold)| = fl(max|q| * fold); max|q| as a 16-bit max over sign-cleared bits,
    // which also flags inf / NaN (>= 0x7C00).
    uint32_t qbits = 0;
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
        const int row = (tid + i * kQThreads) / CV;
        if (row < rows) {
            const uint4 u = *reinterpret_cast<const uint4*>(sq + row * D + col);
            qbits = __vmaxu2(__vmaxu2(qbits, u.x & 0x7FFF7FFFu), u.y & 0x7FFF7FFFu);
            qbits = __vmaxu2(__vmaxu2(qbits, u.z & 0x7FFF7FFFu), u.w & 0x7FFF7FFFu);
        }
    }
    const uint32_t qb = max(qbits & 0xFFFFu, qbits >> 16);
    if (qb >= 0x7C00u) atomicOr(p.status, kStatusNonFinite);
    float amax = warp_max(__fmul_rn(__half2float(__ushort_as_half(static_cast<unsigned short>(qb))), p.fold));
    if ((tid & 31) == 0) s_red[tid >> 5] = amax;
    __syncthreads();
    if (tid == 0) {
        float m = 0.0f;
        for (int w = 0; w < kQThreads / 32; ++w) m = fmaxf(m, s_red[w]);
        float delta, inv;
        int8_scale(m, delta, inv);
        s_inv = inv;
        p.qscales[static_cast<size_t>(unit) * ((p.n + kBlockQ - 1) / kBlockQ) + chunk] = delta;
    }
    __syncthreads();
    const float iq = s_inv;
    const bool clamp = isinf(iq);
    const f2 fold2{p.fold, p.fold}, iq2{iq, iq};
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
        const int row = (tid + i * kQThreads) / CV;
        if (row < rows) {
            const uint4 u = *reinterpret_cast<const uint4*>(sq + row * D + col);
            const uint32_t w[4] = {u.x, u.y, u.z, u.w};
            f2 t[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) t[e] = mul2(mul2(h2f(w[e]), fold2), iq2);
            *reinterpret_cast<uint2*>(p.qcodes + ubase + static_cast<size_t>(r0 + row) * D + col) =
                clamp ? pack_codes8<true>(t) : pack_codes8<false>(t);
        }
    }
}

#ifndef SAB_K1_MINB
#define SAB_K1_MINB 4  // <= 64 registers: more Q-chunk CTAs in flight (C2 K1 78 -> 68 us)
#endif
#ifndef SAB_K1_MINB_G
#define SAB_K1_MINB_G SAB_K1_MINB  // CTAs per SM bound when a thread group sums G >= 2 nodes
#endif
template <int D, int G>
__global__ void __launch_bounds__(kQThreads, G >= 2 ? SAB_K1_MINB_G : SAB_K1_MINB) k1_mean_and_q(PrepassParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    griddep_launch_dependents();  // k1_k_fast may be scheduled behind this grid's last wave
    if (static_cast<int>(blockIdx.x) < p.n_partials) mean_partial<__half, D, G>(p, blockIdx.y, blockIdx.x);
    else q_chunk_fast<D>(p, blockIdx.y, blockIdx.x - p.n_partials, smem);
}

// Smooth + quantize the two 64-token K groups of 128-token chunk `chunk`.  FUSED (k1_fused):
// mean(K) is awaited through the unit's ready flag; else (k1_k_fast) through the PDL wait on
// the k1_mean_and_q grid.
template <int D, bool FUSED>
__device__ __forceinline__ void k_chunk_fast(const PrepassParams& p, int unit, int chunk, uint8_t* smem) {
    constexpr int CV = D / 8;
    constexpr int VPT = kBlockQ * CV / kQThreads;
    const __half* sk = reinterpret_cast<const __half*>(smem);
    __shared__ uint64_t bar;
    __shared__ float s_mean[D];
    __shared__ float s_red[kQThreads / 32][2];
    __shared__ float s_inv[2];
    const int tid = threadIdx.x;
    const int r0 = chunk * kBlockQ;
    const int rows = min(kBlockQ, p.n - r0);
    const size_t ubase = static_cast<size_t>(unit) * p.n * D;
    const uint32_t bytes = static_cast<uint32_t>(rows) * D * 2;
    if (tid == 0) {
        mbar_init(smem_u32(&bar), 1);
        fence_barrier_init();
        mbar_arrive_expect_tx(smem_u32(&bar), bytes);
        bulk_load(smem_u32(smem), static_cast<const __half*>(p.k) + ubase + static_cast<size_t>(r0) * D, bytes,
                  smem_u32(&bar));
    }
    // K is an input: its load is in flight before mean(K) is awaited.
    if constexpr (FUSED) {
        // Every ticket this chunk depends on (the unit's mean partials) is lower than its
        // own, so those CTAs are already running: the wait cannot deadlock.
        if (tid == 0) flag_wait(p.ready + unit);
        __syncthreads();
        if (tid == 0 && atomicAdd(p.kdone + unit, 1) == (p.n + kBlockQ - 1) / kBlockQ - 1) {
            p.kdone[unit] = 0;  // every K chunk of the unit is past its wait: reset for the next call
            p.ready[unit] = 0;
        }
        if (tid < D) s_mean[tid] = __ldcg(p.mean + static_cast<size_t>(unit) * D + tid);
    } else {
        // Every CTA waits, so this grid never completes before its producer.
        griddep_wait();
        griddep_launch_dependents();  // K2 may be scheduled behind this grid's last wave
        if (tid < D) s_mean[tid] = p.smooth ? p.mean[static_cast<size_t>(unit) * D + tid] : 0.0f;
    }
    __syncthreads();
    mbar_wait(smem_u32(&bar), 0);
    const int col = (tid % CV) * 8;
    f2 mc[4];
#pragma unroll
    for (int w = 0; w < 4; ++w) mc[w] = f2{-s_mean[col + 2 * w], -s_mean[col + 2 * w + 1]};
    uint32_t kbits = 0;
    float amax0 = 0.0f, amax1 = 0.0f;
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
        const int row = (tid + i * kQThreads) / CV;
        if (row < rows) {
            const uint4 u = *reinterpret_cast<const uint4*>(sk + row * D + col);
            const uint32_t w[4] = {u.x, u.y, u.z, u.w};
            float a = 0.0f;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                kbits = __vmaxu2(kbits, w[e] & 0x7FFF7FFFu);
                const f2 d = add2(h2f(w[e]), mc[e]);
                a = fmaxf(a, fmaxf(fabsf(d.x), fabsf(d.y)));
            }
            if (i < VPT / 2) amax0 = fmaxf(amax0, a);
            else amax1 = fmaxf(amax1, a);
        }
    }
    if (max(kbits & 0xFFFFu, kbits >> 16) >= 0x7C00u) atomicOr(p.status, kStatusNonFinite);
    amax0 = warp_max(amax0);
    amax1 = warp_max(amax1);
    if ((tid & 31) == 0) {
        s_red[tid >> 5][0] = amax0;
        s_red[tid >> 5][1] = amax1;
    }
    __syncthreads();
    if (tid < 2) {
        float m = 0.0f;
        for (int w = 0; w < kQThreads / 32; ++w) m = fmaxf(m, s_red[w][tid]);
        float delta, inv;
        int8_scale(m, delta, inv);
        s_inv[tid] = inv;
        const int ngk = (p.n + kBlockKV - 1) / kBlockKV;
        const int g = 2 * chunk + tid;
        if (g < ngk) p.kscales[static_cast<size_t>(unit) * ngk + g] = delta;
    }
    __syncthreads();
    const float ik0 = s_inv[0], ik1 = s_inv[1];
    const bool clamp = isinf(ik0) || isinf(ik1);
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
        const int row = (tid + i * kQThreads) / CV;
        if (row < rows) {
            const uint4 u = *reinterpret_cast<const uint4*>(sk + row * D + col);
            const uint32_t w[4] = {u.x, u.y, u.z, u.w};
            const float ik = i < VPT / 2 ? ik0 : ik1;
            const f2 ik2{ik, ik};
            f2 t[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) t[e] = mul2(add2(h2f(w[e]), mc[e]), ik2);
            *reinterpret_cast<uint2*>(p.kcodes + ubase + static_cast<size_t>(r0 + row) * D + col) =
                clamp ? pack_codes8<true>(t) : pack_codes8<false>(t);
        }
    }
    if (p.check_v) {
        bool vfin = true;
        for (int v = tid; v < rows * CV; v += kQThreads) {
            const int row = v / CV, c8 = (v % CV) * 8;
            float x[8];
            load8<__half>(static_cast<const __half*>(p.v) + ubase + static_cast<size_t>(r0 + row) * D + c8, x);
            vfin &= all_finite8(x);
        }
        if (!vfin) atomicOr(p.status, kStatusNonFinite);
    }
}

template <int D>
__global__ void __launch_bounds__(kQThreads) k1_k_fast(PrepassParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    k_chunk_fast<D, false>(p, blockIdx.y, blockIdx.x, smem);
}

// Q chunks in their own grid (SAB_K1_SPLITQ=1 experiment: k1_mean_partials -> k1_q_only ->
// k1_k_fast, the Q chunks free of the partial path's register cap).  Q needs no mean(K); the
// last CTA waits for the mean-partials grid before exiting, so this grid completes only after
// it and k1_k_fast's wait on this grid covers mean(K).
template <int D>
__global__ void __launch_bounds__(kQThreads) k1_q_only(PrepassParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    griddep_launch_dependents();  // k1_k_fast's K loads may start behind this grid
    q_chunk_fast<D>(p, blockIdx.y, blockIdx.x, smem);
    if (blockIdx.x == gridDim.x - 1 && blockIdx.y == gridDim.y - 1) griddep_wait();
}

// ---- fp16, per-block path in ONE launch (opt-in experiment, SAB_K1_FUSED=1; measured
// 1.1-1.35x slower than the two launches, profiles/r02_k1_fused_ab.txt).  Each CTA takes a
// ticket (atomic counter) and runs the work item of that ticket.  Items are ordered in
// stages, stage s = [mean partials of unit s][Q chunks of unit s][K chunks of unit s - lag],
// so a K chunk waits (per-unit flag) only on CTAs with lower tickets -- already running, so
// no deadlock -- and re-reads its K rows from L2 a few units after the mean partials read
// them (lag ~ 1.5 resident waves of items): K comes from DRAM once instead of twice, and
// there is no grid-wide dependency between K's mean and its quantization.
template <int D, int G>
__global__ void __launch_bounds__(kQThreads, SAB_K1_MINB) k1_fused(PrepassParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ int s_ticket;
    griddep_launch_dependents();  // K2 may be scheduled behind this grid's last wave
    if (threadIdx.x == 0) {
        const int t = atomicAdd(p.ticket, 1);
        if (t == static_cast<int>(gridDim.x) - 1) *p.ticket = 0;  // every ticket is taken: reset
        s_ticket = t;
    }
    __syncthreads();
    const int t = s_ticket;
    const int np = p.n_partials, nq = (p.n + kBlockQ - 1) / kBlockQ;
    const int pq = np + nq, lag = p.lag;
    const int t1 = lag * pq, t2 = t1 + (p.units - lag) * (pq + nq);
    int unit, r;
    bool kchunk;
    if (t < t1) {
        unit = t / pq;
        r = t - unit * pq;
        kchunk = false;
    } else if (t < t2) {
        const int tt = t - t1, st = tt / (pq + nq);
        r = tt - st * (pq + nq);
        kchunk = r >= pq;
        unit = kchunk ? st : st + lag;
        if (kchunk) r -= pq;
    } else {
        const int tt = t - t2, st = tt / nq;
        unit = p.units - lag + st;
        r = tt - st * nq;
        kchunk = true;
    }
    if (kchunk) k_chunk_fast<D, true>(p, unit, r, smem);
    else if (r < np) mean_partial<__half, D, G, true>(p, unit, r);
    else q_chunk_fast<D>(p, unit, r - np, smem);
}

// ---------------------------------------------------------------- vB: V^ per channel
// quantize(V, Granularity::per_channel(), Int8) (attention.hpp:376-378; quant.hpp:103-173):
// delta_c = max_t |v[t][c]| / 127 over every token of the unit, codes rne(v * 1/delta_c)
// clamped to [-127, 127].  K2 reads V^ as the K-major B operand of a kind::i8 MMA, so the
// codes are written transposed, [units][d][ldv] with ldv = 64 * ceil(N / 64).
constexpr int kVRows = 256;  // tokens per k1_v_amax CTA

// Pass 1: channel max |v| of kVRows tokens, merged into vamax (float bits; non-negative
// floats order like their bit patterns) with one atomicMax per channel and CTA.
template <typename T, int D>
__global__ void __launch_bounds__(kThreads) k1_v_amax(PrepassParams p) {
    constexpr int CV = D / 8;
    __shared__ int smax[D];
    const int tid = threadIdx.x;
    const int unit = blockIdx.y;
    const int t0 = blockIdx.x * kVRows;
    const int rows = min(kVRows, p.n - t0);
    for (int c = tid; c < D; c += kThreads) smax[c] = 0;
    __syncthreads();
    const int cv = tid % CV;
    float mx[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    bool fin = true;
    const T* src = static_cast<const T*>(p.v) + (static_cast<size_t>(unit) * p.n + t0) * D + cv * 8;
    for (int r = tid / CV; r < rows; r += kThreads / CV) {
        float x[8];
        load8<T>(src + static_cast<size_t>(r) * D, x);
        fin &= all_finite8(x);
#pragma unroll
        for (int i = 0; i < 8; ++i) mx[i] = fmaxf(mx[i], fabsf(x[i]));
    }
    if (!fin) atomicOr(p.status, kStatusNonFinite);
#pragma unroll
    for (int i = 0; i < 8; ++i) atomicMax(&smax[cv * 8 + i], __float_as_int(mx[i]));
    __syncthreads();
    for (int c = tid; c < D; c += kThreads) atomicMax(&p.vamax[static_cast<size_t>(unit) * D + c], smax[c]);
}

// Pass 2: 64 tokens x D channels per CTA, quantized and transposed through shared memory.
// Each work item is 4 consecutive tokens x 8 channels: its 8 channel codes of the 4 tokens
// are packed into one 32-bit word per channel.  The transposed tile keeps 16 words (64
// tokens) per channel with the token-quad index XOR-swizzled by the channel octet, so the
// 16 lanes that share a token quad write 16 different banks.
template <typename T, int D>
__global__ void __launch_bounds__(kThreads) k1_v_quant(PrepassParams p) {
    constexpr int CV = D / 8;
    constexpr int NQ = kBlockKV / 4;  // token quads per tile
    __shared__ float sinv[D];
    __shared__ uint32_t tile[D][NQ];
    const int tid = threadIdx.x;
    const int unit = blockIdx.y;
    const int t0 = blockIdx.x * kBlockKV;
    const int rows = min(kBlockKV, p.n - t0);
    for (int c = tid; c < D; c += kThreads) {
        const float amax = __int_as_float(__ldcg(&p.vamax[static_cast<size_t>(unit) * D + c]));
        // quant.hpp:145-151: an all-zero channel takes delta 1 and codes 0.
        const float delta = amax == 0.0f ? 1.0f : amax / 127.0f;
        sinv[c] = amax == 0.0f ? 0.0f : 1.0f / delta;
        if (blockIdx.x == 0) p.vscales[static_cast<size_t>(unit) * D + c] = delta;
    }
    __syncthreads();
    const T* src = static_cast<const T*>(p.v) + (static_cast<size_t>(unit) * p.n + t0) * D;
    for (int e = tid; e < NQ * CV; e += kThreads) {
        const int cv = e % CV, rq = e / CV;
        uint32_t w[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int r = 4 * rq + k;
            float x[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            if (r < rows) load8<T>(src + static_cast<size_t>(r) * D + cv * 8, x);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                float q = rintf(x[i] * sinv[cv * 8 + i]);  // quant.hpp:95-101 (RNE, then clamp)
                q = fminf(fmaxf(q, -127.0f), 127.0f);
                w[i] |= (static_cast<uint32_t>(static_cast<int>(q)) & 0xffu) << (8 * k);
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) tile[cv * 8 + i][rq ^ (cv % NQ)] = w[i];
    }
    __syncthreads();
    int8_t* dst = p.vcodes + static_cast<size_t>(unit) * D * p.ldv + t0;
    for (int e = tid; e < D * (NQ / 4); e += kThreads) {
        const int c = e / (NQ / 4), q4 = (e % (NQ / 4)) * 4, sw = (c / 8) % NQ;
        *reinterpret_cast<uint4*>(dst + static_cast<size_t>(c) * p.ldv + 4 * q4) =
            make_uint4(tile[c][q4 ^ sw], tile[c][(q4 + 1) ^ sw], tile[c][(q4 + 2) ^ sw], tile[c][(q4 + 3) ^ sw]);
    }
}

template <typename T, int D>
cudaError_t launch_v(const PrepassParams& p, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(p.vamax, 0, sizeof(int) * static_cast<size_t>(p.units) * D, s);
    if (e != cudaSuccess) return e;
    k1_v_amax<T, D><<<dim3((p.n + kVRows - 1) / kVRows, p.units), kThreads, 0, s>>>(p);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    k1_v_quant<T, D><<<dim3((p.n + kBlockKV - 1) / kBlockKV, p.units), kThreads, 0, s>>>(p);
    return cudaGetLastError();
}

// The fp16 per-block path for few-unit calls (K3 shards: C2 on 8 GPUs = 4 units) runs as
// k1_mean_partials -> k1_quantize (Q and K of a chunk together, both loads in flight before
// the PDL wait for mean(K)) instead of (mean partials + Q chunks) -> (K chunks): with few
// units the first kernel's Q chunks are the long pole (C2 8-GPU shard K1 28.5 -> 25 us);
// with many units it is 5-15 % slower.  SAB_K1_ALT=0 / 1 forces either.
bool k1_alt(const PrepassParams& p) {
    static const int mode = [] {
        const char* e = std::getenv("SAB_K1_ALT");
        return e ? (e[0] == '1' ? 1 : 0) : -1;
    }();
    return mode >= 0 ? mode == 1 : p.units <= 8;
}

// SAB_K1_FUSED=1 selects k1_fused (measured slower than the two launches, see
// profiles/r02_experiments.md); SAB_K1_LAG_PCT sets its stage lag in percent of one resident
// wave of CTAs (default 150).
bool k1_fused_on() {
    static const bool on = [] {
        const char* e = std::getenv("SAB_K1_FUSED");
        return e && e[0] == '1';
    }();
    return on;
}

template <int D, int G>
cudaError_t launch_k1_fused(PrepassParams p, cudaStream_t s) {
    constexpr int smem = kBlockQ * D * 2;
    static std::atomic<int> resident_cache{0};  // CTAs of k1_fused resident on a (B200) device at once
    cudaError_t e = cudaFuncSetAttribute(k1_fused<D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    int resident = resident_cache.load(std::memory_order_relaxed);
    if (resident == 0) {
        int dev = 0, sms = 0, per_sm = 0;
        if ((e = cudaGetDevice(&dev)) != cudaSuccess ||
            (e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess ||
            (e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k1_fused<D, G>, kQThreads, smem)) !=
                cudaSuccess)
            return e;
        resident = std::max(1, sms * per_sm);
        resident_cache.store(resident, std::memory_order_relaxed);
    }
    static const int pct = [] {
        const char* e = std::getenv("SAB_K1_LAG_PCT");
        return e ? std::max(0, std::atoi(e)) : 150;
    }();
    const int nq = (p.n + kBlockQ - 1) / kBlockQ;
    const long long per_stage = p.n_partials + 2LL * nq;
    const long long lag_items = static_cast<long long>(resident) * pct / 100;
    p.lag = static_cast<int>(std::min<long long>(p.units, std::max<long long>(1, (lag_items + per_stage - 1) / per_stage)));
    const long long items = per_stage * p.units;
    if (items > 0x7FFFFFFFLL) return cudaErrorInvalidValue;
    k1_fused<D, G><<<static_cast<unsigned>(items), kQThreads, smem, s>>>(p);
    return cudaGetLastError();
}

bool k1_splitq_on() {
    static const bool on = [] {
        const char* e = std::getenv("SAB_K1_SPLITQ");
        return e && e[0] == '1';
    }();
    return on;
}

template <typename T, int D>
cudaError_t launch_qk(const PrepassParams& p, cudaStream_t s) {
    constexpr int NG = kThreads / (D / 8);
    if (std::is_same<T, __half>::value && p.smooth && !p.per_token && !p.rope && k1_splitq_on()) {
        const int ntq = (p.n + kBlockQ - 1) / kBlockQ;
        constexpr int smem = kBlockQ * D * 2;
        const int g = p.nodes_per_cta >= NG ? p.nodes_per_cta / NG : 1;
        const dim3 grid(p.n_partials, p.units);
        switch (g) {
            case 1: k1_mean_partials<__half, D, 1><<<grid, kThreads, 0, s>>>(p); break;
            case 2: k1_mean_partials<__half, D, 2><<<grid, kThreads, 0, s>>>(p); break;
            case 4: k1_mean_partials<__half, D, 4><<<grid, kThreads, 0, s>>>(p); break;
            default: return cudaErrorInvalidValue;
        }
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        if ((e = cudaFuncSetAttribute(k1_q_only<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)) != cudaSuccess ||
            (e = launch_pdl(k1_q_only<D>, dim3(ntq, p.units), dim3(kQThreads), smem, s, p)) != cudaSuccess ||
            (e = cudaFuncSetAttribute(k1_k_fast<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)) != cudaSuccess)
            return e;
        return launch_pdl(k1_k_fast<D>, dim3(ntq, p.units), dim3(kQThreads), smem, s, p);
    }
    if (std::is_same<T, __half>::value && p.smooth && !p.per_token && !p.rope && k1_fused_on()) {
        const int g = p.nodes_per_cta >= NG ? p.nodes_per_cta / NG : 1;
        return g == 1 ? launch_k1_fused<D, 1>(p, s) : g == 2 ? launch_k1_fused<D, 2>(p, s) : launch_k1_fused<D, 4>(p, s);
    }
    if (std::is_same<T, __half>::value && p.smooth && !p.per_token && !p.rope && !k1_alt(p)) {
        const int ntq = (p.n + kBlockQ - 1) / kBlockQ;
        constexpr int smem = kBlockQ * D * 2;
        const int g = p.nodes_per_cta >= NG ? p.nodes_per_cta / NG : 1;
        cudaError_t e;
        if (g == 1) {
            e = cudaFuncSetAttribute(k1_mean_and_q<D, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            if (e == cudaSuccess) k1_mean_and_q<D, 1><<<dim3(p.n_partials + ntq, p.units), kQThreads, smem, s>>>(p);
        } else if (g == 2) {
            e = cudaFuncSetAttribute(k1_mean_and_q<D, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            if (e == cudaSuccess) k1_mean_and_q<D, 2><<<dim3(p.n_partials + ntq, p.units), kQThreads, smem, s>>>(p);
        } else {
            e = cudaFuncSetAttribute(k1_mean_and_q<D, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            if (e == cudaSuccess) k1_mean_and_q<D, 4><<<dim3(p.n_partials + ntq, p.units), kQThreads, smem, s>>>(p);
        }
        if (e != cudaSuccess) return e;
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        e = cudaFuncSetAttribute(k1_k_fast<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        return launch_pdl(k1_k_fast<D>, dim3(ntq, p.units), dim3(kQThreads), smem, s, p);
    }
    if (p.smooth) {
        const dim3 grid(p.n_partials, p.units);
        const int g = p.nodes_per_cta >= NG ? p.nodes_per_cta / NG : 1;
        switch (g) {  // nodes_per_cta() <= 64 -> at most 4 nodes per thread group
            case 1: k1_mean_partials<T, D, 1><<<grid, kThreads, 0, s>>>(p); break;
            case 2: k1_mean_partials<T, D, 2><<<grid, kThreads, 0, s>>>(p); break;
            case 4: k1_mean_partials<T, D, 4><<<grid, kThreads, 0, s>>>(p); break;
            default: return cudaErrorInvalidValue;
        }
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    const dim3 grid((p.n + kBlockQ - 1) / kBlockQ, p.units);
    constexpr int smem = 2 * kBlockQ * D * static_cast<int>(sizeof(T));
    cudaError_t e = cudaFuncSetAttribute(k1_quantize<T, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    if (p.smooth) return launch_pdl(k1_quantize<T, D>, grid, dim3(kQThreads), smem, s, p);
    k1_quantize<T, D><<<grid, kQThreads, smem, s>>>(p);
    return cudaGetLastError();
}

template <typename T, int D>
cudaError_t launch_typed(const PrepassParams& p, cudaStream_t s) {
    cudaError_t e = launch_qk<T, D>(p, s);
    if (e == cudaSuccess && p.vcodes) e = launch_v<T, D>(p, s);
    return e;
}

}  // namespace

cudaError_t launch_prepass(const PrepassParams& p, cudaStream_t s) {
    if (p.d == 128) return p.in_f32 ? launch_typed<float, 128>(p, s) : launch_typed<__half, 128>(p, s);
    if (p.d == 64) return p.in_f32 ? launch_typed<float, 64>(p, s) : launch_typed<__half, 64>(p, s);
    return cudaErrorInvalidValue;
}

}  // namespace sab
