// sab_attention.cu -- K2, the SageAttn-B attention kernel for sm_100a.
//
// Replaces the q-block / kv-block engine of attention.hpp:383-541:
//   detail::int8_tile_nt (265-279)          -> tcgen05.mma kind::i8, INT32 accumulators in TMEM
//   s = (float(acc) * dQ) * dK (409-414)    -> one FFMA per element with dQ*dK*log2(e) (exp2 domain)
//   causal tile classes (79-94, 399-427)    -> fully masked KV tiles are never issued; the element
//                                              mask runs only on the diagonal / ragged tail tile
//   online softmax (429-443)                -> registers, two threads per query row
//   per-token scales (variant T, 410-413)   -> per-element dQ[row] * dK[key]; one pass against the
//                                              stale max, exact two-pass fallback (softmax_half_pt)
//   P~ V with binary16 operands (447-475)   -> P packed to fp16 into TMEM (aliasing S),
//                                              tcgen05.mma kind::f16 with A from TMEM, V from SMEM,
//                                              FP32 accumulator in TMEM (the pv_fp32_accumulator arm)
//   O = diag(l)^-1 O + overflow check (524-540) -> epilogue from TMEM, status word on non-finite O
//
// One CTA = one unit x 256 query rows = two 128-row query tiles A and B that
// share every K^/V tile.  KV tiles are 64 keys = one K quantization group
// (attention.hpp:345), so each S tile has a single dequant factor.
// Warp roles (576 threads):
//   warps 0-7  softmax + epilogue of tile A, warps 8-15 of tile B: each warp owns 16
//              query rows (16 TMEM lanes); threads t and t+16 split a row's 64 keys
//              (tcgen05.ld 16x32bx2), so 4 softmax warps share each SM sub-partition
//              (the exponentials are latency-bound at 2 warps per sub-partition and
//              MUFU-bound at 4; see scripts/micro/softmax_row.cu)
//   warp  16   TMA producer (Q^ of both tiles once; K^ and V per 64-key tile on one
//              barrier, STAGES-deep ring)
//   warp  17   MMA issuer of both tiles (warp-uniform loop in uniform registers, one
//              elected lane issues): per KV tile j, PV_A(j) once P_A(j) is in TMEM, then
//              bias + QK_A(j+2) into the same S buffer, then the same for tile B.
// S bias: each S tile starts with one kind::f16 MMA of constant operands that writes
// the binary32 value 2^23 + 2^22 (bits 0x4B400000) into every accumulator; the
// kind::i8 MMAs then accumulate INT32 products onto those bits, so the softmax reads
// float(2^23 + 2^22 + acc) with no per-element integer-to-float conversion.
// TMEM (512 columns): S_x[b] = [128x + 64b, +64), double-buffered per tile x,
//                      with P_x(j) stored as fp16x2 over the first 32 columns of
//                      S_x[j%2] (the A operand of the TMEM-sourced PV MMA);
//                      O_A [256, 256+D), O_B [256+D, 256+2D) fp32 accumulators.
// The tensor pipe runs one thread's tcgen05 ops in order, so issuing QK_x(j+2)
// after PV_x(j) keeps P_x(j) intact until it has been read, and QK_x(j+1) runs
// while softmax x(j) computes.
// Rescaling of O is lazy (only when a row max grows by more than 2^8), which is
// exact in real arithmetic because l and O share the stale max.
#include <cuda.h>
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cuda_fp16.h>

#include "sab_internal.h"
#include "sab_ptx.cuh"

namespace sab {

#ifdef SAB_TRACE
// Debug timeline (SAB_TRACE builds only): clock64 stamps of one CTA's pipeline
// events, trace[(role * kTraceTiles + tile) * 8 + event].  Roles: 0/1 softmax
// warp 0 of tile A/B, 2/3 MMA issuer of tile A/B, 4 TMA producer.
__device__ long long* g_trace = nullptr;
__device__ int g_trace_cta = 0;
long long* h_trace_ptr = nullptr;
int h_trace_cta = 0;
#endif

namespace {

#ifdef SAB_TRACE
constexpr int kTraceTiles = 512;
#define SAB_STAMP(role, tile, ev)                                                                      \
    do {                                                                                              \
        if (g_trace && blockIdx.x == static_cast<unsigned>(g_trace_cta) && (tile) < kTraceTiles)      \
            g_trace[((role) * kTraceTiles + (tile)) * 8 + (ev)] = clock64();                            \
    } while (0)
#else
#define SAB_STAMP(role, tile, ev) \
    do {                          \
    } while (0)
#endif

constexpr int kBM = 128;
constexpr int kBN = 64;    // keys per KV tile = one K scale group
constexpr int kThreads = 576;  // 16 softmax warps + TMA producer + MMA issuer
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescaleThreshold = 8.0f;  // log2 units
constexpr float kRescaleLimit = 256.0f;    // 2^kRescaleThreshold
constexpr uint32_t kMagicI = 0x4B400000u;  // bits of 2^23 + 2^22
constexpr int kMaskedAcc = 0;              // sentinel below any biased S value (bits of +0.0f)
// Exponentials (of every 16) evaluated by exp2_poly2 on the FMA pipe instead of MUFU,
// per head dim (d=64 is MUFU-bound, d=128 closer to the tensor/SMEM bound).
// Which pairs of each 8 take the FMA-pipe exponential: pair index p with
// ((2p + rot) & 15) >= 16 - POLY.  Only the instruction schedule changes (C3 +1.4 % at
// rot 2 for d=64, C2 +0.6 % at rot 8 for d=128, profiles/r02_polyrot_ab.txt).
#ifndef SAB_POLYROT64
#define SAB_POLYROT64 2
#endif
#ifndef SAB_POLYROT128
#define SAB_POLYROT128 8
#endif
#ifndef SAB_POLY128
#define SAB_POLY128 2
#endif
#ifndef SAB_POLY64
#define SAB_POLY64 2
#endif
template <int D>
constexpr int poly_per16() { return D == 64 ? SAB_POLY64 : SAB_POLY128; }
template <int D>
constexpr int poly_rot() { return D == 64 ? SAB_POLYROT64 : SAB_POLYROT128; }
constexpr float kMagicF = 12582912.0f;     // 2^23 + 2^22

// ------------------------------------------------------------ packed fp32 math
struct f2 {
    float x, y;
};

__device__ __forceinline__ f2 ffma2(f2 a, f2 b, f2 c) {
    f2 d;
    asm("{\n\t.reg .b64 a, b, c, d;\n\t"
        "mov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\tmov.b64 c, {%6, %7};\n\t"
        "fma.rn.f32x2 d, a, b, c;\n\tmov.b64 {%0, %1}, d;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return d;
}

__device__ __forceinline__ f2 fadd2(f2 a, f2 b) {
    f2 d;
    asm("{\n\t.reg .b64 a, b, d;\n\t"
        "mov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
        "add.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}

// 2^x on the FMA pipe for a pair: x = j + f with j = rint(x), f in [-0.5, 0.5];
// 2^f by a degree-3 minimax polynomial (max rel. error 7.5e-5, below the
// binary16 rounding P~ gets next); j is added to the exponent field.
__device__ __forceinline__ f2 exp2_poly2(f2 x) {
    x.x = fmaxf(x.x, -126.0f);
    x.y = fmaxf(x.y, -126.0f);
    const f2 t = fadd2(x, f2{kMagicF, kMagicF});                   // rint(x) in the low mantissa bits
    const f2 f = ffma2(fadd2(t, f2{-kMagicF, -kMagicF}), f2{-1.0f, -1.0f}, x);  // x - rint(x), exact
    f2 p = ffma2(f2{0.05517154186964035f, 0.05517154186964035f}, f, f2{0.24261118471622467f, 0.24261118471622467f});
    p = ffma2(p, f, f2{0.6932610273361206f, 0.6932610273361206f});
    p = ffma2(p, f, f2{0.9999280571937561f, 0.9999280571937561f});
    return f2{__uint_as_float(__float_as_uint(p.x) + (__float_as_uint(t.x) << 23)),
              __uint_as_float(__float_as_uint(p.y) + (__float_as_uint(t.y) << 23))};
}

// Binary16 P~V accumulator (AttnParams::pv16): a kind::f16 MMA with c_format F16 keeps one
// value per 32-bit TMEM column, in the low half (upper half zero; scripts/micro/f16acc.cu).
__device__ __forceinline__ float f16acc_get(uint32_t cell) {
    return __half2float(__ushort_as_half(static_cast<unsigned short>(cell & 0xFFFFu)));
}
__device__ __forceinline__ uint32_t f16acc_put(float x) {
    return static_cast<uint32_t>(__half_as_ushort(__float2half_rn(x)));
}

template <int D>
struct Cfg {
#ifndef SAB_STAGES128
#define SAB_STAGES128 6
#endif
#ifndef SAB_NB64
#define SAB_NB64 2
#endif
#ifndef SAB_STAGES64
#define SAB_STAGES64 8
#endif
    static constexpr int kStages = D == 128 ? SAB_STAGES128 : SAB_STAGES64;  // K^/V ring depth
    // S buffers per query tile: 3 when O is narrow enough (d=64: 2 x 3 x 64 + 2 x 64 = 512
    // TMEM columns), else 2.  A deeper S ring gives QK_x(j+NB) more slack behind PV_x(j).
    static constexpr int kNB = D == 64 ? SAB_NB64 : 2;
    static constexpr int kOffO = 2 * kNB * 64;  // TMEM column of O_A
    static constexpr int kQBytes = kBM * D;
    static constexpr int kKBytes = kBN * D;
    static constexpr int kVBytes = kBN * D * 2;
    static constexpr int kVChunk = kBN * 64 * 2;  // one 64-column SW128 panel of V
    static constexpr uint32_t kSwizzleQK = D == 128 ? kSwizzle128B : kSwizzle64B;
    static constexpr uint32_t kSboQK = 8 * D;     // 8 rows of D int8
    static constexpr int kOffQ = 0;
    static constexpr int kOffK = kOffQ + 2 * kQBytes;
    static constexpr int kOffV = kOffK + kStages * kKBytes;
    // Constant fp16 operands of the bias MMA (A: 2048, B: 384; 16 * 2048 * 384 = 2^23 + 2^22).
    static constexpr int kOffBiasA = kOffV + kStages * kVBytes;
    static constexpr int kOffBiasB = kOffBiasA + 8192;
    static constexpr int kOffBar = kOffBiasB + 4096;
    static constexpr int kSmemBytes = kOffBar + 1024 + 1024;  // barriers + alignment slack
};

// One K2 work item: a unit's query-tile pair (qt0, qt0 + 1), or a KV chunk of it.
struct Item {
    int it;  // index in the launch's item order (>= p.items: no more work)
    int unit, pair, chunk, qt0, nkv_a, nkv_b, nkv, j0, nch;
    int has_b;
};

struct Bars {  // must fit the 1024 bytes reserved at Cfg::kOffBar
    uint64_t q_full;
    uint64_t kv_full[16], kv_empty[16];
    uint64_t s_full[2][3], p_full[2][3], pv_done[2][3], o_final[2];
    // Persistent work loop: the producer publishes each work item in a 2-slot ring;
    // q_free: the item's last QK^T MMA has read Q^ (its buffer may be refilled);
    // o_free[x]: the item's epilogue has read O_x (the next item's first PV may overwrite it).
    uint64_t item_full[2], item_empty[2], q_free, o_free[2];
    Item items[2];  // the decoded items of the ring (consumers read them in place)
    uint32_t tmem_base;
    int split_last;  // KV split: this CTA finished its pair's last chunk and merges
};

__device__ __forceinline__ void softmax_bar_sync() {  // the 16 softmax warps (threads 0-511)
    asm volatile("bar.sync 1, 512;" ::: "memory");
}

// Opaque copy: stops the compiler from keeping the 128 per-key mask predicates
// of pass 1 alive (in registers) until pass 2.
__device__ __forceinline__ int opaque(int v) {
    int r;
    asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
    return r;
}

// Max of N biased S accumulators as integers (2^23 + 2^22 + acc: positive
// binary32 values, ordered like their bit patterns): 4 independent chains.
// With MASK, columns >= lim are excluded.
template <bool MASK, int N>
__device__ __forceinline__ int group_max(const uint32_t (&r)[N], int lim) {
    int mi[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) mi[e] = kMaskedAcc;
#pragma unroll
    for (int c = 0; c < N; c += 8)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            int a = static_cast<int>(r[c + e]), b = static_cast<int>(r[c + 4 + e]);
            if (MASK) {
                a = (c + e >= lim) ? kMaskedAcc : a;
                b = (c + 4 + e >= lim) ? kMaskedAcc : b;
            }
            mi[e] = max(mi[e], max(a, b));
        }
    return max(max(mi[0], mi[1]), max(mi[2], mi[3]));
}

// Softmax of one 64-key S tile row, shared by two threads of a warp: thread t
// (< 16) holds keys [0, 32) and thread t + 16 keys [32, 64) of TMEM lane t
// (r, loaded by the caller with tcgen05.ld 16x32bx2).  S holds INT32 accumulators of one K scale group with
// dequant factor cg = dQ*dK*log2 e.  P is written as fp16x2 over the first 32
// columns of the same S region (tcgen05.st 16x32bx2: thread t's 16 packed pairs
// go to columns [16*half, 16*half + 16)), the A operand of the PV MMA.  Updates
// the running max m (log2 units) and this thread's partial row sum l; returns the
// O rescale factor (1 when the warp skips the lazy rescale).  `dump` receives
// the raw half row.
template <bool MASK, bool CAUSAL, int POLY, int ROT>
__device__ __forceinline__ float softmax_half(const uint32_t (&r)[32], uint32_t ts, int half, float cg, int kb, int qi,
                                              int n, float& m, float& l, bool& rescale, int32_t* dump,
                                              int trole = -1, int ttile = 0) {
    // Keys kb + 32*half + c are valid for c < lim: key < N and, when causal, key <= query.
    const int lim = (CAUSAL ? min(n, qi + 1) : n) - kb - 32 * half;
    if (trole >= 0) SAB_STAMP(trole, ttile, 5);
    if (dump) {
#pragma unroll
        for (int c = 0; c < 32; c += 4)  // the raw INT32 accumulators (bias removed)
            *reinterpret_cast<int4*>(dump + c) = make_int4(r[c] - kMagicI, r[c + 1] - kMagicI, r[c + 2] - kMagicI,
                                                           r[c + 3] - kMagicI);
    }
    // Row max on the INT32 accumulators: acc -> acc*cg is monotone for cg > 0, so
    // this is the reference's binary32 row max (attention.hpp:431-432) up to the
    // final scaling.  The two halves of a row meet by a shuffle.
    int imax = group_max<MASK>(r, lim);
    imax = max(imax, __shfl_xor_sync(0xffffffffu, imax, 16));
    const float mx = (MASK && imax == kMaskedAcc) ? -INFINITY : (__int_as_float(imax) - kMagicF) * cg;
    const float m_new = fmaxf(m, mx);
    rescale = __any_sync(0xffffffffu, m_new > m + kRescaleThreshold);
    float alpha = 1.0f;
    if (rescale) {
        // A row with no visible key yet (a KV-split chunk right of a causal row) keeps
        // m = -inf: nothing to rescale.
        alpha = m_new == -INFINITY ? 1.0f : ex2(m - m_new);
        m = m_new;
    }
    if (trole >= 0) SAB_STAMP(trole, ttile, 6);
    const float mref = (m == -INFINITY) ? 0.0f : m;
    // p = 2^(float(acc) * cg - m).  The S accumulators arrive biased: their bits are
    // bits(2^23 + 2^22) + acc (the bias MMA, see k2_attention), i.e. the binary32 value
    // 2^23 + 2^22 + acc exactly for |acc| < 2^22 (|acc| <= 127^2 * 128 here), so
    // float(acc) * cg - m is half an FFMA2 per element with no conversion.
    const f2 cg2{cg, cg};
    const float bgs = -fmaf(kMagicF, cg, mref);
    const f2 bg{bgs, bgs};
    const int lim2 = MASK ? opaque(lim) : lim;
    f2 acc[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
    uint32_t pk[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const int c = 2 * i;
        const f2 t = ffma2(f2{__uint_as_float(r[c]), __uint_as_float(r[c + 1])}, cg2, bg);
        f2 pp;
#ifdef SAB_SK_NOEXP  // timing skeleton: no exponentials (wrong results)
        pp = t;
#else
        if (((c + ROT) & 15) >= 16 - POLY) {  // part of the exponentials on the FMA pipe
            pp = exp2_poly2(t);
        } else {
            pp = f2{ex2(t.x), ex2(t.y)};
        }
#endif
        if (MASK) {
            pp.x = (c >= lim2) ? 0.0f : pp.x;
            pp.y = (c + 1 >= lim2) ? 0.0f : pp.y;
        }
        pk[i] = pack_half2(pp.x, pp.y);
        acc[i & 3] = i < 4 ? pp : fadd2(acc[i & 3], pp);  // (the first four start the chains)
    }
    if (trole >= 0) SAB_STAMP(trole, ttile, 7);
    tmem_st16x2_16(ts, pk);
    const f2 sum = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
    l = fmaf(l, alpha, sum.x + sum.y);
    return alpha;
}

// SageDiagnostics::measure_static_scale (attention.hpp:479-488): the per-token-scale codes
// of this tile row (quantize(P~, per_token, Int8), quant.hpp:128-173: delta = max/127,
// inv = 1/delta, clamp(rint(p * inv))) against the static-scale codes rint(p * 127)
// (quantize_p_static, quant.hpp:258-279).  p holds this thread's 32 values of the row
// (masked entries 0); the row's two threads meet by a shuffle.  Rows past the last
// token are not part of the reference's tile and are skipped.
__device__ __forceinline__ void count_static_scale_mismatches(const float (&p)[32], bool row_valid, bool first,
                                                              unsigned long long* diag) {
    float pm = 0.0f;
#pragma unroll
    for (int c = 0; c < 32; ++c) pm = fmaxf(pm, p[c]);
    pm = fmaxf(pm, __shfl_xor_sync(0xffffffffu, pm, 16));
    const float delta = pm == 0.0f ? 1.0f : __fdiv_rn(pm, 127.0f);
    const float inv = pm == 0.0f ? 0.0f : __fdiv_rn(1.0f, delta);
    int mism = 0;
#pragma unroll
    for (int c = 0; c < 32; ++c) {
        const float cs = fminf(rintf(__fmul_rn(p[c], 127.0f)), 127.0f);
        const float ct = fminf(fmaxf(rintf(__fmul_rn(p[c], inv)), -127.0f), 127.0f);
        mism += cs != ct;
    }
    mism = __reduce_add_sync(0xffffffffu, row_valid ? mism : 0);
    if ((threadIdx.x & 31) == 0 && mism) atomicAdd(diag + (first ? 0 : 1), static_cast<unsigned long long>(mism));
}

// SAGEAttn-vB variant of softmax_half (INT8 P~V, attention.hpp:476-505): the running max
// is exact (no lazy threshold) so every p lies in [0, 1], and P~ is stored as the static-scale
// codes rne(p * 127) (quantize_p_static, quant.hpp:258-279), four per TMEM column (thread t's
// 8 words go to columns [8*half, 8*half + 8)), the A operand of the kind::i8 PV MMA.  All
// exponentials are MUFU ex2 of float(acc) * cg - m (one rounding), so the codes are the
// reference's up to an ulp of the exponent.  Returns the O rescale factor 2^(m_old - m).
template <bool MASK, bool CAUSAL, bool DIAG>
__device__ __forceinline__ float softmax_half_i8(const uint32_t (&r)[32], uint32_t ts, int half, float cg, int kb,
                                                 int qi, int n, float& m, float& l, bool& rescale,
                                                 unsigned long long* diag, bool first) {
    const int lim = (CAUSAL ? min(n, qi + 1) : n) - kb - 32 * half;
    int imax = group_max<MASK>(r, lim);
    imax = max(imax, __shfl_xor_sync(0xffffffffu, imax, 16));
    const float mx = (MASK && imax == kMaskedAcc) ? -INFINITY : (__int_as_float(imax) - kMagicF) * cg;
    const float m_new = fmaxf(m, mx);
    rescale = __any_sync(0xffffffffu, m_new > m);
    const float alpha = (m_new > m) ? ex2(m - m_new) : 1.0f;
    m = m_new;
    const float mref = (m == -INFINITY) ? 0.0f : m;
    const f2 cg2{cg, cg};
    const int lim2 = MASK ? opaque(lim) : lim;
    f2 acc[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
    uint32_t pk[8];
    float pd[DIAG ? 32 : 1];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        uint32_t b[4];
#pragma unroll
        for (int e = 0; e < 4; e += 2) {
            const int c = 4 * i + e;
            const f2 a = fadd2(f2{__uint_as_float(r[c]), __uint_as_float(r[c + 1])}, f2{-kMagicF, -kMagicF});
            const f2 t = ffma2(a, cg2, f2{-mref, -mref});
            f2 pp{ex2(t.x), ex2(t.y)};
            if (MASK) {
                pp.x = (c >= lim2) ? 0.0f : pp.x;
                pp.y = (c + 1 >= lim2) ? 0.0f : pp.y;
            }
            if (DIAG) {
                pd[c] = pp.x;
                pd[c + 1] = pp.y;
            }
            acc[(2 * i + e / 2) & 3] = fadd2(acc[(2 * i + e / 2) & 3], pp);
            // rne(p * 127): the product rounded to binary32 (quant.hpp:96), then 2^23 + 2^22
            // added so the code sits in the low mantissa byte.
            const f2 q = fadd2(ffma2(pp, f2{127.0f, 127.0f}, f2{0.0f, 0.0f}), f2{kMagicF, kMagicF});
            b[e] = __float_as_uint(q.x);
            b[e + 1] = __float_as_uint(q.y);
        }
        pk[i] = __byte_perm(__byte_perm(b[0], b[1], 0x0040), __byte_perm(b[2], b[3], 0x0040), 0x5410);
    }
    tmem_st16x2_8(ts, pk);
    if (DIAG) count_static_scale_mismatches(reinterpret_cast<const float(&)[32]>(pd), qi < n, first, diag);
    const f2 sum = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
    l = fmaf(l, alpha, sum.x + sum.y);
    return alpha;
}

// SAGEAttn-T variant of softmax_half: per-token scales, so the dequant factor
// w = dQ[row] * dK[key] * log2 e differs per element and the row max is taken on
// the scaled scores (attention.hpp:409-414 with per_token group_of, quant.hpp:56-63).
// dkp points at this thread's 32 key scales (K1 pads each unit's scale row to a
// multiple of 64, so the float4 loads stay in bounds); r is overwritten with the
// scores.  Same contract as softmax_half otherwise.
template <bool MASK, bool CAUSAL, int POLY>
__device__ __forceinline__ float softmax_half_pt(uint32_t (&r)[32], uint32_t ts, int half, float dq, const float* dkp,
                                                 int kb, int qi, int n, float& m, float& l, bool& rescale,
                                                 int32_t* dump, bool first) {
    const int lim = (CAUSAL ? min(n, qi + 1) : n) - kb - 32 * half;
    if (dump) {
#pragma unroll
        for (int c = 0; c < 32; c += 4)  // the raw INT32 accumulators (bias removed)
            *reinterpret_cast<int4*>(dump + c) = make_int4(r[c] - kMagicI, r[c + 1] - kMagicI, r[c + 2] - kMagicI,
                                                           r[c + 3] - kMagicI);
    }
    const int lim2 = MASK ? opaque(lim) : lim;
    if (!first) {
        // Lazy rescaling keeps m until a row max exceeds it by 2^8, so after the first tile
        // the exponentials run in one pass against the current m, and the exact two-pass
        // path below is taken only if some p of the warp exceeds 2^8.
        f2 acc[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
        float pm[4] = {0.f, 0.f, 0.f, 0.f};
        uint32_t pk[16];
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            const float4 dk4 = __ldg(reinterpret_cast<const float4*>(dkp) + g);
            const f2 w0 = ffma2(f2{dq, dq}, f2{dk4.x, dk4.y}, f2{0.0f, 0.0f});
            const f2 w1 = ffma2(f2{dq, dq}, f2{dk4.z, dk4.w}, f2{0.0f, 0.0f});
#pragma unroll
            for (int e = 0; e < 4; e += 2) {
                const int c = 4 * g + e;
                const f2 a = fadd2(f2{__uint_as_float(r[c]), __uint_as_float(r[c + 1])}, f2{-kMagicF, -kMagicF});
                const f2 t = ffma2(a, e == 0 ? w0 : w1, f2{-m, -m});
                f2 pp;
                if ((c & 15) >= 16 - POLY) {
                    pp = exp2_poly2(t);
                } else {
                    pp = f2{ex2(t.x), ex2(t.y)};
                }
                if (MASK) {
                    pp.x = (c >= lim2) ? 0.0f : pp.x;
                    pp.y = (c + 1 >= lim2) ? 0.0f : pp.y;
                }
                pk[c / 2] = pack_half2(pp.x, pp.y);
                acc[g & 3] = (g < 4 && e == 0) ? pp : fadd2(acc[g & 3], pp);
                pm[g & 3] = fmaxf(pm[g & 3], fmaxf(pp.x, pp.y));
            }
        }
        const float pmax = fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3]));
        if (!__any_sync(0xffffffffu, pmax > kRescaleLimit)) {
            tmem_st16x2_16(ts, pk);
            const f2 sum = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
            l += sum.x + sum.y;
            rescale = false;
            return 1.0f;
        }
    }
    float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
    for (int g = 0; g < 8; ++g) {
        const float4 dk4 = __ldg(reinterpret_cast<const float4*>(dkp) + g);
        const f2 w0 = ffma2(f2{dq, dq}, f2{dk4.x, dk4.y}, f2{0.0f, 0.0f});
        const f2 w1 = ffma2(f2{dq, dq}, f2{dk4.z, dk4.w}, f2{0.0f, 0.0f});
#pragma unroll
        for (int e = 0; e < 4; e += 2) {
            const int c = 4 * g + e;
            // float(acc) exactly: the biased bits minus 2^23 + 2^22.
            const f2 a = fadd2(f2{__uint_as_float(r[c]), __uint_as_float(r[c + 1])}, f2{-kMagicF, -kMagicF});
            f2 sv = ffma2(a, e == 0 ? w0 : w1, f2{0.0f, 0.0f});
            if (MASK) {
                sv.x = (c >= lim2) ? -INFINITY : sv.x;
                sv.y = (c + 1 >= lim2) ? -INFINITY : sv.y;
            }
            mx4[g & 3] = fmaxf(mx4[g & 3], fmaxf(sv.x, sv.y));
            r[c] = __float_as_uint(sv.x);
            r[c + 1] = __float_as_uint(sv.y);
        }
    }
    float mx = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
    const float m_new = fmaxf(m, mx);
    rescale = __any_sync(0xffffffffu, m_new > m + kRescaleThreshold);
    float alpha = 1.0f;
    if (rescale) {
        // A row with no visible key yet (a KV-split chunk right of a causal row) keeps
        // m = -inf: nothing to rescale.
        alpha = m_new == -INFINITY ? 1.0f : ex2(m - m_new);
        m = m_new;
    }
    const float mref = (m == -INFINITY) ? 0.0f : m;
    f2 acc[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
    uint32_t pk[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const int c = 2 * i;
        const f2 t = fadd2(f2{__uint_as_float(r[c]), __uint_as_float(r[c + 1])}, f2{-mref, -mref});
        f2 pp;
        if ((c & 15) >= 16 - POLY) {
            pp = exp2_poly2(t);
        } else {
            pp = f2{ex2(t.x), ex2(t.y)};
        }
        if (MASK) {
            pp.x = (c >= lim2) ? 0.0f : pp.x;
            pp.y = (c + 1 >= lim2) ? 0.0f : pp.y;
        }
        pk[i] = pack_half2(pp.x, pp.y);
        acc[i & 3] = i < 4 ? pp : fadd2(acc[i & 3], pp);
    }
    tmem_st16x2_16(ts, pk);
    const f2 sum = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
    l = fmaf(l, alpha, sum.x + sum.y);
    return alpha;
}

// SAGEAttn-vT: per-token scales (softmax_half_pt's exact pass) with the vB P~ store:
// scores w*acc per element, exact row max, MUFU exponentials, static-scale INT8 codes.
template <bool MASK, bool CAUSAL, bool DIAG>
__device__ __forceinline__ float softmax_half_pt_i8(uint32_t (&r)[32], uint32_t ts, int half, float dq,
                                                    const float* dkp, int kb, int qi, int n, float& m, float& l,
                                                    bool& rescale, unsigned long long* diag, bool first) {
    const int lim = (CAUSAL ? min(n, qi + 1) : n) - kb - 32 * half;
    const int lim2 = MASK ? opaque(lim) : lim;
    float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
    for (int g = 0; g < 8; ++g) {
        const float4 dk4 = __ldg(reinterpret_cast<const float4*>(dkp) + g);
        const f2 w0 = ffma2(f2{dq, dq}, f2{dk4.x, dk4.y}, f2{0.0f, 0.0f});
        const f2 w1 = ffma2(f2{dq, dq}, f2{dk4.z, dk4.w}, f2{0.0f, 0.0f});
#pragma unroll
        for (int e = 0; e < 4; e += 2) {
            const int c = 4 * g + e;
            const f2 a = fadd2(f2{__uint_as_float(r[c]), __uint_as_float(r[c + 1])}, f2{-kMagicF, -kMagicF});
            f2 sv = ffma2(a, e == 0 ? w0 : w1, f2{0.0f, 0.0f});
            if (MASK) {
                sv.x = (c >= lim) ? -INFINITY : sv.x;
                sv.y = (c + 1 >= lim) ? -INFINITY : sv.y;
            }
            mx4[g & 3] = fmaxf(mx4[g & 3], fmaxf(sv.x, sv.y));
            r[c] = __float_as_uint(sv.x);
            r[c + 1] = __float_as_uint(sv.y);
        }
    }
    float mx = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
    const float m_new = fmaxf(m, mx);
    rescale = __any_sync(0xffffffffu, m_new > m);
    const float alpha = (m_new > m) ? ex2(m - m_new) : 1.0f;
    m = m_new;
    const float mref = (m == -INFINITY) ? 0.0f : m;
    f2 acc[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
    uint32_t pk[8];
    float pd[DIAG ? 32 : 1];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        uint32_t b[4];
#pragma unroll
        for (int e = 0; e < 4; e += 2) {
            const int c = 4 * i + e;
            const f2 t = fadd2(f2{__uint_as_float(r[c]), __uint_as_float(r[c + 1])}, f2{-mref, -mref});
            f2 pp{ex2(t.x), ex2(t.y)};
            if (MASK) {
                pp.x = (c >= lim2) ? 0.0f : pp.x;
                pp.y = (c + 1 >= lim2) ? 0.0f : pp.y;
            }
            if (DIAG) {
                pd[c] = pp.x;
                pd[c + 1] = pp.y;
            }
            acc[(2 * i + e / 2) & 3] = fadd2(acc[(2 * i + e / 2) & 3], pp);
            const f2 q = fadd2(ffma2(pp, f2{127.0f, 127.0f}, f2{0.0f, 0.0f}), f2{kMagicF, kMagicF});
            b[e] = __float_as_uint(q.x);
            b[e + 1] = __float_as_uint(q.y);
        }
        pk[i] = __byte_perm(__byte_perm(b[0], b[1], 0x0040), __byte_perm(b[2], b[3], 0x0040), 0x5410);
    }
    tmem_st16x2_8(ts, pk);
    if (DIAG) count_static_scale_mismatches(reinterpret_cast<const float(&)[32]>(pd), qi < n, first, diag);
    const f2 sum = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
    l = fmaf(l, alpha, sum.x + sum.y);
    return alpha;
}

// KV tiles of query-tile pair `pair` (the longer, tile B, when it exists).
__host__ __device__ __forceinline__ int pair_kv_tiles(int pair, int ntq, int ntk, bool causal) {
    if (!causal) return ntk;
    const bool has_b = 2 * pair + 1 < ntq;
    return min(has_b ? 4 * pair + 4 : 4 * pair + 2, ntk);
}

// First pair whose KV range extends past tile t0 (pair_kv_tiles is nondecreasing in the
// pair index; t0 is below the longest pair's count for every existing chunk).
__host__ __device__ __forceinline__ int split_pmin(int t0, int npair, int ntq, int ntk, bool causal) {
    if (!causal) return 0;
    int pm = min(t0 / 4, npair - 1);
    while (pm > 0 && pair_kv_tiles(pm - 1, ntq, ntk, true) > t0) --pm;
    while (pm < npair - 1 && pair_kv_tiles(pm, ntq, ntk, true) <= t0) ++pm;
    return pm;
}

// One softmax thread's 32 output values of row qi, columns [col, col + 32), to O.
__device__ __forceinline__ void st_global_v8(void* dst, const uint32_t (&w)[8]) {  // one 32-byte store
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst), "r"(w[0]), "r"(w[1]), "r"(w[2]),
                 "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
                 : "memory");
}

template <int D, bool OUT_F32>
__device__ __forceinline__ void store_o32(const AttnParams& p, int unit, int qi, int col, const float (&v)[32]) {
    const size_t off = (static_cast<size_t>(unit) * p.n + qi) * D + col;
    if (p.o_v8) {  // 32-byte stores (O 32-byte aligned): half the store instructions, whole sectors
        if (OUT_F32) {
            float* dst = static_cast<float*>(p.o) + off;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                uint32_t w[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) w[i] = __float_as_uint(v[8 * e + i]);
                st_global_v8(dst + 8 * e, w);
            }
        } else {
            __half* dst = static_cast<__half*>(p.o) + off;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                uint32_t w[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) w[i] = pack_half2(v[16 * e + 2 * i], v[16 * e + 2 * i + 1]);
                st_global_v8(dst + 16 * e, w);
            }
        }
        return;
    }
    if (OUT_F32) {
        float4* dst = reinterpret_cast<float4*>(static_cast<float*>(p.o) + off);
#pragma unroll
        for (int e = 0; e < 8; ++e) dst[e] = make_float4(v[4 * e], v[4 * e + 1], v[4 * e + 2], v[4 * e + 3]);
    } else {
        uint4* dst = reinterpret_cast<uint4*>(static_cast<__half*>(p.o) + off);
#pragma unroll
        for (int e = 0; e < 4; ++e)
            dst[e] = make_uint4(pack_half2(v[8 * e], v[8 * e + 1]), pack_half2(v[8 * e + 2], v[8 * e + 3]),
                                pack_half2(v[8 * e + 4], v[8 * e + 5]), pack_half2(v[8 * e + 6], v[8 * e + 7]));
    }
}

// KV-split epilogue, run by the 16 softmax warps of every chunk CTA of a split pair
// once the chunk's O is final in TMEM (FP16-P~V path only: the INT8 path never splits).
// The pair's chunks count themselves in on a per-pair counter as they finish.  Every
// chunk but the last writes its unnormalised O (against its own row max m, log2 units)
// and (m, l) to the workspace, then bumps a second, "written" counter; the last one waits
// for those writes (its peers are past their compute, so only stores are outstanding),
// resets both counters and merges the peers' partials with its own O read from TMEM:
//   M = max_s m_s,  O = sum_s 2^(m_s - M) O_s / sum_s 2^(m_s - M) l_s
// (the online-softmax identity of attention.hpp:429-443 across chunks).  Partials are
// stored column-group-major ([item][d/4][256 rows] float4) so a warp's accesses coalesce.
template <int D, bool OUT_F32>
__device__ __forceinline__ void split_epilogue(const AttnParams& p, Bars* bars, uint32_t t_o, int unit, int pair,
                                            int npair, int chunk, int nch, int x, int row, int half, int qi,
                                            bool valid, float m, float l) {
    const size_t pair_idx = static_cast<size_t>(unit) * npair + pair;
    int* arrive = p.split_cnt + 2 * pair_idx;
    int* written = arrive + 1;
    const size_t item0 = pair_idx * p.nchunk;
    const int r = x * kBM + row;
    if (!valid || m == -INFINITY) {  // no key of this chunk is visible to the row
        m = -INFINITY;
        l = 0.0f;
    }
    softmax_bar_sync();  // both tiles' O are final
    if (threadIdx.x == 0) bars->split_last = atomicAdd(arrive, 1) == nch - 1;
    softmax_bar_sync();
    const bool last = bars->split_last;
    if (!last) {
        if (half == 0) p.part_ml[(item0 + chunk) * 256 + r] = make_float2(m, l);
        if (valid) {
            float4* po = reinterpret_cast<float4*>(p.part_o) + (item0 + chunk) * (D / 4) * 256 + r;
#pragma unroll 1
            for (int c = 0; c < D / 2; c += 32) {
                uint32_t o[32];
                tmem_ld16x2_32o<D / 2>(t_o + c, o);
                tmem_wait_ld();
                const int g0 = (half * (D / 2) + c) / 4;
#pragma unroll
                for (int e = 0; e < 8; ++e)
                    po[(g0 + e) * 256] = make_float4(__uint_as_float(o[4 * e]), __uint_as_float(o[4 * e + 1]),
                                                     __uint_as_float(o[4 * e + 2]), __uint_as_float(o[4 * e + 3]));
            }
        }
        __threadfence();
        softmax_bar_sync();
        if (threadIdx.x == 0) atomicAdd(written, 1);
        return;
    }
    if (threadIdx.x == 0) {
        while (atomicAdd(written, 0) < nch - 1) __nanosleep(32);
        *arrive = 0;  // ready for the next call
        *written = 0;
        __threadfence();
    }
    softmax_bar_sync();
    // Every term is accumulated in chunk order, the CTA's own chunk in its place, so the
    // result is bit-identical whichever chunk finishes last.
    float mm = m;
    for (int s = 0; s < nch; ++s)
        if (s != chunk) mm = fmaxf(mm, __ldcg(&p.part_ml[(item0 + s) * 256 + r]).x);
    float lsum = 0.0f;
    for (int s = 0; s < nch; ++s) {
        const float2 ml = s == chunk ? make_float2(m, l) : __ldcg(&p.part_ml[(item0 + s) * 256 + r]);
        if (ml.x != -INFINITY) lsum += ex2(ml.x - mm) * ml.y;
    }
    const float inv_l = 1.0f / lsum;
    bool finite = true;
#pragma unroll 1
    for (int c = 0; c < D / 2; c += 32) {
        float v[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = 0.0f;
        const int g0 = (half * (D / 2) + c) / 4;
#pragma unroll 1
        for (int s = 0; s < nch; ++s) {
            if (s == chunk && !valid) continue;  // (warp-uniform) this tile has no O in this chunk
            const float2 ml = s == chunk ? make_float2(m, l) : __ldcg(&p.part_ml[(item0 + s) * 256 + r]);
            // A row with no visible key in chunk s contributes nothing; the TMEM load of the own
            // chunk is warp-collective, so that case weighs its (zero) O by 0 instead of skipping.
            if (s != chunk && ml.x == -INFINITY) continue;
            const float w = ml.x == -INFINITY ? 0.0f : ex2(ml.x - mm);
            uint32_t t[32];  // chunk s's 32 columns: this CTA's own O from TMEM, a peer's from L2
            if (s == chunk) {
                tmem_ld16x2_32o<D / 2>(t_o + c, t);
                tmem_wait_ld();
            } else {
                const float4* src = reinterpret_cast<const float4*>(p.part_o) + (item0 + s) * (D / 4) * 256 + r;
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const float4 q4 = __ldcg(src + (g0 + e) * 256);
                    t[4 * e] = __float_as_uint(q4.x);
                    t[4 * e + 1] = __float_as_uint(q4.y);
                    t[4 * e + 2] = __float_as_uint(q4.z);
                    t[4 * e + 3] = __float_as_uint(q4.w);
                }
            }
#pragma unroll
            for (int e = 0; e < 32; ++e) v[e] = fmaf(w, __uint_as_float(t[e]), v[e]);
        }
#pragma unroll
        for (int e = 0; e < 32; ++e) {
            v[e] *= inv_l;
            finite &= isfinite(v[e]);
        }
        if (qi < p.n) store_o32<D, OUT_F32>(p, unit, qi, half * (D / 2) + c, v);
    }
    if (qi < p.n && !finite) atomicOr(p.status, kStatusOverflow);
}

// Item `it` of the launch's linear item order (the order the hardware block scheduler
// would dispatch the non-persistent grid in).
template <bool CAUSAL, bool DUMP>
__device__ __forceinline__ Item decode_item(const AttnParams& p, int it, int ntq, int ntk, int npair) {
    Item w;
    w.it = it;
    w.chunk = 0;
    if (DUMP) {
        w.unit = p.dump_unit;
        w.pair = p.dump_qtile / 2;
    } else if (p.kv_chunk > 0) {
        // KV split: items are enumerated chunk-major, longest pairs first inside a chunk.
        // Pair work (KV tiles) is nondecreasing in the pair index, so chunk c exists for
        // pairs [split_pmin(c), npair) -- no empty items, no item table.
        int idx = it;
        for (;; ++w.chunk) {
            const int cnt = (npair - split_pmin(w.chunk * p.kv_chunk, npair, ntq, ntk, CAUSAL)) * p.units;
            if (idx < cnt) break;
            idx -= cnt;
        }
        w.unit = idx % p.units;
        w.pair = npair - 1 - idx / p.units;
    } else {
        // Raster: units are taken in groups whose K^/V fit in L2 together (group_units,
        // chosen by the host), so each K^/V tile is fetched from HBM about once and
        // re-read from L2 by every query-tile pair of its unit.  Inside a group the
        // longest pairs go first (causal work grows with the pair index).
        const int gu = p.group_units;
        const int g = it / (gu * npair);
        const int r = it - g * gu * npair;
        const int gsz = min(gu, p.units - g * gu);
        w.unit = g * gu + r % gsz;
        w.pair = npair - 1 - r / gsz;
    }
    w.qt0 = 2 * w.pair;
    w.has_b = w.qt0 + 1 < ntq;
    // Causal: query tile qt (rows < 128(qt+1)) needs KV tiles j with 64j <= 128qt + 127.
    w.nkv_a = CAUSAL ? min(2 * w.qt0 + 2, ntk) : ntk;
    w.nkv_b = w.has_b ? (CAUSAL ? min(2 * w.qt0 + 4, ntk) : ntk) : 0;
    // KV split: this item covers the pair's KV tiles [j0, j0 + kv_chunk); pairs with a
    // single chunk run the unsplit epilogue.  Kernel loops count j from j0 (ring stages,
    // barrier phases); kb / TMA coordinates use j0 + j.
    w.j0 = 0;
    w.nch = 1;
    if (!DUMP && p.kv_chunk > 0) {
        const int nkv_full = max(w.nkv_a, w.nkv_b);
        w.nch = (nkv_full + p.kv_chunk - 1) / p.kv_chunk;
        w.j0 = w.chunk * p.kv_chunk;
        const int j1 = min(nkv_full, w.j0 + p.kv_chunk);
        w.nkv_a = max(0, min(w.nkv_a, j1) - w.j0);
        w.nkv_b = max(0, min(w.nkv_b, j1) - w.j0);
    }
    w.nkv = max(w.nkv_a, w.nkv_b);
    return w;
}

// Consumer side of the item ring: waits for item number n_it of this CTA and returns its
// decoded form in shared memory.  Consumers read its fields in place (volatile: at the point
// of use, so they do not hold registers across the softmax loop) until release_item.
__device__ __forceinline__ const volatile Item* take_item(Bars* bars, int n_it) {
    const int slot = n_it & 1;
    mbar_wait(smem_u32(&bars->item_full[slot]), (n_it >> 1) & 1);
    return &bars->items[slot];
}

// The warp is done with item n_it (one arrival per warp): its slot may be refilled.
__device__ __forceinline__ void release_item(Bars* bars, int n_it, int lane) {
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_u32(&bars->item_empty[n_it & 1]));
}

// Phase parity of S buffer b's (j / NB)-th use in the current item: `ph` holds, per
// buffer, the parity of its uses by earlier items (S tiles index buffers item-locally,
// j % NB, so the unrolled loop keeps compile-time buffer addresses).
__device__ __forceinline__ uint32_t buf_parity(uint32_t ph, int b, int use) { return ((ph >> b) ^ use) & 1u; }

// Advances the per-buffer parities past an item of n S tiles.
template <int NB>
__device__ __forceinline__ uint32_t advance_parity(uint32_t ph, int n) {
#pragma unroll
    for (int b = 0; b < NB; ++b) ph ^= (static_cast<uint32_t>((n + NB - 1 - b) / NB) & 1u) << b;
    return ph;
}

// One work item of a softmax warp (tile x = warp / 8): the online softmax over the item's
// KV tiles, then the epilogue (or the KV-split epilogue).  ph: S-buffer parities (see
// buf_parity); co: earlier items with work for tile x (o_final / o_free phases).
// SPLIT: the item is one chunk of a KV-split pair (split_epilogue).
template <int D, bool CAUSAL, bool OUT_F32, bool DUMP, bool PT, bool VI8, bool SPLIT>
__device__ __forceinline__ void softmax_item(const AttnParams& p, Bars* bars, uint32_t tbase, int warp, int lane,
                                             const volatile Item* wi, uint32_t ph, int co, int n_it) {
    using C = Cfg<D>;
    constexpr int NB = C::kNB;
    const int n = p.n;
    const int ntq = (n + kBM - 1) / kBM;
    const int ntk = (n + kBN - 1) / kBN;
    const int npair = (ntq + 1) / 2;
    const int x = warp / 8;
    const int lane_base = (warp % 4) * 32 + ((warp % 8) / 4) * 16;
    const int half = lane / 16;
    const int row = lane_base + (lane % 16);
    const uint32_t lane_off = static_cast<uint32_t>(lane_base) << 16;
    const uint32_t t_o = tbase + lane_off + C::kOffO + x * D;
    // The item's fields, once into (warp-uniform) registers.
    const int it_unit = __shfl_sync(0xffffffffu, wi->unit, 0);
    const int it_j0 = __shfl_sync(0xffffffffu, wi->j0, 0);
    const int it_qt = __shfl_sync(0xffffffffu, wi->qt0, 0) + x;
#define SAB_UNIT it_unit
#define SAB_J0 it_j0
#define SAB_QT it_qt
#define SAB_QI (it_qt * kBM + row)
    const int nkv_x = __shfl_sync(0xffffffffu, x == 0 ? wi->nkv_a : wi->nkv_b, 0);
    float m = -INFINITY, l = 0.0f;
    if (nkv_x > 0) {
        // Scale rows: per block [units][ntq] / [units][ntk]; per token (T) [units][npad],
        // npad = ntk * 64 (K1 pads each unit's rows so 64-key tiles stay in bounds).
        const int npad = ntk * kBN;
        const float qsl = PT ? (SAB_QI < n ? p.qscales[static_cast<size_t>(SAB_UNIT) * npad + SAB_QI] : 1.0f) * kLog2e
                             : p.qscales[static_cast<size_t>(SAB_UNIT) * ntq + SAB_QT] * kLog2e;
        const float* ksc = p.kscales + static_cast<size_t>(SAB_UNIT) * (PT ? npad : ntk);
        // The K scale of the next KV tile is fetched one iteration ahead.
        float ks_next = PT ? 0.0f : __ldg(ksc + SAB_J0);
        const bool tr = (warp % 8) == 0 && lane == 0;
        // Software pipeline: S(j+1) is loaded from TMEM while P(j) is stored and
        // handed to the MMA issuer, so the load latency is off the per-tile chain.
        uint32_t r[32];
        if (tr) SAB_STAMP(x, 0, 0);
        if (threadIdx.x == 0) SAB_STAMP(4, 400 + n_it, 1);  // per-item timeline (SAB_TRACE builds)
        mbar_wait(smem_u32(&bars->s_full[x][0]), buf_parity(ph, 0, 0));
        tc_fence_after();
        tmem_ld16x2_32(tbase + lane_off + x * (NB * 64), r);
#pragma unroll(PT ? 1 : 2)  // B: compile-time buffer parity per copy (+1-2 %); T would spill
        for (int j = 0; j < nkv_x; ++j) {
            const float ks_cur = ks_next;
            if (!PT && j + 1 < nkv_x) ks_next = __ldg(ksc + SAB_J0 + j + 1);
            const int b = j % NB;
            tmem_wait_ld_dep(r);
            if (tr) SAB_STAMP(x, j, 1);
            const uint32_t t_s = tbase + lane_off + x * (NB * 64) + b * 64;
            int32_t* dump = (DUMP && SAB_QT == p.dump_qtile)
                                ? p.s_dump + (static_cast<size_t>(j) * kBM + row) * kBN + 32 * half
                                : nullptr;
            const int kb = (SAB_J0 + j) * kBN;
            // Dequant factor of this 64-key group: dQ * dK * log2(e), so that p = 2^(s - m).
            const float cg = qsl * ks_cur;
            const bool need_mask = (kb + kBN > n) || (CAUSAL && kb + kBN - 1 > SAB_QT * kBM);
            bool rescale;
            float alpha;
            if (VI8 && PT) {
                const float* dkp = ksc + kb + 32 * half;
                if (p.diag)  // static-scale diagnostics (rare, slow path)
                    alpha = need_mask ? softmax_half_pt_i8<true, CAUSAL, true>(r, t_s, half, qsl, dkp, kb, SAB_QI, n,
                                                                               m, l, rescale, p.diag, SAB_J0 + j == 0)
                                      : softmax_half_pt_i8<false, CAUSAL, true>(r, t_s, half, qsl, dkp, kb, SAB_QI,
                                                                                n, m, l, rescale, p.diag,
                                                                                SAB_J0 + j == 0);
                else if (need_mask)
                    alpha = softmax_half_pt_i8<true, CAUSAL, false>(r, t_s, half, qsl, dkp, kb, SAB_QI, n, m, l,
                                                                    rescale, nullptr, false);
                else
                    alpha = softmax_half_pt_i8<false, CAUSAL, false>(r, t_s, half, qsl, dkp, kb, SAB_QI, n, m, l,
                                                                     rescale, nullptr, false);
            } else if (VI8) {
                if (p.diag)
                    alpha = need_mask ? softmax_half_i8<true, CAUSAL, true>(r, t_s, half, cg, kb, SAB_QI, n, m, l,
                                                                            rescale, p.diag, SAB_J0 + j == 0)
                                      : softmax_half_i8<false, CAUSAL, true>(r, t_s, half, cg, kb, SAB_QI, n, m, l,
                                                                             rescale, p.diag, SAB_J0 + j == 0);
                else if (need_mask)
                    alpha = softmax_half_i8<true, CAUSAL, false>(r, t_s, half, cg, kb, SAB_QI, n, m, l, rescale,
                                                                 nullptr, false);
                else
                    alpha = softmax_half_i8<false, CAUSAL, false>(r, t_s, half, cg, kb, SAB_QI, n, m, l, rescale,
                                                                  nullptr, false);
            } else if (PT) {
                const float* dkp = ksc + kb + 32 * half;
                if (need_mask)
                    alpha = softmax_half_pt<true, CAUSAL, poly_per16<D>()>(r, t_s, half, qsl, dkp, kb, SAB_QI, n,
                                                                           m, l, rescale, dump, j == 0);
                else
                    alpha = softmax_half_pt<false, CAUSAL, poly_per16<D>()>(r, t_s, half, qsl, dkp, kb, SAB_QI, n,
                                                                            m, l, rescale, dump, j == 0);
            } else if (need_mask) {
                alpha = softmax_half<true, CAUSAL, poly_per16<D>(), poly_rot<D>()>(r, t_s, half, cg, kb, SAB_QI, n, m, l, rescale,
                                                                    dump, tr ? x : -1, j);
            } else {
                alpha = softmax_half<false, CAUSAL, poly_per16<D>(), poly_rot<D>()>(r, t_s, half, cg, kb, SAB_QI, n, m, l, rescale,
                                                                     dump, tr ? x : -1, j);
            }
            if (tr) SAB_STAMP(x, j, 2);
            if (rescale && j > 0) {
                // O_x must hold P(j-1)V(j-1) before it is rescaled: PV_x(j-1) has finished
                // accumulating (per-buffer barriers keep the phase unambiguous; PV_x(j-1+NB)
                // needs P from a later step).  Thread halves split O's columns.
                const int pj = j - 1;
                mbar_wait(smem_u32(&bars->pv_done[x][pj % NB]), buf_parity(ph, pj % NB, pj / NB));
                tc_fence_after();
#pragma unroll 1
                for (int c = 0; c < D / 2; c += 32) {
                    uint32_t o[32];
                    tmem_ld16x2_32o<D / 2>(t_o + c, o);
                    tmem_wait_ld();
                    if (VI8) {
                        // INT32 O: O <- rne(alpha * O).  The rounding (<= 0.5 of a code product
                        // per move of the row max) is far below P~'s own 1/254 step.  Done on the
                        // FMA/ALU pipes: y + (2^23 + 2^22) leaves rne(y) in the low mantissa bits
                        // for |y| < 2^22 (alpha <= 1 keeps |y| <= |O|); a chunk holding a larger
                        // value takes the cvt.rni path (XU pipe, shared with the exponentials).
                        float y[32];
                        float ymax = 0.0f;
#pragma unroll
                        for (int e = 0; e < 32; ++e) {
                            y[e] = static_cast<float>(static_cast<int>(o[e])) * alpha;
                            ymax = fmaxf(ymax, fabsf(y[e]));
                        }
                        if (ymax < 4194304.0f) {
#pragma unroll
                            for (int e = 0; e < 32; ++e)
                                o[e] = __float_as_uint(y[e] + kMagicF) - kMagicI;
                        } else {
#pragma unroll
                            for (int e = 0; e < 32; ++e) o[e] = static_cast<uint32_t>(__float2int_rn(y[e]));
                        }
                    } else if (p.pv16) {
                        // Binary16 O: O <- rn16(alpha * O), the reference's snap of the rescaled
                        // accumulator (attention.hpp:450-453).
#pragma unroll
                        for (int e = 0; e < 32; ++e) o[e] = f16acc_put(f16acc_get(o[e]) * alpha);
                    } else {
#pragma unroll
                        for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
                    }
                    tmem_st16x2_32o<D / 2>(t_o + c, o);
                }
            }
            tmem_wait_st();  // P (and rescaled O) are in TMEM
            if (tr) SAB_STAMP(x, j, 3);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&bars->p_full[x][b]));  // one arrival per warp
            if (tr) SAB_STAMP(x, j, 4);
            if (j + 1 < nkv_x) {  // S(j+1) is issued into TMEM registers now; waited at the loop top
                if (tr) SAB_STAMP(x, j + 1, 0);
                const int nj = j + 1;
                mbar_wait(smem_u32(&bars->s_full[x][nj % NB]), buf_parity(ph, nj % NB, nj / NB));
                tc_fence_after();
                tmem_ld16x2_32(tbase + lane_off + x * (NB * 64) + (nj % NB) * 64, r);
            }
        }

        // -------------------------------------------------------- epilogue
        mbar_wait(smem_u32(&bars->o_final[x]), co & 1);
        tc_fence_after();
        if (threadIdx.x == 0) SAB_STAMP(4, kTraceTiles - 1, 3);
        if (threadIdx.x == 0) SAB_STAMP(4, 400 + n_it, 3);
        l += __shfl_xor_sync(0xffffffffu, l, 16);  // the two column halves of the row
        if (!DUMP && !SPLIT && !VI8) {
            // Both column blocks of O come out of TMEM behind one wait; O_x is then released to
            // the next item's first PV (persistent launches) before the normalise-and-store.
            const float inv_l = 1.0f / l;
            bool finite = true;
            uint32_t o[D / 2];
#pragma unroll
            for (int c = 0; c < D / 2; c += 32)
                tmem_ld16x2_32o<D / 2>(t_o + c, *reinterpret_cast<uint32_t(*)[32]>(o + c));
            tmem_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&bars->o_free[x]));
            if (p.pv16) {  // binary16 accumulator cells -> fp32 (an infinite cell is the overflow)
#pragma unroll
                for (int e = 0; e < D / 2; ++e) o[e] = __float_as_uint(f16acc_get(o[e]));
            }
#pragma unroll
            for (int c = 0; c < D / 2; c += 32) {
                float v[32];
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                    finite &= isfinite(__uint_as_float(o[c + e]));
                    v[e] = __uint_as_float(o[c + e]) * inv_l;
                }
                if (SAB_QI < n) store_o32<D, OUT_F32>(p, SAB_UNIT, SAB_QI, half * (D / 2) + c, v);
            }
            if (SAB_QI < n && !finite) atomicOr(p.status, kStatusOverflow);
        } else if (!DUMP && !SPLIT) {  // VI8 (KV-split chunks: split_epilogue below)
            const float inv_l = 1.0f / l;
            bool finite = true;
#pragma unroll 1
            for (int c = 0; c < D / 2; c += 32) {
                uint32_t o[32];
                tmem_ld16x2_32o<D / 2>(t_o + c, o);
                tmem_wait_ld();
                float v[32];
                if (VI8) {
                    // (float(acc) * dP) * dV[c] (attention.hpp:494-495), then 1/l (536-538).
                    const float4* vs4 = reinterpret_cast<const float4*>(
                        p.vscales + static_cast<size_t>(SAB_UNIT) * D + half * (D / 2) + c);
#pragma unroll
                    for (int e4 = 0; e4 < 8; ++e4) {
                        const float4 vs = __ldg(vs4 + e4);
                        const float wv[4] = {vs.x, vs.y, vs.z, vs.w};
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const int e = 4 * e4 + i;
                            v[e] = ((static_cast<float>(static_cast<int>(o[e])) * (1.0f / 127.0f)) * wv[i]) *
                                   inv_l;
                        }
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < 32; ++e) {
                        finite &= isfinite(__uint_as_float(o[e]));
                        v[e] = __uint_as_float(o[e]) * inv_l;
                    }
                }
                if (SAB_QI < n) store_o32<D, OUT_F32>(p, SAB_UNIT, SAB_QI, half * (D / 2) + c, v);
            }
            if (SAB_QI < n && !finite) atomicOr(p.status, kStatusOverflow);
        }
        if (threadIdx.x == 0) SAB_STAMP(4, kTraceTiles - 1, 4);
        if (threadIdx.x == 0) SAB_STAMP(4, 400 + n_it, 4);
    }
    if constexpr (!DUMP && !VI8 && SPLIT)
        split_epilogue<D, OUT_F32>(p, bars, t_o, SAB_UNIT, wi->pair, npair, wi->chunk, wi->nch, x, row, half, SAB_QI,
                                   nkv_x > 0, m, l);
    if (nkv_x > 0 && (DUMP || SPLIT || VI8)) {  // O_x has been read: the next item's first PV may overwrite it
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&bars->o_free[x]));
    }
#undef SAB_UNIT
#undef SAB_J0
#undef SAB_QT
#undef SAB_QI
}


// KSPLIT: the launch has a KV-split plan (kv_chunk > 0).  A separate instantiation: the
// split epilogue's code in the item loop would cost the common kernel its registers.
template <int D, bool CAUSAL, bool OUT_F32, bool DUMP, bool PT, bool VI8, bool KSPLIT>
__global__ void __launch_bounds__(kThreads, 1)
    k2_attention(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                 const __grid_constant__ CUtensorMap tm_v, const AttnParams p) {
    using C = Cfg<D>;
    constexpr int S = C::kStages;
    constexpr int NB = C::kNB;
    static_assert(sizeof(Bars) <= 1024, "barrier block overflows its reservation");
    static_assert(C::kOffO + 2 * D <= 512, "TMEM budget");
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    Bars* bars = reinterpret_cast<Bars*>(smem + C::kOffBar);
    const uint32_t sQ = smem_u32(smem + C::kOffQ);
    const uint32_t sK = smem_u32(smem + C::kOffK);
    const uint32_t sV = smem_u32(smem + C::kOffV);

    // Warp index through a shuffle so the compiler knows it is warp-uniform: the role
    // branches below are then uniform and the MMA issuer's loop state lives in
    // uniform registers (no per-MMA R2UR / election sequences).
    const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x / 32), 0);
    const int lane = threadIdx.x % 32;
    const int n = p.n;
    const int ntq = (n + kBM - 1) / kBM;
    const int ntk = (n + kBN - 1) / kBN;
    const int npair = (ntq + 1) / 2;

    if (threadIdx.x == 0) SAB_STAMP(4, kTraceTiles - 1, 0);  // CTA lifecycle (SAB_TRACE builds)
    {  // constant operands of the bias MMA, written once through the generic proxy
        uint4* bias = reinterpret_cast<uint4*>(smem + C::kOffBiasA);
        const uint4 a2048 = make_uint4(0x68006800u, 0x68006800u, 0x68006800u, 0x68006800u);
        const uint4 b384 = make_uint4(0x5E005E00u, 0x5E005E00u, 0x5E005E00u, 0x5E005E00u);
        for (int i = threadIdx.x; i < (8192 + 4096) / 16; i += kThreads) bias[i] = i < 8192 / 16 ? a2048 : b384;
        fence_proxy_async_smem();  // visible to the tensor core (async proxy)
    }
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&bars->q_full), 1);
        for (int s = 0; s < S; ++s) {
            mbar_init(smem_u32(&bars->kv_full[s]), 1);
            mbar_init(smem_u32(&bars->kv_empty[s]), 1);
        }
        for (int x = 0; x < 2; ++x) {
            for (int b = 0; b < C::kNB; ++b) {
                mbar_init(smem_u32(&bars->s_full[x][b]), 1);
                mbar_init(smem_u32(&bars->p_full[x][b]), 8);  // one arrival per softmax warp
                mbar_init(smem_u32(&bars->pv_done[x][b]), 1);
            }
            mbar_init(smem_u32(&bars->o_final[x]), 1);
            mbar_init(smem_u32(&bars->o_free[x]), 8);  // one arrival per softmax warp of tile x
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(smem_u32(&bars->item_full[i]), 1);
            mbar_init(smem_u32(&bars->item_empty[i]), 17);  // MMA warp + 16 softmax warps
        }
        mbar_init(smem_u32(&bars->q_free), 1);
        fence_barrier_init();
    }
    if (warp == 16) tmem_alloc<512>(smem_u32(&bars->tmem_base));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = bars->tmem_base;
    if (threadIdx.x == 0) SAB_STAMP(4, kTraceTiles - 1, 1);
    // Everything above is independent of K1; Q^/K^/scales/V are read only below.
    griddep_wait();
    if (threadIdx.x == 0) SAB_STAMP(4, kTraceTiles - 1, 2);

    // Work loop.  Every role walks the same sequence of items; barrier phases run on
    // state that continues across items (K^/V ring tiles g, S-buffer parities ph[x], items
    // with work for tile x co[x]), so an item's prologue (Q^ and K^/V loads, the first QK^T
    // MMAs) overlaps the previous item's epilogue.  Non-persistent launches (p.persist 0:
    // one CTA per item) run the loop once.
    const int n_items = DUMP ? 1 : p.items;
    if (warp == 16) {
        // ------------------------------------------------------------ TMA producer + scheduler
        if (lane == 0) {
            tma_prefetch_desc(&tm_q);
            tma_prefetch_desc(&tm_k);
            tma_prefetch_desc(&tm_v);
        }
        int it = DUMP ? 0 : static_cast<int>(blockIdx.x);
        uint32_t g = 0;
        for (int n_it = 0;; ++n_it) {
            const int slot = n_it & 1;
            const Item w = decode_item<CAUSAL, DUMP>(p, it < n_items ? it : 0, ntq, ntk, npair);
            if (lane == 0) {
                if (n_it >= 2) mbar_wait(smem_u32(&bars->item_empty[slot]), ((n_it - 2) >> 1) & 1);
                bars->items[slot] = w;
                bars->items[slot].it = it;
                mbar_arrive(smem_u32(&bars->item_full[slot]));
            }
            __syncwarp();
            if (it >= n_items) break;
            if (lane == 0) {
                if (n_it >= 1) mbar_wait(smem_u32(&bars->q_free), (n_it - 1) & 1);
                mbar_arrive_expect_tx(smem_u32(&bars->q_full), (w.has_b ? 2 : 1) * C::kQBytes);
                tma_load_3d(sQ, &tm_q, smem_u32(&bars->q_full), 0, w.qt0 * kBM, w.unit);
                if (w.has_b)
                    tma_load_3d(sQ + C::kQBytes, &tm_q, smem_u32(&bars->q_full), 0, (w.qt0 + 1) * kBM, w.unit);
                for (int j = 0; j < w.nkv; ++j, ++g) {
                    const int s = g % S;
                    const uint32_t ph = (g / S) & 1;
                    SAB_STAMP(4, j, 0);
                    mbar_wait(smem_u32(&bars->kv_empty[s]), ph ^ 1);
                    SAB_STAMP(4, j, 1);
                    const uint32_t full = smem_u32(&bars->kv_full[s]);
#ifdef SAB_SK_NOKV  // timing skeleton: K^/V loaded for the first ring fill only (wrong results)
                    if (g >= S) {
                        mbar_arrive(full);
                        continue;
                    }
#endif
                    mbar_arrive_expect_tx(full, C::kKBytes + (VI8 ? kBN * D : C::kVBytes));
                    const int key0 = (w.j0 + j) * kBN;
                    tma_load_3d(sK + s * C::kKBytes, &tm_k, full, 0, key0, w.unit);
                    if (VI8) {  // V^ transposed: D channel rows of 64 key codes (K-major B operand)
                        tma_load_3d(sV + s * C::kVBytes, &tm_v, full, key0, 0, w.unit);
                    } else {
#pragma unroll
                        for (int c = 0; c < D / 64; ++c)
                            tma_load_3d(sV + s * C::kVBytes + c * C::kVChunk, &tm_v, full, c * 64, key0, w.unit);
                    }
                }
                // Next item: dynamic (an atomic counter after the first, static item per CTA)
                // when persistent; the loop ends after one item otherwise.
                it = (!DUMP && p.persist) ? atomicAdd(p.sched, 1) + static_cast<int>(gridDim.x) : n_items;
            } else {
                g += w.nkv;
            }
            it = __shfl_sync(0xffffffffu, it, 0);
        }
        if (!DUMP && p.persist && lane == 0) {
            // The last CTA out resets the scheduler for the next launch on this workspace.
            __threadfence();
            if (atomicAdd(p.sched + 1, 1) == static_cast<int>(gridDim.x) - 1) {
                p.sched[0] = 0;
                p.sched[1] = 0;
                __threadfence();
            }
        }
        __syncwarp();
    } else if (warp == 17) {
        // ------------------------------------------------------------ MMA issuer (both tiles)
        // The whole warp runs the loop (uniform operands); one elected lane issues.  Per KV
        // tile j: PV_A(j), QK_A(j+2), PV_B(j), QK_B(j+2) -- one K^/V wait per tile for both
        // query tiles, and the two tiles' softmax phases interleave on the tensor pipe.
        constexpr uint32_t idesc_qk = make_idesc(2 /*S32*/, 1 /*S8*/, 1 /*S8*/, 0, 0, kBM, kBN);
        // P~V accumulator: F32 (SAB_PV_FP32), or F16 (SAB_PV_FP16, the paper's mma f16.f16.f16).
        const uint32_t idesc_pv = p.pv16 ? make_idesc(0 /*F16*/, 0 /*F16*/, 0 /*F16*/, 0, 1 /*V MN-major*/, kBM, D)
                                         : make_idesc(1 /*F32*/, 0 /*F16*/, 0 /*F16*/, 0, 1 /*V MN-major*/, kBM, D);
        // Descriptors are advanced by adding (byte offset >> 4) to the start-address field.
        const uint64_t dq0 = make_smem_desc(sQ, 16, C::kSboQK, C::kSwizzleQK);
        const uint64_t dk0 = make_smem_desc(sK, 16, C::kSboQK, C::kSwizzleQK);
        const uint64_t dv0 = VI8 ? make_smem_desc(sV, 16, 8 * 64, kSwizzle64B)
                                 : make_smem_desc(sV, C::kVChunk, 1024, kSwizzle128B);
        constexpr uint32_t idesc_pv8 = make_idesc(2 /*S32*/, 1 /*S8*/, 1 /*S8*/, 0, 0, kBM, D);
        constexpr uint32_t idesc_bias = make_idesc(1 /*F32*/, 0 /*F16*/, 0 /*F16*/, 0, 0, kBM, kBN);
        const uint64_t d_bias_a = make_smem_desc(smem_u32(smem + C::kOffBiasA), 128, 256, kSwizzleNone);
        const uint64_t d_bias_b = make_smem_desc(smem_u32(smem + C::kOffBiasB), 128, 256, kSwizzleNone);
        uint32_t g = 0;
        uint32_t ph[2] = {0u, 0u};
        int co[2] = {0, 0};
        for (int n_it = 0;; ++n_it) {
            const volatile Item* wi = take_item(bars, n_it);
            // Broadcast through a shuffle so the compiler knows the loop state is warp-uniform
            // (uniform registers: no per-MMA R2UR sequences).
            if (__shfl_sync(0xffffffffu, wi->it, 0) >= n_items) break;
            const int nkv_a = __shfl_sync(0xffffffffu, wi->nkv_a, 0);
            const int nkv_b = __shfl_sync(0xffffffffu, wi->nkv_b, 0);
            const int nkv = max(nkv_a, nkv_b);
            mbar_wait(smem_u32(&bars->q_full), n_it & 1);
            // QK_x(j) into S_x[j % NB].  Issued after PV_x(j-2), which read P_x(j-2)
            // from that buffer (tcgen05 ops of one thread execute in issue order).
            auto issue_qk = [&](int x, int j) {
                const int s = (g + j) % S;
                const uint64_t dq = dq0 + static_cast<uint64_t>((x * C::kQBytes) >> 4);
                const uint64_t dk = dk0 + static_cast<uint64_t>((s * C::kKBytes) >> 4);
                const int sb = j % NB;
                const uint32_t t_s = tbase + x * (NB * 64) + sb * 64;
                if (elect_one()) {
                    // Bias MMA: S = 2^23 + 2^22 as binary32 (bits 0x4B400000) from constant fp16
                    // operands, then the INT32 QK^T products accumulate onto those bits, so the
                    // softmax reads float(2^23 + 2^22 + acc) directly.
#ifndef SAB_SK_NOBIAS  // timing skeleton: no bias MMA (wrong results)
                    umma_f16_ss(t_s, d_bias_a, d_bias_b, idesc_bias, 0u);
#endif
#pragma unroll
                    for (int kk = 0; kk < D / 32; ++kk)
                        umma_i8_ss(t_s, dq + static_cast<uint64_t>(kk * 2), dk + static_cast<uint64_t>(kk * 2),
                                   idesc_qk,
#ifdef SAB_SK_NOBIAS
                                   kk > 0 ? 1u : 0u);
#else
                                   1u);
#endif
                    umma_commit(smem_u32(&bars->s_full[x][sb]));
                }
                __syncwarp();
            };
            auto wait_kv = [&](int j) {
                if (lane == 0) SAB_STAMP(2, j, 0);
                mbar_wait(smem_u32(&bars->kv_full[(g + j) % S]), ((g + j) / S) & 1);
                tc_fence_after();
                if (lane == 0) SAB_STAMP(2, j, 1);
            };
            // Q^ is free for the next item once the item's last QK^T MMA has completed.
            auto release_q = [&]() {
                if (elect_one()) umma_commit(smem_u32(&bars->q_free));
                __syncwarp();
            };
            for (int j = 0; j < NB && j < nkv; ++j) {
                wait_kv(j);
                if (j < nkv_a) issue_qk(0, j);
                if (j < nkv_b) issue_qk(1, j);
            }
            if (nkv <= NB) release_q();
            for (int j = 0; j < nkv; ++j) {
                const int s = (g + j) % S;
                const bool next = j + NB < nkv;
                if (next) wait_kv(j + NB);
#pragma unroll
                for (int x = 0; x < 2; ++x) {
                    const int nkv_x = x == 0 ? nkv_a : nkv_b;
                    if (j < nkv_x) {  // O_x += P_x(j) V(j), P from TMEM
                        const int sb = j % NB;
                        if (j == 0 && co[x] > 0) {  // the previous item's epilogue has read O_x
                            mbar_wait(smem_u32(&bars->o_free[x]), (co[x] - 1) & 1);
                            tc_fence_after();
                        }
                        if (lane == 0) SAB_STAMP(2 + x, j, 3);
                        mbar_wait(smem_u32(&bars->p_full[x][sb]), buf_parity(ph[x], sb, j / NB));
                        tc_fence_after();
                        if (lane == 0) SAB_STAMP(2 + x, j, 4);
                        const uint64_t dv = dv0 + static_cast<uint64_t>((s * C::kVBytes) >> 4);
                        const uint32_t t_p = tbase + x * (NB * 64) + sb * 64;
                        const uint32_t t_o = tbase + C::kOffO + x * D;
                        if (elect_one()) {
                            if (VI8) {  // INT32 O_x += P~^(j) V^(j): 2 x K=32 codes, P~^ from TMEM
#pragma unroll
                                for (int kk = 0; kk < kBN / 32; ++kk)
                                    umma_i8_ts(t_o, t_p + kk * 8, dv + static_cast<uint64_t>(kk * 2), idesc_pv8,
                                               (j > 0 || kk > 0) ? 1u : 0u);
                            } else {
#pragma unroll
                                for (int kk = 0; kk < kBN / 16; ++kk)
                                    umma_f16_ts(t_o, t_p + kk * 8, dv + static_cast<uint64_t>(kk * (2048 >> 4)),
                                                idesc_pv, (j > 0 || kk > 0) ? 1u : 0u);
                            }
                            umma_commit(smem_u32(&bars->pv_done[x][sb]));
                            if (j == nkv_x - 1) umma_commit(smem_u32(&bars->o_final[x]));
                        }
                        __syncwarp();
                        if (lane == 0) SAB_STAMP(2 + x, j, 5);
                    }
                    if (next && j + NB < nkv_x) issue_qk(x, j + NB);
                }
                if (next && j + NB == nkv - 1) release_q();
                if (elect_one()) umma_commit(smem_u32(&bars->kv_empty[s]));  // K^(j), V(j) free once these MMAs finish
                __syncwarp();
            }
            release_item(bars, n_it, lane);
            g += nkv;
            for (int x = 0; x < 2; ++x) {
                const int nkv_x = x == 0 ? nkv_a : nkv_b;
                ph[x] = advance_parity<NB>(ph[x], nkv_x);
                co[x] += nkv_x > 0;
            }
        }
        __syncwarp();
    } else if (warp < 16) {
        // ------------------------------------------------------------ softmax warpgroups
        // Tile x = warp / 8.  Warp w covers TMEM lanes [32(w%4) + 16((w%8)/4), +16); its
        // threads t and t+16 share one query row (t % 16) and split the columns.
        const int x = warp / 8;
        uint32_t ph = 0u;
        int co = 0;
        for (int n_it = 0;; ++n_it) {
            const volatile Item* wi = take_item(bars, n_it);
            if (__shfl_sync(0xffffffffu, wi->it, 0) >= n_items) break;
            const int nkv_x = __shfl_sync(0xffffffffu, x == 0 ? wi->nkv_a : wi->nkv_b, 0);
            if (threadIdx.x == 0) SAB_STAMP(4, 400 + n_it, 0);
            if (KSPLIT && wi->nch > 1)
                softmax_item<D, CAUSAL, OUT_F32, false, PT, false, true>(p, bars, tbase, warp, lane, wi, ph, co, n_it);
            else
                softmax_item<D, CAUSAL, OUT_F32, DUMP, PT, VI8, false>(p, bars, tbase, warp, lane, wi, ph, co, n_it);
            if (threadIdx.x == 0) SAB_STAMP(4, 400 + n_it, 5);
            release_item(bars, n_it, lane);
            ph = advance_parity<C::kNB>(ph, nkv_x);
            co += nkv_x > 0;
        }
    }

    if (threadIdx.x == 0) SAB_STAMP(4, kTraceTiles - 1, 5);
    tc_fence_before();
    __syncthreads();
    if (warp == 16) {
        tc_fence_after();
        tmem_dealloc<512>(tbase);
        if (lane == 0) SAB_STAMP(4, kTraceTiles - 1, 6);
    }
}

// ------------------------------------------------------------------ host side
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn get_encode() {
    static EncodeFn fn = [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return static_cast<EncodeFn>(nullptr);
        return reinterpret_cast<EncodeFn>(ptr);
    }();
    return fn;
}

// (inner=d, tokens, units) tensor map with a (box_x, box_y, 1) box.
bool make_map(CUtensorMap* tm, const void* base, CUtensorMapDataType dt, int elem, int d, int n, int units, int box_x,
              int box_y, CUtensorMapSwizzle sw) {
    EncodeFn enc = get_encode();
    if (!enc) return false;
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(n), static_cast<cuuint64_t>(units)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(d) * elem, static_cast<cuuint64_t>(d) * n * elem};
    const cuuint32_t box[3] = {static_cast<cuuint32_t>(box_x), static_cast<cuuint32_t>(box_y), 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    return enc(tm, dt, 3, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// SMs of the current device (one persistent K2 CTA each).
int sm_count() {
    int dev = 0, n = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
}

// SAB_K2_PERSIST: unset -> heuristic (launch_k2), 0 -> never, 1 -> always.
int k2_persist_mode() {
    static const int mode = [] {
        const char* e = std::getenv("SAB_K2_PERSIST");
        return e ? (e[0] == '0' ? 0 : 1) : -1;
    }();
    return mode;
}

// Raster groups: as few groups as keep each group's K^ (int8) and V (fp16) within
// ~32 MB of the 126 MB L2, balanced in size (24-48 MB measured best on C2 and C4;
// scripts/rounds/r01/l2sweep.sh).
int raster_group_units(const AttnParams& p, int d) {
    static const size_t budget = [] {  // SAB_L2_GROUP_MB overrides the default (tuning)
        const char* e = std::getenv("SAB_L2_GROUP_MB");
        const long mb = e ? std::atol(e) : 32;
        return static_cast<size_t>(mb > 0 ? mb : 32) << 20;
    }();
    const size_t kv_unit = static_cast<size_t>(p.n) * d * 3;
    const size_t per_group = std::max<size_t>(1, budget / kv_unit);
    const size_t groups = (static_cast<size_t>(p.units) + per_group - 1) / per_group;
    return static_cast<int>((static_cast<size_t>(p.units) + groups - 1) / groups);
}

template <int D, bool CAUSAL, bool OUT_F32, bool DUMP, bool PT, bool VI8, bool KSPLIT>
cudaError_t launch_k2_split(const AttnParams& p, cudaStream_t s) {
    using C = Cfg<D>;
    CUtensorMap tq, tk, tv;
    const CUtensorMapSwizzle swqk = D == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
    if (!make_map(&tq, p.qcodes, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, D, p.n, p.units, D, kBM, swqk) ||
        !make_map(&tk, p.kcodes, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, D, p.n, p.units, D, kBN, swqk) ||
        !(VI8 ? make_map(&tv, p.vcodes, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, p.ldv, D, p.units, kBN, D,
                         CU_TENSOR_MAP_SWIZZLE_64B)
              : make_map(&tv, p.v16, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, D, p.n, p.units, 64, kBN,
                         CU_TENSOR_MAP_SWIZZLE_128B)))
        return cudaErrorInvalidValue;
    AttnParams pp = p;
    pp.group_units = raster_group_units(p, D);
    auto kern = k2_attention<D, CAUSAL, OUT_F32, DUMP, PT, VI8, KSPLIT>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    if (e != cudaSuccess) return e;
    const int ntq = (p.n + kBM - 1) / kBM;
    const int npair = (ntq + 1) / 2, ntk = (p.n + kBN - 1) / kBN;
    long long items = DUMP ? 1 : static_cast<long long>(npair) * p.units;
    if (!DUMP && p.kv_chunk > 0) {  // one item per (unit, pair, chunk)
        items = 0;
        for (int c = 0; c < p.nchunk; ++c)
            items += static_cast<long long>(npair - split_pmin(c * p.kv_chunk, npair, ntq, ntk, CAUSAL)) * p.units;
    }
    pp.items = static_cast<int>(items);
    // Persistent (one CTA per SM walks the items, the next item's Q^/K^/V loads and first
    // QK^T MMAs overlapping the current item's epilogue) where the per-item fixed cost
    // matters: causal grids (uneven items, C2 +2.5 %) and short ones (<= 8 items per SM:
    // C4 N=1K +11..19 %).  Long uniform grids (C3, C4 N>=4K non-causal) measured 1-2 %
    // faster with one CTA per item.  SAB_K2_PERSIST=0 / 1 forces either.
    const int sms = sm_count();
    const int mode = k2_persist_mode();
    pp.persist = !DUMP && items > sms && (mode == 1 || (mode < 0 && (CAUSAL || items <= 8LL * sms)));
    const unsigned grid = static_cast<unsigned>(pp.persist ? sms : items);
#ifdef SAB_TRACE
    cudaMemcpyToSymbolAsync(g_trace, &h_trace_ptr, sizeof(h_trace_ptr), 0, cudaMemcpyHostToDevice, s);
    cudaMemcpyToSymbolAsync(g_trace_cta, &h_trace_cta, sizeof(int), 0, cudaMemcpyHostToDevice, s);
#endif
    return launch_pdl(kern, dim3(grid), dim3(kThreads), C::kSmemBytes, s, tq, tk, tv, pp);
}

template <int D, bool CAUSAL, bool OUT_F32, bool DUMP, bool PT, bool VI8>
cudaError_t launch_k2(const AttnParams& p, cudaStream_t s) {
    if constexpr (!DUMP && !VI8)  // the INT8 P~V path and the INT32 dump never split
        if (p.kv_chunk > 0) return launch_k2_split<D, CAUSAL, OUT_F32, DUMP, PT, VI8, true>(p, s);
    return launch_k2_split<D, CAUSAL, OUT_F32, DUMP, PT, VI8, false>(p, s);
}

template <bool DUMP, bool PT, bool VI8 = false>
cudaError_t dispatch_pt(const AttnParams& p, cudaStream_t s) {
    const bool c = p.causal != 0, f = p.out_f32 != 0;
    if (p.d == 128) {
        if (c)
            return f ? launch_k2<128, true, true, DUMP, PT, VI8>(p, s) : launch_k2<128, true, false, DUMP, PT, VI8>(p, s);
        return f ? launch_k2<128, false, true, DUMP, PT, VI8>(p, s) : launch_k2<128, false, false, DUMP, PT, VI8>(p, s);
    }
    if (p.d == 64) {
        if (c)
            return f ? launch_k2<64, true, true, DUMP, PT, VI8>(p, s) : launch_k2<64, true, false, DUMP, PT, VI8>(p, s);
        return f ? launch_k2<64, false, true, DUMP, PT, VI8>(p, s) : launch_k2<64, false, false, DUMP, PT, VI8>(p, s);
    }
    return cudaErrorInvalidValue;
}

// The INT32 S dump does not read the scales, so it only needs the per-block build.
template <bool DUMP>
cudaError_t dispatch(const AttnParams& p, cudaStream_t s) {
    if (!DUMP && p.vcodes)  // SAGEAttn-vT / -vB
        return p.per_token ? dispatch_pt<false, true, true>(p, s) : dispatch_pt<false, false, true>(p, s);
    if (!DUMP && p.per_token) return dispatch_pt<false, true>(p, s);
    return dispatch_pt<DUMP, false>(p, s);
}

}  // namespace

// KV-split plan.  K2 runs one CTA per (unit, query-tile pair); a pair's work is its KV
// tile count (all ntk tiles, or min(4p+4, ntk) when causal).  When the longest pair is
// well above the average work per SM -- few units per device under K3 sharding (C2 on
// 8 GPUs: 4 units = 128 CTAs, longest pair 128 tiles vs 57 per SM), or short sequences --
// the block scheduler cannot balance the grid, so pairs longer than about the per-SM
// work are cut into chunks of that length (at least 16 tiles, at most 32 chunks).
// SAB_KV_SPLIT=<tiles> forces a chunk length (tests), SAB_KV_SPLIT=0 disables the split.
void kv_split_plan(int64_t units, int n, int causal, int* kv_chunk, int* nchunk) {
    static const int forced = [] {
        const char* e = std::getenv("SAB_KV_SPLIT");
        return e ? std::atoi(e) : -1;
    }();
    constexpr int kSms = 148;  // B200
    *kv_chunk = 0;
    *nchunk = 1;
    if (forced == 0 || units < 1 || n < 1) return;
    const int ntq = (n + kBM - 1) / kBM, ntk = (n + kBN - 1) / kBN, npair = (ntq + 1) / 2;
    int64_t per_unit = 0;
    int longest = 0;
    for (int pr = 0; pr < npair; ++pr) {
        const int len = pair_kv_tiles(pr, ntq, ntk, causal != 0);
        per_unit += len;
        longest = std::max(longest, len);
    }
    const double per_sm = static_cast<double>(per_unit) * static_cast<double>(units) / kSms;
    int len;
    if (forced > 0) {
        len = forced;
    } else {
        // Cut the longest pairs to about the per-SM work: chunks cost a CTA prologue and a
        // partial write each, so as few as balance needs (C2's 4-unit shard: 2 x 64 tiles).
        if (longest <= 1.15 * per_sm) return;
        const int nch = static_cast<int>(std::ceil(longest / std::max(16.0, 1.15 * per_sm)));
        if (nch < 2) return;
        len = (longest + nch - 1) / nch;
    }
    if (len >= longest) return;
    int nch = (longest + len - 1) / len;
    if (nch > 32) {
        nch = 32;
        len = (longest + 31) / 32;
        nch = (longest + len - 1) / len;
    }
    *kv_chunk = len;
    *nchunk = nch;
}

cudaError_t launch_attention(const AttnParams& p, cudaStream_t s) { return dispatch<false>(p, s); }

cudaError_t launch_qk_dump(const AttnParams& p, cudaStream_t s) {
    AttnParams q = p;
    q.out_f32 = 1;
    return dispatch<true>(q, s);
}

}  // namespace sab

#ifdef SAB_TRACE
extern "C" void sab_debug_set_trace(void* dev_buf, int cta) {
    sab::h_trace_ptr = static_cast<long long*>(dev_buf);
    sab::h_trace_cta = cta;
}
#endif
