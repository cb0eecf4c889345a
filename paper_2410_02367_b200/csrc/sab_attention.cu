// sab_attention.cu -- K2, the SageAttn-B attention kernel for sm_100a.
//
// Replaces the q-block / kv-block engine of attention.hpp:383-541:
//   detail::int8_tile_nt (265-279)          -> tcgen05.mma kind::i8, INT32 accumulators in TMEM
//   s = (float(acc) * dQ) * dK (409-414)    -> one FMUL per element with dQ*dK*log2(e)
//   causal tile classes (79-94, 399-427)    -> fully masked KV tiles never issued; element
//                                              mask only on the diagonal / ragged tail tile
//   online softmax (429-443)                -> registers, one thread per query row, exp2 on MUFU
//   P~ V with binary16 operands (447-475)   -> P packed to fp16 into TMEM (aliasing S),
//                                              tcgen05.mma kind::f16 with A from TMEM, V from SMEM,
//                                              FP32 accumulator in TMEM (the pv_fp32_accumulator arm)
//   O = diag(l)^-1 O + overflow check (524-540) -> epilogue from TMEM, status word on non-finite O
//
// One CTA = one (unit, 128-query tile).  Warp roles (192 threads):
//   warps 0-3  softmax + epilogue (thread i owns query row i = TMEM lane i)
//   warp  4    TMA producer (Q^ once; K^ and V per 128-key tile, STAGES-deep ring)
//   warp  5    MMA issuer (single thread): QK^T(j) into S[j%2], then P(j-1)V(j-1) into O
// TMEM (512 columns): S0 [0,128), S1 [128,256) int32; P(j) fp16x2 over S[j%2] [0,64);
//                      O [256, 256+D) fp32.
// Rescaling of O is lazy (only when a row max grows by more than 2^8), which
// is exact in real arithmetic because l and O share the stale max.
#include <cuda.h>
#include <cuda_fp16.h>

#include "sab_internal.h"
#include "sab_ptx.cuh"

namespace sab {
namespace {

constexpr int kBM = 128;
constexpr int kBN = kTileN;
constexpr int kThreads = 192;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescaleThreshold = 8.0f;  // log2 units

template <int D>
struct Cfg {
    static constexpr int kStages = D == 128 ? 3 : 4;
    static constexpr int kQBytes = kBM * D;
    static constexpr int kKBytes = kBN * D;
    static constexpr int kVBytes = kBN * D * 2;
    static constexpr int kVChunk = kBN * 64 * 2;  // one 64-column SW128 panel of V
    static constexpr uint32_t kSwizzleQK = D == 128 ? kSwizzle128B : kSwizzle64B;
    static constexpr uint32_t kSboQK = 8 * D;     // 8 rows of D int8
    static constexpr int kOffQ = 0;
    static constexpr int kOffK = kOffQ + kQBytes;
    static constexpr int kOffV = kOffK + kStages * kKBytes;
    static constexpr int kOffBar = kOffV + kStages * kVBytes;
    static constexpr int kSmemBytes = kOffBar + 256 + 1024;  // barriers + alignment slack
};

struct Bars {
    uint64_t q_full;
    uint64_t k_full[4], k_empty[4], v_full[4], v_empty[4];
    uint64_t s_full[2], p_full[2];
    uint64_t pv_done, o_final;
    uint32_t tmem_base;
};

template <int D, bool CAUSAL, bool OUT_F32, bool DUMP>
__global__ void __launch_bounds__(kThreads, 1)
    k2_attention(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                 const __grid_constant__ CUtensorMap tm_v, const AttnParams p) {
    using C = Cfg<D>;
    constexpr int S = C::kStages;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    Bars* bars = reinterpret_cast<Bars*>(smem + C::kOffBar);
    const uint32_t sQ = smem_u32(smem + C::kOffQ);
    const uint32_t sK = smem_u32(smem + C::kOffK);
    const uint32_t sV = smem_u32(smem + C::kOffV);

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const int n = p.n;
    const int ntq = (n + kBM - 1) / kBM;
    const int ntk = (n + kBN - 1) / kBN;
    const int ngk = (n + kBlockKV - 1) / kBlockKV;

    int unit, qt;
    if (DUMP) {
        unit = p.dump_unit;
        qt = p.dump_qtile;
    } else {  // longest query tiles first (causal work grows with qt)
        unit = blockIdx.x % p.units;
        qt = ntq - 1 - static_cast<int>(blockIdx.x / p.units);
    }
    const int nkv = CAUSAL ? min(qt + 1, ntk) : ntk;

    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&bars->q_full), 1);
        for (int s = 0; s < S; ++s) {
            mbar_init(smem_u32(&bars->k_full[s]), 1);
            mbar_init(smem_u32(&bars->k_empty[s]), 1);
            mbar_init(smem_u32(&bars->v_full[s]), 1);
            mbar_init(smem_u32(&bars->v_empty[s]), 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(smem_u32(&bars->s_full[b]), 1);
            mbar_init(smem_u32(&bars->p_full[b]), 128);
        }
        mbar_init(smem_u32(&bars->pv_done), 1);
        mbar_init(smem_u32(&bars->o_final), 1);
        fence_barrier_init();
    }
    if (warp == 4) tmem_alloc<512>(smem_u32(&bars->tmem_base));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = bars->tmem_base;
    const uint32_t tO = tbase + 256;

    if (warp == 4) {
        // ------------------------------------------------------------ TMA producer
        if (lane == 0) {
            tma_prefetch_desc(&tm_q);
            tma_prefetch_desc(&tm_k);
            tma_prefetch_desc(&tm_v);
            mbar_arrive_expect_tx(smem_u32(&bars->q_full), C::kQBytes);
            tma_load_3d(sQ, &tm_q, smem_u32(&bars->q_full), 0, qt * kBM, unit);
            for (int j = 0; j < nkv; ++j) {
                const int s = j % S;
                const uint32_t ph = (j / S) & 1;
                mbar_wait(smem_u32(&bars->k_empty[s]), ph ^ 1);
                mbar_arrive_expect_tx(smem_u32(&bars->k_full[s]), C::kKBytes);
                tma_load_3d(sK + s * C::kKBytes, &tm_k, smem_u32(&bars->k_full[s]), 0, j * kBN, unit);
                mbar_wait(smem_u32(&bars->v_empty[s]), ph ^ 1);
                mbar_arrive_expect_tx(smem_u32(&bars->v_full[s]), C::kVBytes);
#pragma unroll
                for (int c = 0; c < D / 64; ++c)
                    tma_load_3d(sV + s * C::kVBytes + c * C::kVChunk, &tm_v, smem_u32(&bars->v_full[s]), c * 64,
                                j * kBN, unit);
            }
        }
        __syncwarp();
    } else if (warp == 5) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            constexpr uint32_t idesc_qk = make_idesc(2 /*S32*/, 1 /*S8*/, 1 /*S8*/, 0, 0, kBM, kBN);
            constexpr uint32_t idesc_pv = make_idesc(1 /*F32*/, 0 /*F16*/, 0 /*F16*/, 0, 1 /*V MN-major*/, kBM, D);
            mbar_wait(smem_u32(&bars->q_full), 0);
            tc_fence_after();
            for (int j = 0; j <= nkv; ++j) {
                if (j < nkv) {
                    const int s = j % S;
                    mbar_wait(smem_u32(&bars->k_full[s]), (j / S) & 1);
                    tc_fence_after();
                    const uint32_t d_tmem = tbase + (j & 1) * 128;
#pragma unroll
                    for (int kk = 0; kk < D / 32; ++kk) {
                        const uint64_t a = make_smem_desc(sQ + kk * 32, 16, C::kSboQK, C::kSwizzleQK);
                        const uint64_t b = make_smem_desc(sK + s * C::kKBytes + kk * 32, 16, C::kSboQK, C::kSwizzleQK);
                        umma_i8_ss(d_tmem, a, b, idesc_qk, kk > 0);
                    }
                    umma_commit(smem_u32(&bars->k_empty[s]));
                    umma_commit(smem_u32(&bars->s_full[j & 1]));
                }
                if (j >= 1) {
                    const int jp = j - 1;
                    const int sp = jp % S;
                    mbar_wait(smem_u32(&bars->p_full[jp & 1]), (jp >> 1) & 1);
                    mbar_wait(smem_u32(&bars->v_full[sp]), (jp / S) & 1);
                    tc_fence_after();
                    const uint32_t p_tmem = tbase + (jp & 1) * 128;
#pragma unroll
                    for (int kk = 0; kk < kBN / 16; ++kk) {
                        const uint64_t b =
                            make_smem_desc(sV + sp * C::kVBytes + kk * 2048, C::kVChunk, 1024, kSwizzle128B);
                        umma_f16_ts(tO, p_tmem + kk * 8, b, idesc_pv, (jp > 0 || kk > 0) ? 1u : 0u);
                    }
                    umma_commit(smem_u32(&bars->v_empty[sp]));
                    umma_commit(smem_u32(&bars->pv_done));
                    if (jp == nkv - 1) umma_commit(smem_u32(&bars->o_final));
                }
            }
        }
        __syncwarp();
    } else {
        // ------------------------------------------------------------ softmax warps 0-3
        const int row = warp * 32 + lane;
        const uint32_t trow = tbase + (static_cast<uint32_t>(warp * 32) << 16);
        const int qi = qt * kBM + row;
        const float qsl = p.qscales[static_cast<size_t>(unit) * ntq + qt] * kLog2e;
        const float* ksc = p.kscales + static_cast<size_t>(unit) * ngk;
        float m = -INFINITY, l = 0.0f;

        for (int j = 0; j < nkv; ++j) {
            const int sb = j & 1;
            mbar_wait(smem_u32(&bars->s_full[sb]), (j >> 1) & 1);
            tc_fence_after();
            uint32_t sr[kBN];
#pragma unroll
            for (int c = 0; c < kBN / 32; ++c) tmem_ld32(trow + sb * 128 + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[c * 32]));
            tmem_wait_ld();

            if (DUMP) {
                int32_t* dst = p.s_dump + (static_cast<size_t>(j) * kBM + row) * kBN;
#pragma unroll
                for (int c = 0; c < kBN; c += 4)
                    *reinterpret_cast<int4*>(dst + c) = make_int4(sr[c], sr[c + 1], sr[c + 2], sr[c + 3]);
            }

            const int kb = j * kBN;
            const int g0 = 2 * j;
            const float c0 = qsl * ksc[g0];
            const float c1 = (g0 + 1 < ngk) ? qsl * ksc[g0 + 1] : 0.0f;
            float x[kBN];
#pragma unroll
            for (int c = 0; c < kBN; ++c) x[c] = static_cast<float>(static_cast<int32_t>(sr[c])) * (c < 64 ? c0 : c1);
            const bool need_mask = (kb + kBN > n) || (CAUSAL && kb + kBN - 1 > qt * kBM);
            if (need_mask) {
#pragma unroll
                for (int c = 0; c < kBN; ++c) {
                    const int key = kb + c;
                    if (key >= n || (CAUSAL && key > qi)) x[c] = -INFINITY;
                }
            }
            float mx = x[0];
#pragma unroll
            for (int c = 1; c < kBN; ++c) mx = fmaxf(mx, x[c]);
            const float m_new = fmaxf(m, mx);
            const bool rescale = __any_sync(0xffffffffu, m_new > m + kRescaleThreshold);
            float mu = m, alpha = 1.0f;
            if (rescale) {
                mu = m_new;
                alpha = ex2(m - m_new);
            }
            const float mref = (mu == -INFINITY) ? 0.0f : mu;
            float sum = 0.0f;
            uint32_t pk[kBN / 2];
#pragma unroll
            for (int c = 0; c < kBN; c += 2) {
                const float p0 = ex2(x[c] - mref);
                const float p1 = ex2(x[c + 1] - mref);
                sum += p0 + p1;
                pk[c / 2] = pack_half2(p0, p1);
            }
            l = l * alpha + sum;
            m = mu;

            if (rescale && j > 0) {
                // O must hold P(j-1)V(j-1) before it is rescaled; PV(j-2) is already
                // complete (it precedes QK(j) in the tcgen05 pipe), so the pv_done phase
                // counter is j-1 or j here and parity (j-1)&1 is unambiguous.
                mbar_wait(smem_u32(&bars->pv_done), (j - 1) & 1);
                tc_fence_after();
#pragma unroll
                for (int c = 0; c < D / 32; ++c) {
                    uint32_t o[32];
                    tmem_ld32(trow + 256 + c * 32, o);
                    tmem_wait_ld();
#pragma unroll
                    for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
                    tmem_st32(trow + 256 + c * 32, o);
                }
            }
#pragma unroll
            for (int c = 0; c < kBN / 64; ++c)
                tmem_st32(trow + sb * 128 + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&pk[c * 32]));
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(smem_u32(&bars->p_full[sb]));
        }

        // ------------------------------------------------------------ epilogue
        mbar_wait(smem_u32(&bars->o_final), 0);
        tc_fence_after();
        if (!DUMP) {
            const float inv_l = 1.0f / l;
            bool finite = true;
#pragma unroll
            for (int c = 0; c < D / 32; ++c) {
                uint32_t o[32];
                tmem_ld32(trow + 256 + c * 32, o);
                tmem_wait_ld();
                float v[32];
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                    finite &= isfinite(__uint_as_float(o[e]));
                    v[e] = __uint_as_float(o[e]) * inv_l;
                }
                if (qi < n) {
                    const size_t off = (static_cast<size_t>(unit) * n + qi) * D + c * 32;
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
            }
            if (qi < n && !finite) atomicOr(p.status, kStatusOverflow);
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 4) {
        tc_fence_after();
        tmem_dealloc<512>(tbase);
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

// (inner=d, tokens, units) tensor map with a (box_x, 128, 1) box.
bool make_map(CUtensorMap* tm, const void* base, CUtensorMapDataType dt, int elem, int d, int n, int units, int box_x,
              CUtensorMapSwizzle sw) {
    EncodeFn enc = get_encode();
    if (!enc) return false;
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(n), static_cast<cuuint64_t>(units)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(d) * elem, static_cast<cuuint64_t>(d) * n * elem};
    const cuuint32_t box[3] = {static_cast<cuuint32_t>(box_x), 128, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    return enc(tm, dt, 3, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int D, bool CAUSAL, bool OUT_F32, bool DUMP>
cudaError_t launch_k2(const AttnParams& p, cudaStream_t s) {
    using C = Cfg<D>;
    CUtensorMap tq, tk, tv;
    const CUtensorMapSwizzle swqk = D == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
    if (!make_map(&tq, p.qcodes, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, D, p.n, p.units, D, swqk) ||
        !make_map(&tk, p.kcodes, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, D, p.n, p.units, D, swqk) ||
        !make_map(&tv, p.v16, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, D, p.n, p.units, 64, CU_TENSOR_MAP_SWIZZLE_128B))
        return cudaErrorInvalidValue;
    auto kern = k2_attention<D, CAUSAL, OUT_F32, DUMP>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    if (e != cudaSuccess) return e;
    const int ntq = (p.n + kBM - 1) / kBM;
    const unsigned grid = DUMP ? 1u : static_cast<unsigned>(ntq) * static_cast<unsigned>(p.units);
    kern<<<grid, kThreads, C::kSmemBytes, s>>>(tq, tk, tv, p);
    return cudaGetLastError();
}

template <bool DUMP>
cudaError_t dispatch(const AttnParams& p, cudaStream_t s) {
    const bool c = p.causal != 0, f = p.out_f32 != 0;
    if (p.d == 128) {
        if (c) return f ? launch_k2<128, true, true, DUMP>(p, s) : launch_k2<128, true, false, DUMP>(p, s);
        return f ? launch_k2<128, false, true, DUMP>(p, s) : launch_k2<128, false, false, DUMP>(p, s);
    }
    if (p.d == 64) {
        if (c) return f ? launch_k2<64, true, true, DUMP>(p, s) : launch_k2<64, true, false, DUMP>(p, s);
        return f ? launch_k2<64, false, true, DUMP>(p, s) : launch_k2<64, false, false, DUMP>(p, s);
    }
    return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_attention(const AttnParams& p, cudaStream_t s) { return dispatch<false>(p, s); }

cudaError_t launch_qk_dump(const AttnParams& p, cudaStream_t s) {
    AttnParams q = p;
    q.out_f32 = 1;
    return dispatch<true>(q, s);
}

}  // namespace sab
