/*
 * sage_oracle.c -- CPU restatement of the SageAttn-B forward path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the CUDA library
 * under paper_2410_02367_b200/csrc) links, loads or calls this file.  It is
 * imported by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg, and only as the checker.
 *
 * Every function restates one piece of the reference (a header-only C++20
 * CPU emulation under /root/reference/proj/include/sageattn/) in plain C11.
 * The restatement is pinned bit-for-bit against the reference itself
 * (compiled by oracle/Makefile into oracle/_ref/) by tests/test_oracle.py
 * and against the committed golden vectors in tests/golden/.
 *
 * Build: gcc -std=c11 -O2 -ffp-contract=off -fPIC -shared (oracle/Makefile).
 * -ffp-contract=off keeps the binary32 `rescale*l + row_sum` update
 * un-fused, matching the reference's default x86-64 build.
 *
 * Layout: one (batch, head) "unit" is a row-major tokens x head_dim slice,
 * the same as Tensor4::slice (tensor.hpp:83-93).  Units are independent
 * (SURVEY F2), so every entry point works on one unit and the *_units
 * wrappers fan units out over pthreads.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_ERR_SHAPE 1
#define ORC_ERR_NONFINITE 2
#define ORC_ERR_OVERFLOW 3
#define ORC_ERR_NOMEM 8

/* ------------------------------------------------------------------------ */
/* binary16 rounding (half.hpp:37-109).                                     */
/* ------------------------------------------------------------------------ */

/* Nearest binary16 value to x (ties to even), returned as a double.
 * Restates round_to_half + half_to_double (half.hpp:39-98) with a
 * "round by magic addition" formulation: adding C = 1.5 * 2^(e_ulp + 52)
 * makes the double adder round x to a multiple of the binary16 ulp 2^e_ulp
 * with RNE in a single correctly rounded step.  Overflow (|r| > 65504)
 * saturates to infinity as in half.hpp:73.  NaN propagates. */
double orc_snap_half(double x)
{
    if (x != x) return x;
    double ax = fabs(x);
    if (ax == 0.0 || isinf(ax)) return x;
    int e2;
    (void)frexp(ax, &e2);           /* ax = f * 2^e2, f in [0.5, 1) */
    int e = e2 - 1;                 /* floor(log2 ax) */
    int ulp_exp = (e < -14) ? -24 : e - 10;
    if (ulp_exp > 5) ulp_exp = 5;   /* beyond the binary16 range: ulp 32 at 2^15 */
    double c = ldexp(1.5, ulp_exp + 52);
    volatile double t = ax + c;     /* volatile: keep the double rounding step */
    double r = t - c;
    if (r > 65504.0) r = INFINITY;
    return x < 0 ? -r : r;
}

/* IEEE binary16 bit pattern of orc_snap_half(x). */
uint16_t orc_half_bits(double x)
{
    double r = orc_snap_half(x);
    uint16_t sign = signbit(r) ? 0x8000u : 0u;
    double a = fabs(r);
    if (r != r) return (uint16_t)(sign | 0x7E00u);
    if (isinf(a)) return (uint16_t)(sign | 0x7C00u);
    if (a == 0.0) return sign;
    if (a < ldexp(1.0, -14)) return (uint16_t)(sign | (uint16_t)ldexp(a, 24));
    int e2;
    double f = frexp(a, &e2);       /* a = f * 2^e2 */
    int exp_field = e2 - 1 + 15;
    uint16_t mant = (uint16_t)(ldexp(f, 11) - 1024.0);
    return (uint16_t)(sign | (uint16_t)(exp_field << 10) | mant);
}

/* ------------------------------------------------------------------------ */
/* K smoothing (quant.hpp:187-242) and 1/sqrt(d) folding (quant.hpp:244-252) */
/* ------------------------------------------------------------------------ */

/* Pairwise binary32 column sum over token rows [t0, t1): leaves of <= 8
 * tokens are summed sequentially from 0.0f, longer ranges split at
 * t0 + n/2.  Restates detail::pairwise_column_sum (quant.hpp:203-213). */
float orc_pairwise_column_sum(const float* base, int stride, int c, int t0, int t1)
{
    int n = t1 - t0;
    if (n <= 8) {
        float s = 0.0f;
        for (int t = t0; t < t1; ++t) s += base[(size_t)t * stride + c];
        return s;
    }
    int mid = t0 + n / 2;
    float lo = orc_pairwise_column_sum(base, stride, c, t0, mid);
    float hi = orc_pairwise_column_sum(base, stride, c, mid, t1);
    return lo + hi;
}

/* mean_k[c] = pairwise_sum(K[:, c]) * (1.0f / N)   (quant.hpp:228, 235). */
void orc_mean_k(const float* k, int n, int d, float* mean)
{
    const float inv_n = 1.0f / (float)n;
    for (int c = 0; c < d; ++c) mean[c] = orc_pairwise_column_sum(k, d, c, 0, n) * inv_n;
}

/* K_s = K - mean_k (quant.hpp:236-238); mean is written when non-NULL. */
void orc_smooth_k(const float* k, int n, int d, float* ks, float* mean_out)
{
    float* mean = (float*)malloc(sizeof(float) * (size_t)d);
    orc_mean_k(k, n, d, mean);
    for (int t = 0; t < n; ++t)
        for (int c = 0; c < d; ++c) ks[(size_t)t * d + c] = k[(size_t)t * d + c] - mean[c];
    if (mean_out) memcpy(mean_out, mean, sizeof(float) * (size_t)d);
    free(mean);
}

/* s_d = float(1 / sqrt(double(d)))  (quant.hpp:249). */
float orc_fold_factor(int d) { return (float)(1.0 / sqrt((double)d)); }

/* q_f = q * s_d elementwise in binary32 (quant.hpp:250). */
void orc_fold_q(const float* q, size_t count, int d, float* qf)
{
    const float s = orc_fold_factor(d);
    for (size_t i = 0; i < count; ++i) qf[i] = q[i] * s;
}

/* ------------------------------------------------------------------------ */
/* RoPE (the product's sab_prepass_rope; PAPER.md:397 fuses quantization    */
/* into the RoPE kernel).  The reference has no RoPE: this restates the      */
/* rotation as sab_prepass_rope defines it -- binary32, every product and    */
/* sum rounded -- so the fused K1 can be compared with                       */
/* prepass(rope(q), rope(k)) bit for bit.  layout 1: pairs (2i, 2i+1);       */
/* layout 2: pairs (i, i + d/2).  x' = x_a c - x_b s, x_b' = x_a s + x_b c.  */
/* cs / sn: [n][d/2]; x: units x n x d, rotated in place.                   */
/* ------------------------------------------------------------------------ */
void orc_rope(float* x, int units, int n, int d, const float* cs, const float* sn, int layout)
{
    const int h = d / 2;
    for (int u = 0; u < units; ++u)
        for (int t = 0; t < n; ++t) {
            float* row = x + ((size_t)u * n + t) * d;
            for (int i = 0; i < h; ++i) {
                const int a = layout == 1 ? 2 * i : i, b = layout == 1 ? 2 * i + 1 : i + h;
                const float c = cs[(size_t)t * h + i], s = sn[(size_t)t * h + i];
                const float xa = row[a], xb = row[b];
                const float ac = xa * c, bs = xb * s, as = xa * s, bc = xb * c;
                row[a] = ac - bs;
                row[b] = as + bc;
            }
        }
}

/* ------------------------------------------------------------------------ */
/* INT8 per-block dynamic quantizer (quant.hpp:95-173, INT8 arm only).      */
/* ------------------------------------------------------------------------ */

static int8_t orc_code(float x, float inv)
{
    /* quant.hpp:95-101: nearbyintf under the default RNE mode, then clamp. */
    float r = nearbyintf(x * inv);
    if (r > 127.0f) r = 127.0f;
    if (r < -127.0f) r = -127.0f;
    return (int8_t)r;
}

/* Quantizes a rows x cols matrix in groups of `block` consecutive rows:
 * delta = max|group| / 127, inv = 1 / delta, codes = clamp(rne(x*inv)).
 * An all-zero group takes delta = 1 and inv = 0 (quant.hpp:141-152).
 * Returns ORC_ERR_NONFINITE on a non-finite element (quant.hpp:136-139). */
int orc_quantize_int8_rows(const float* a, int rows, int cols, int block, int8_t* codes, float* scales)
{
    for (size_t i = 0; i < (size_t)rows * cols; ++i)
        if (!isfinite(a[i])) return ORC_ERR_NONFINITE;
    int groups = (rows + block - 1) / block;
    for (int g = 0; g < groups; ++g) {
        int r0 = g * block, r1 = r0 + block < rows ? r0 + block : rows;
        float amax = 0.0f;
        for (int r = r0; r < r1; ++r)
            for (int c = 0; c < cols; ++c) {
                float v = fabsf(a[(size_t)r * cols + c]);
                if (v > amax) amax = v;
            }
        float delta, inv;
        if (amax == 0.0f) {
            delta = 1.0f;
            inv = 0.0f;
        } else {
            delta = amax / 127.0f;
            inv = 1.0f / delta;
        }
        scales[g] = delta;
        for (int r = r0; r < r1; ++r)
            for (int c = 0; c < cols; ++c)
                codes[(size_t)r * cols + c] = orc_code(a[(size_t)r * cols + c], inv);
    }
    return ORC_OK;
}

/* Per-channel INT8 quantizer (quant.hpp:128-173 with Granularity::per_channel,
 * group_of(r, c) = c, quant.hpp:46-63): delta_c = max_t |a[t][c]| / 127. */
int orc_quantize_int8_cols(const float* a, int rows, int cols, int8_t* codes, float* scales)
{
    for (size_t i = 0; i < (size_t)rows * cols; ++i)
        if (!isfinite(a[i])) return ORC_ERR_NONFINITE;
    for (int c = 0; c < cols; ++c) {
        float amax = 0.0f;
        for (int r = 0; r < rows; ++r) {
            float v = fabsf(a[(size_t)r * cols + c]);
            if (v > amax) amax = v;
        }
        float inv;
        if (amax == 0.0f) {
            scales[c] = 1.0f;
            inv = 0.0f;
        } else {
            scales[c] = amax / 127.0f;
            inv = 1.0f / scales[c];
        }
        for (int r = 0; r < rows; ++r) codes[(size_t)r * cols + c] = orc_code(a[(size_t)r * cols + c], inv);
    }
    return ORC_OK;
}

/* The B-path prepass for one unit: fold+quantize Q in 128-token blocks and
 * smooth+quantize K in 64-token blocks (attention.hpp:336-360). */
int orc_prepass_unit(const float* q, const float* k, int n, int d, int block_q, int block_kv, int smooth,
                     int8_t* qcodes, float* qscales, int8_t* kcodes, float* kscales, float* mean)
{
    size_t cnt = (size_t)n * d;
    float* tmp = (float*)malloc(sizeof(float) * cnt);
    if (!tmp) return ORC_ERR_NOMEM;
    for (size_t i = 0; i < cnt; ++i)
        if (!isfinite(q[i]) || !isfinite(k[i])) { free(tmp); return ORC_ERR_NONFINITE; }
    if (smooth) {
        orc_smooth_k(k, n, d, tmp, mean);
    } else {
        memcpy(tmp, k, sizeof(float) * cnt);
        if (mean) memset(mean, 0, sizeof(float) * (size_t)d);
    }
    int st = orc_quantize_int8_rows(tmp, n, d, block_kv, kcodes, kscales);
    if (st == ORC_OK) {
        orc_fold_q(q, cnt, d, tmp);
        st = orc_quantize_int8_rows(tmp, n, d, block_q, qcodes, qscales);
    }
    free(tmp);
    return st;
}

/* ------------------------------------------------------------------------ */
/* INT8 S-stage tile (attention.hpp:264-279).                               */
/* ------------------------------------------------------------------------ */

void orc_int8_tile_nt(const int8_t* qc, const int8_t* kc, int d, int r0, int bq, int c0, int bkv, int32_t* acc,
                      int acc_stride)
{
    for (int r = 0; r < bq; ++r) {
        const int8_t* qrow = qc + (size_t)(r0 + r) * d;
        for (int c = 0; c < bkv; ++c) {
            const int8_t* krow = kc + (size_t)(c0 + c) * d;
            int32_t s = 0;
            for (int x = 0; x < d; ++x) s += (int32_t)qrow[x] * (int32_t)krow[x];
            acc[(size_t)r * acc_stride + c] = s;
        }
    }
}

/* ------------------------------------------------------------------------ */
/* SAGEAttn-B tiled engine for one unit (attention.hpp:318-545, Fp16Acc).   */
/* ------------------------------------------------------------------------ */

/* Causal tile class (attention.hpp:83-94): 0 Full, 1 Diagonal, 2 Skip. */
int orc_causal_tile(int i, int j, int block_q, int block_kv, int n)
{
    int r0 = i * block_q;
    int r1 = (r0 + block_q < n ? r0 + block_q : n) - 1;
    int c0 = j * block_kv;
    int c1 = (c0 + block_kv < n ? c0 + block_kv : n) - 1;
    if (c0 > r1) return 2;
    if (c1 <= r0) return 0;
    return 1;
}

/* Runs query tiles [qt0, qt1) of one unit from already-quantized operands.
 * pv_fp32 selects SageOptions::pv_fp32_accumulator (attention.hpp:454-471);
 * otherwise the binary16 accumulator rounds after every addition
 * (matmul.hpp:63-73).  out rows outside the tile range are untouched.
 * Returns ORC_ERR_OVERFLOW when the binary16 accumulator overflowed
 * (attention.hpp:531-533).  macs[0..1] accumulate the SageDiagnostics MAC
 * counters (attention.hpp:404, 445) when non-NULL. */
static int orc_sage_tiles_v(const int8_t* qc, const float* qs, const int8_t* kc, const float* ks, const float* v,
                            int n, int d, int causal, int pv_fp32, int pv_int8, int block_q, int block_kv, int gq,
                            int gk, int qt0, int qt1, float* out, uint64_t* macs)
{
    const int n_kv = (n + block_kv - 1) / block_kv;
    int32_t* acc = (int32_t*)malloc(sizeof(int32_t) * (size_t)block_q * block_kv);
    float* s = (float*)malloc(sizeof(float) * (size_t)block_q * block_kv);
    double* p16 = (double*)malloc(sizeof(double) * (size_t)block_q * block_kv);
    double* o = (double*)malloc(sizeof(double) * (size_t)block_q * d);
    float* m = (float*)malloc(sizeof(float) * (size_t)block_q);
    float* l = (float*)malloc(sizeof(float) * (size_t)block_q);
    float* rs = (float*)malloc(sizeof(float) * (size_t)block_q);
    double* v16 = (double*)malloc(sizeof(double) * (size_t)n * d);
    int8_t* vc = pv_int8 ? (int8_t*)malloc((size_t)n * d) : NULL;
    float* vs = pv_int8 ? (float*)malloc(sizeof(float) * (size_t)d) : NULL;
    int8_t* pc = (int8_t*)malloc((size_t)block_q * block_kv);
    int status = ORC_OK;
    if (!acc || !s || !p16 || !o || !m || !l || !rs || !v16 || !pc || (pv_int8 && (!vc || !vs))) {
        status = ORC_ERR_NOMEM;
        goto done;
    }

    if (pv_int8) {
        /* SAGEAttn-vB/vT: V -> per-channel INT8 (attention.hpp:376-378). */
        status = orc_quantize_int8_cols(v, n, d, vc, vs);
        if (status != ORC_OK) goto done;
    } else {
        /* V -> binary16 grid (attention.hpp:371-375). */
        for (size_t i = 0; i < (size_t)n * d; ++i) v16[i] = orc_snap_half((double)v[i]);
    }

    for (int i = qt0; i < qt1; ++i) {
        const int r0 = i * block_q;
        const int bq = (block_q < n - r0) ? block_q : n - r0;
        for (int r = 0; r < bq; ++r) {
            m[r] = -INFINITY;
            l[r] = 0.0f;
            for (int c = 0; c < d; ++c) o[(size_t)r * d + c] = 0.0;
        }
        for (int j = 0; j < n_kv; ++j) {
            const int c0 = j * block_kv;
            const int bkv = (block_kv < n - c0) ? block_kv : n - c0;
            int kind = 0;
            if (causal) {
                kind = orc_causal_tile(i, j, block_q, block_kv, n);
                if (kind == 2) continue;
            }
            if (macs) macs[0] += (uint64_t)bq * bkv * d;
            orc_int8_tile_nt(qc, kc, d, r0, bq, c0, bkv, acc, block_kv);
            /* s = (float(acc) * dq) * dk  (attention.hpp:409-414); scale groups of gq / gk
             * tokens (Granularity::group_of, quant.hpp:56-63: per_block(b) -> r / b,
             * per_token -> r). */
            for (int r = 0; r < bq; ++r) {
                const float dq = qs[(r0 + r) / gq];
                for (int c = 0; c < bkv; ++c)
                    s[r * block_kv + c] = ((float)acc[r * block_kv + c] * dq) * ks[(c0 + c) / gk];
            }
            if (kind == 1)
                for (int r = 0; r < bq; ++r)
                    for (int c = 0; c < bkv; ++c)
                        if (c0 + c > r0 + r) s[r * block_kv + c] = -INFINITY;
            /* Online softmax in binary32 (attention.hpp:430-443). */
            for (int r = 0; r < bq; ++r) {
                float mx = m[r];
                for (int c = 0; c < bkv; ++c) mx = fmaxf(mx, s[r * block_kv + c]);
                rs[r] = expf(m[r] - mx);
                float sum = 0.0f;
                for (int c = 0; c < bkv; ++c) {
                    float sv = s[r * block_kv + c];
                    float p = (sv == -INFINITY) ? 0.0f : expf(sv - mx);
                    s[r * block_kv + c] = p;
                    sum += p;
                }
                m[r] = mx;
                l[r] = rs[r] * l[r] + sum;
            }
            if (macs) macs[1] += (uint64_t)bq * bkv * d;
            if (pv_int8) {
                /* INT8 P~V (attention.hpp:476-505): P~ -> static-scale codes
                 * rne(p * 127) (quantize_p_static, quant.hpp:258-279), O rescaled in
                 * binary32, INT32 dot products dequantized by (acc * dP) * dV[c]. */
                const float dp = 1.0f / 127.0f;
                for (int r = 0; r < bq; ++r)
                    for (int c = 0; c < bkv; ++c) {
                        const float pv = s[r * block_kv + c];
                        if (!(pv >= 0.0f && pv <= 1.0f + 1e-6f)) { status = ORC_ERR_SHAPE; goto done; }
                        pc[r * block_kv + c] = orc_code(pv, 127.0f);
                    }
                for (int r = 0; r < bq; ++r) {
                    double* orow = o + (size_t)r * d;
                    for (int c = 0; c < d; ++c) orow[c] = (double)((float)orow[c] * rs[r]);
                    for (int c = 0; c < d; ++c) {
                        int32_t a = 0;
                        for (int kk = 0; kk < bkv; ++kk)
                            a += (int32_t)pc[r * block_kv + kk] * (int32_t)vc[(size_t)(c0 + kk) * d + c];
                        orow[c] = (double)((float)orow[c] + ((float)a * dp) * vs[c]);
                    }
                }
                continue;
            }
            /* O rescale and P~ V with the binary16 (or binary32) accumulator
             * (attention.hpp:447-475). */
            for (int r = 0; r < bq; ++r) {
                double* orow = o + (size_t)r * d;
                for (int c = 0; c < d; ++c) {
                    float scaled = rs[r] * (float)orow[c];
                    orow[c] = pv_fp32 ? (double)scaled : orc_snap_half((double)scaled);
                }
                for (int c = 0; c < bkv; ++c) p16[r * block_kv + c] = orc_snap_half((double)s[r * block_kv + c]);
            }
            for (int r = 0; r < bq; ++r) {
                double* orow = o + (size_t)r * d;
                for (int kk = 0; kk < bkv; ++kk) {
                    const double pv = p16[r * block_kv + kk];
                    if (pv == 0.0) continue;
                    const double* vrow = v16 + (size_t)(c0 + kk) * d;
                    if (pv_fp32) {
                        const float pf = (float)pv;
                        for (int c = 0; c < d; ++c) orow[c] = (double)((float)orow[c] + pf * (float)vrow[c]);
                    } else {
                        for (int c = 0; c < d; ++c) orow[c] = orc_snap_half(orow[c] + pv * vrow[c]);
                    }
                }
            }
        }
        /* O = diag(l)^-1 O (attention.hpp:524-540). */
        for (int r = 0; r < bq; ++r) {
            const float inv_l = 1.0f / l[r];
            for (int c = 0; c < d; ++c) {
                double src = o[(size_t)r * d + c];
                if (!pv_int8 && !isfinite(src)) { status = ORC_ERR_OVERFLOW; goto done; }
                out[(size_t)(r0 + r) * d + c] = (float)src * inv_l;
            }
        }
    }
done:
    free(acc); free(s); free(p16); free(o); free(m); free(l); free(rs); free(v16); free(vc); free(vs); free(pc);
    return status;
}

int orc_sage_tiles(const int8_t* qc, const float* qs, const int8_t* kc, const float* ks, const float* v, int n, int d,
                   int causal, int pv_fp32, int block_q, int block_kv, int gq, int gk, int qt0, int qt1, float* out,
                   uint64_t* macs)
{
    return orc_sage_tiles_v(qc, qs, kc, ks, v, n, d, causal, pv_fp32, 0, block_q, block_kv, gq, gk, qt0, qt1, out,
                            macs);
}

/* The variant B tile loop: scale groups equal to the tiles (per_block(128 / 64)). */
int orc_sage_b_tiles(const int8_t* qc, const float* qs, const int8_t* kc, const float* ks, const float* v, int n,
                     int d, int causal, int pv_fp32, int block_q, int block_kv, int qt0, int qt1, float* out,
                     uint64_t* macs)
{
    return orc_sage_tiles(qc, qs, kc, ks, v, n, d, causal, pv_fp32, block_q, block_kv, block_q, block_kv, qt0, qt1,
                          out, macs);
}

/* Whole SAGEAttn forward for one unit (attention.hpp:318-545): variant B =
 * PerBlock(128/64) + Fp16Acc, variant T (per_token) = PerToken + Fp16Acc with the
 * same 128 x 64 tiles (kernel_config_for, attention.hpp:48-55). */
/* pv_int8 selects PvPath::Int8 (variants vB / vT, kernel_config_for, attention.hpp:52-53). */
int orc_sage_unit_v(const float* q, const float* k, const float* v, int n, int d, int causal, int smooth, int pv_fp32,
                    int per_token, int pv_int8, float* out, uint64_t* macs)
{
    const int bq = 128, bkv = 64;
    const int gq = per_token ? 1 : bq, gk = per_token ? 1 : bkv;
    for (size_t i = 0; i < (size_t)n * d; ++i)
        if (!isfinite(v[i])) return ORC_ERR_NONFINITE;
    int8_t* qc = (int8_t*)malloc((size_t)n * d);
    int8_t* kc = (int8_t*)malloc((size_t)n * d);
    float* qs = (float*)malloc(sizeof(float) * (size_t)((n + gq - 1) / gq));
    float* ks = (float*)malloc(sizeof(float) * (size_t)((n + gk - 1) / gk));
    int st = ORC_ERR_NOMEM;
    if (qc && kc && qs && ks) {
        st = orc_prepass_unit(q, k, n, d, gq, gk, smooth, qc, qs, kc, ks, NULL);
        if (st == ORC_OK)
            st = orc_sage_tiles_v(qc, qs, kc, ks, v, n, d, causal, pv_fp32, pv_int8, bq, bkv, gq, gk, 0,
                                  (n + bq - 1) / bq, out, macs);
    }
    free(qc); free(kc); free(qs); free(ks);
    return st;
}

int orc_sage_unit(const float* q, const float* k, const float* v, int n, int d, int causal, int smooth, int pv_fp32,
                  int per_token, float* out, uint64_t* macs)
{
    return orc_sage_unit_v(q, k, v, n, d, causal, smooth, pv_fp32, per_token, 0, out, macs);
}

int orc_sage_b_unit(const float* q, const float* k, const float* v, int n, int d, int causal, int smooth,
                    int pv_fp32, float* out, uint64_t* macs)
{
    return orc_sage_unit(q, k, v, n, d, causal, smooth, pv_fp32, 0, out, macs);
}

/* Exact binary64 attention for one unit (attention.hpp:110-149). */
/* naive_attention (attention.hpp:107-149) for query rows [r0, r1) of one unit; out is
 * (r1 - r0) x d.  Used for the exact-attention column at sizes where whole units are too
 * slow in binary64 (bench.py parity, large-shape tests). */
void orc_naive_rows(const float* q, const float* k, const float* v, int n, int d, int causal, int r0, int r1,
                    double* out)
{
    const double inv_sqrt_d = 1.0 / sqrt((double)d);
    double* s = (double*)malloc(sizeof(double) * (size_t)n);
    for (int t = r0; t < r1; ++t) {
        const int lim = causal ? t + 1 : n;
        double mx = -INFINITY;
        for (int j = 0; j < lim; ++j) {
            double a = 0.0;
            for (int c = 0; c < d; ++c) a += (double)q[(size_t)t * d + c] * k[(size_t)j * d + c];
            s[j] = a * inv_sqrt_d;
            if (s[j] > mx) mx = s[j];
        }
        double den = 0.0;
        for (int j = 0; j < lim; ++j) { s[j] = exp(s[j] - mx); den += s[j]; }
        double* orow = out + (size_t)(t - r0) * d;
        for (int c = 0; c < d; ++c) orow[c] = 0.0;
        for (int j = 0; j < lim; ++j)
            for (int c = 0; c < d; ++c) orow[c] += s[j] * v[(size_t)j * d + c];
        for (int c = 0; c < d; ++c) orow[c] /= den;
    }
    free(s);
}

void orc_naive_unit(const float* q, const float* k, const float* v, int n, int d, int causal, double* out)
{
    orc_naive_rows(q, k, v, n, d, causal, 0, n, out);
}

/* ------------------------------------------------------------------------ */
/* Unit fan-out over threads (exact by SURVEY F2).                          */
/* ------------------------------------------------------------------------ */

typedef struct {
    const float *q, *k, *v;
    float* out;
    double* out64;
    int units, n, d, causal, smooth, pv_fp32, naive, per_token, pv_int8;
    int next;
    int status;
    uint64_t macs[2];
    pthread_mutex_t mu;
} orc_job;

static void* orc_worker(void* arg)
{
    orc_job* job = (orc_job*)arg;
    uint64_t macs[2] = {0, 0};
    for (;;) {
        pthread_mutex_lock(&job->mu);
        int u = job->next++;
        pthread_mutex_unlock(&job->mu);
        if (u >= job->units) break;
        size_t off = (size_t)u * job->n * job->d;
        int st = ORC_OK;
        if (job->naive)
            orc_naive_unit(job->q + off, job->k + off, job->v + off, job->n, job->d, job->causal, job->out64 + off);
        else
            st = orc_sage_unit_v(job->q + off, job->k + off, job->v + off, job->n, job->d, job->causal,
                                 job->smooth, job->pv_fp32, job->per_token, job->pv_int8, job->out + off, macs);
        if (st != ORC_OK) {
            pthread_mutex_lock(&job->mu);
            if (job->status == ORC_OK) job->status = st;
            pthread_mutex_unlock(&job->mu);
        }
    }
    pthread_mutex_lock(&job->mu);
    job->macs[0] += macs[0];
    job->macs[1] += macs[1];
    pthread_mutex_unlock(&job->mu);
    return NULL;
}

static int orc_run(orc_job* job, int threads, uint64_t* macs)
{
    if (threads < 1) threads = 1;
    if (threads > job->units) threads = job->units;
    pthread_t* tid = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    pthread_mutex_init(&job->mu, NULL);
    for (int i = 0; i < threads; ++i) pthread_create(&tid[i], NULL, orc_worker, job);
    for (int i = 0; i < threads; ++i) pthread_join(tid[i], NULL);
    pthread_mutex_destroy(&job->mu);
    free(tid);
    if (macs) { macs[0] = job->macs[0]; macs[1] = job->macs[1]; }
    return job->status;
}

/* Any of the four variants: per_token (T / vT) and pv_int8 (vB / vT). */
int orc_sage_v(const float* q, const float* k, const float* v, int units, int n, int d, int causal, int smooth,
               int pv_fp32, int per_token, int pv_int8, int threads, float* out, uint64_t* macs)
{
    if (units < 1 || n < 1 || d < 1) return ORC_ERR_SHAPE;
    orc_job job;
    memset(&job, 0, sizeof(job));
    job.q = q; job.k = k; job.v = v; job.out = out;
    job.units = units; job.n = n; job.d = d; job.causal = causal; job.smooth = smooth; job.pv_fp32 = pv_fp32;
    job.per_token = per_token;
    job.pv_int8 = pv_int8;
    return orc_run(&job, threads, macs);
}

int orc_sage(const float* q, const float* k, const float* v, int units, int n, int d, int causal, int smooth,
             int pv_fp32, int per_token, int threads, float* out, uint64_t* macs)
{
    return orc_sage_v(q, k, v, units, n, d, causal, smooth, pv_fp32, per_token, 0, threads, out, macs);
}

int orc_sage_b(const float* q, const float* k, const float* v, int units, int n, int d, int causal, int smooth,
               int pv_fp32, int threads, float* out, uint64_t* macs)
{
    return orc_sage(q, k, v, units, n, d, causal, smooth, pv_fp32, 0, threads, out, macs);
}

int orc_naive(const float* q, const float* k, const float* v, int units, int n, int d, int causal, int threads,
              double* out)
{
    if (units < 1 || n < 1 || d < 1) return ORC_ERR_SHAPE;
    orc_job job;
    memset(&job, 0, sizeof(job));
    job.q = q; job.k = k; job.v = v; job.out64 = out;
    job.units = units; job.n = n; job.d = d; job.causal = causal; job.naive = 1;
    return orc_run(&job, threads, NULL);
}
