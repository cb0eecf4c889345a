// ref_driver.cpp -- C-ABI wrapper around the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file against
// /root/reference/proj/include (the reference's own sources, where they lie;
// nothing is copied into this repo) into oracle/_ref/libsageref.so.  The
// result is used (1) to pin the C restatement in oracle/sage_oracle.c,
// (2) to generate tests/golden/ fixtures, and (3) as the reference CPU arm
// of bench.py.  It is never linked into the product library.
//
// Every entry point catches the reference's exceptions and maps them to the
// status codes of include/sageattn_b200.h (1 invalid_argument, 3
// overflow_error), copying the what() text into a thread-local buffer.
#include <sageattn/attention.hpp>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

using namespace sageattn;

namespace {

thread_local std::string g_msg;

int fail(const std::exception& e, int code) {
    g_msg = e.what();
    return code;
}

Tensor4f make4(const float* src, int b, int h, int n, int d) {
    Tensor4f t(b, h, n, d);
    std::memcpy(t.data.data(), src, sizeof(float) * t.size());
    return t;
}

}  // namespace

extern "C" {

const char* ref_last_message() { return g_msg.c_str(); }

uint16_t ref_round_to_half(double x) { return round_to_half(x).bits; }

double ref_snap_to_half(double x) { return snap_to_half(x); }

// smooth_k (quant.hpp:220-242) over a whole (B,H,N,d) tensor.
int ref_smooth_k(const float* k, int b, int h, int n, int d, float* ks, float* mean) {
    try {
        auto [out, st] = smooth_k(make4(k, b, h, n, d));
        std::memcpy(ks, out.data.data(), sizeof(float) * out.size());
        std::memcpy(mean, st.mean_k.data(), sizeof(float) * st.mean_k.size());
        return 0;
    } catch (const std::invalid_argument& e) { return fail(e, 1); }
}

// Q path of the prepass: fold_scale_into_q then per_block(block_q) INT8
// quantize per unit (attention.hpp:342-359).
int ref_quantize_q(const float* q, int b, int h, int n, int d, int block_q, int8_t* codes, float* scales) {
    try {
        const Tensor4f qf = fold_scale_into_q(make4(q, b, h, n, d), d);
        const int groups = (n + block_q - 1) / block_q;
        for (int u = 0; u < b * h; ++u) {
            QuantizedMatrix qm = quantize(qf.slice(u / h, u % h), Granularity::per_block(block_q), QuantDtype::Int8);
            std::memcpy(codes + size_t(u) * n * d, qm.codes.data(), qm.codes.size());
            std::memcpy(scales + size_t(u) * groups, qm.scales.data(), sizeof(float) * groups);
        }
        return 0;
    } catch (const std::invalid_argument& e) { return fail(e, 1); }
}

// K path of the prepass: smooth_k (optional) then per_block(block_kv) INT8
// quantize per unit (attention.hpp:336-360).
int ref_quantize_k(const float* k, int b, int h, int n, int d, int block_kv, int smooth, int8_t* codes,
                   float* scales) {
    try {
        Tensor4f src = make4(k, b, h, n, d);
        if (smooth) src = smooth_k(src).first;
        const int groups = (n + block_kv - 1) / block_kv;
        for (int u = 0; u < b * h; ++u) {
            QuantizedMatrix qm = quantize(src.slice(u / h, u % h), Granularity::per_block(block_kv), QuantDtype::Int8);
            std::memcpy(codes + size_t(u) * n * d, qm.codes.data(), qm.codes.size());
            std::memcpy(scales + size_t(u) * groups, qm.scales.data(), sizeof(float) * groups);
        }
        return 0;
    } catch (const std::invalid_argument& e) { return fail(e, 1); }
}

// The T-path prepass (kernel_config_for(T), attention.hpp:50): Granularity::per_token()
// for both psi_Q (folded Q) and psi_K (smoothed K) (attention.hpp:255-262, 344-359).
int ref_quantize_qk_per_token(const float* q, const float* k, int b, int h, int n, int d, int smooth, int8_t* qcodes,
                              float* qscales, int8_t* kcodes, float* kscales) {
    try {
        const Tensor4f qf = fold_scale_into_q(make4(q, b, h, n, d), d);
        Tensor4f ks = make4(k, b, h, n, d);
        if (smooth) ks = smooth_k(ks).first;
        for (int u = 0; u < b * h; ++u) {
            QuantizedMatrix qm = quantize(qf.slice(u / h, u % h), Granularity::per_token(), QuantDtype::Int8);
            QuantizedMatrix km = quantize(ks.slice(u / h, u % h), Granularity::per_token(), QuantDtype::Int8);
            std::memcpy(qcodes + size_t(u) * n * d, qm.codes.data(), qm.codes.size());
            std::memcpy(qscales + size_t(u) * n, qm.scales.data(), sizeof(float) * n);
            std::memcpy(kcodes + size_t(u) * n * d, km.codes.data(), km.codes.size());
            std::memcpy(kscales + size_t(u) * n, km.scales.data(), sizeof(float) * n);
        }
        return 0;
    } catch (const std::invalid_argument& e) { return fail(e, 1); }
}

// sage_attention(in, SageVariant v, opts) (attention.hpp:547-550) for v = 0 (T), 1 (B), 2 (vT), 3 (vB).
int ref_sage_attention_variant(const float* q, const float* k, const float* v, int b, int h, int n, int d, int causal,
                               int variant, int smooth, int pv_fp32, float* out) {
    try {
        AttentionInput in{make4(q, b, h, n, d), make4(k, b, h, n, d), make4(v, b, h, n, d), causal != 0};
        SageOptions opt;
        opt.smooth_k = smooth != 0;
        opt.pv_fp32_accumulator = pv_fp32 != 0;
        static const SageVariant kV[4] = {SageVariant::T, SageVariant::B, SageVariant::VT, SageVariant::VB};
        if (variant < 0 || variant > 3) return 1;
        Tensor4f o = sage_attention(in, kV[variant], opt);
        std::memcpy(out, o.data.data(), sizeof(float) * o.size());
        return 0;
    } catch (const std::invalid_argument& e) { return fail(e, 1); } catch (const std::overflow_error& e) {
        return fail(e, 3);
    }
}

// SageDiagnostics static-scale counters (attention.hpp:58-69, 479-488) of sage_attention(in,
// VT|VB) with measure_static_scale = true: counts = {elements, first-block, later-block mismatches}.
int ref_static_scale_counts(const float* q, const float* k, const float* v, int b, int h, int n, int d, int causal,
                            int per_token, uint64_t* counts) {
    try {
        AttentionInput in{make4(q, b, h, n, d), make4(k, b, h, n, d), make4(v, b, h, n, d), causal != 0};
        SageDiagnostics diag;
        diag.measure_static_scale = true;
        SageOptions opt;
        opt.diagnostics = &diag;
        (void)sage_attention(in, per_token ? SageVariant::VT : SageVariant::VB, opt);
        counts[0] = diag.static_scale_elements;
        counts[1] = diag.static_scale_first_block_mismatches;
        counts[2] = diag.static_scale_later_block_mismatches;
        return 0;
    } catch (const std::invalid_argument& e) { return fail(e, 1); }
}

// quantize(a, Granularity::per_channel(), Int8) (quant.hpp:128-173): V^ of the vB/vT paths.
int ref_quantize_per_channel(const float* a, int rows, int cols, int8_t* codes, float* scales) {
    try {
        Matrix<float> m(rows, cols);
        std::memcpy(&m(0, 0), a, sizeof(float) * size_t(rows) * cols);
        QuantizedMatrix qm = quantize(m, Granularity::per_channel(), QuantDtype::Int8);
        std::memcpy(codes, qm.codes.data(), qm.codes.size());
        std::memcpy(scales, qm.scales.data(), sizeof(float) * qm.scales.size());
        return 0;
    } catch (const std::invalid_argument& e) { return fail(e, 1); }
}

// detail::int8_tile_nt (attention.hpp:265-279) on raw code matrices.
int ref_int8_tile(const int8_t* qc, const int8_t* kc, int n, int d, int r0, int bq, int c0, int bkv, int32_t* out) {
    QuantizedMatrix qm, km;
    qm.rows = km.rows = n;
    qm.cols = km.cols = d;
    qm.codes.assign(reinterpret_cast<const uint8_t*>(qc), reinterpret_cast<const uint8_t*>(qc) + size_t(n) * d);
    km.codes.assign(reinterpret_cast<const uint8_t*>(kc), reinterpret_cast<const uint8_t*>(kc) + size_t(n) * d);
    Matrix<int32_t> acc(bq, bkv);
    detail::int8_tile_nt(qm, km, r0, bq, c0, bkv, acc);
    std::memcpy(out, acc.data.data(), sizeof(int32_t) * acc.data.size());
    return 0;
}

// int8_matmul_i32acc (matmul.hpp:31-50) for known-answer tests.
int ref_int8_matmul(const int8_t* a, const int8_t* b, int m, int k, int n, int32_t* out) {
    try {
        Matrix<int32_t> r = int8_matmul_i32acc(MatView<int8_t>(a, m, k, k), MatView<int8_t>(b, k, n, n));
        std::memcpy(out, r.data.data(), sizeof(int32_t) * r.data.size());
        return 0;
    } catch (const std::invalid_argument& e) { return fail(e, 1); }
}

// fp16_matmul_fp16acc (matmul.hpp:75-96) on binary16-grid doubles.
int ref_fp16_matmul(const double* a, const double* b, int m, int k, int n, double* out) {
    try {
        Matrix<double> r = fp16_matmul_fp16acc(MatView<double>(a, m, k, k), MatView<double>(b, k, n, n));
        std::memcpy(out, r.data.data(), sizeof(double) * r.data.size());
        return 0;
    } catch (const std::invalid_argument& e) { return fail(e, 1); } catch (const std::overflow_error& e) {
        return fail(e, 3);
    }
}

// apply_causal_tiling (attention.hpp:83-94): 0 Full, 1 Diagonal, 2 Skip, -1 error.
int ref_causal_tile(int i, int j, int bq, int bkv, int n) {
    try {
        return int(apply_causal_tiling(i, j, bq, bkv, n));
    } catch (const std::invalid_argument& e) { return fail(e, -1); }
}

// sage_attention(in, KernelConfig{PerBlock, Fp16Acc, block_q, block_kv}, opts)
// on the whole tensor (attention.hpp:318-545).
int ref_sage_attention(const float* q, const float* k, const float* v, int b, int h, int n, int d, int causal,
                       int block_q, int block_kv, int smooth, int pv_fp32, float* out, uint64_t* macs) {
    try {
        AttentionInput in{make4(q, b, h, n, d), make4(k, b, h, n, d), make4(v, b, h, n, d), causal != 0};
        SageDiagnostics diag;
        SageOptions opt;
        opt.smooth_k = smooth != 0;
        opt.pv_fp32_accumulator = pv_fp32 != 0;
        opt.diagnostics = &diag;
        KernelConfig cfg = kernel_config_for(SageVariant::B);
        cfg.block_q = block_q;
        cfg.block_kv = block_kv;
        Tensor4f o = sage_attention(in, cfg, opt);
        std::memcpy(out, o.data.data(), sizeof(float) * o.size());
        if (macs) {
            macs[0] = diag.s_stage_macs;
            macs[1] = diag.pv_stage_macs;
        }
        return 0;
    } catch (const std::invalid_argument& e) { return fail(e, 1); } catch (const std::overflow_error& e) {
        return fail(e, 3);
    }
}

// Same call made one (b,h) unit at a time on `threads` host threads; bit
// identical to the whole-tensor call.  Used as the CPU baseline.
int ref_sage_attention_mt(const float* q, const float* k, const float* v, int units, int n, int d, int causal,
                          int smooth, int pv_fp32, int threads, float* out) {
    std::atomic<int> next{0}, status{0};
    auto work = [&]() {
        for (;;) {
            const int u = next.fetch_add(1);
            if (u >= units) return;
            const size_t off = size_t(u) * n * d;
            int st = ref_sage_attention(q + off, k + off, v + off, 1, 1, n, d, causal, 128, 64, smooth, pv_fp32,
                                        out + off, nullptr);
            if (st) status.store(st);
        }
    };
    threads = std::max(1, std::min(threads, units));
    std::vector<std::thread> pool;
    for (int i = 1; i < threads; ++i) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
    return status.load();
}

// naive_attention (attention.hpp:110-149): exact binary64 attention.
int ref_naive_attention(const float* q, const float* k, const float* v, int b, int h, int n, int d, int causal,
                        double* out) {
    try {
        AttentionInput in{make4(q, b, h, n, d), make4(k, b, h, n, d), make4(v, b, h, n, d), causal != 0};
        Tensor4d o = naive_attention(in);
        std::memcpy(out, o.data.data(), sizeof(double) * o.size());
        return 0;
    } catch (const std::invalid_argument& e) { return fail(e, 1); }
}

// Bounded CPU sample for bench timing: query tiles `tiles[0..n_tiles)` of
// one unit, computed with the reference's own building blocks
// (smooth_k, fold_scale_into_q, quantize, detail::int8_tile_nt,
// apply_causal_tiling, snap_to_half, fp16_accumulate_row) in the order of
// attention.hpp:357-541.  tests/test_oracle.py checks it reproduces the
// matching rows of ref_sage_attention bit-for-bit.
int ref_sage_b_tiles(const float* q, const float* k, const float* v, int n, int d, int causal, int pv_fp32,
                     const int* tiles, int n_tiles, float* out) {
    try {
        const int bq = 128, bkv = 64;
        const Tensor4f ks = smooth_k(make4(k, 1, 1, n, d)).first;
        const Tensor4f qf = fold_scale_into_q(make4(q, 1, 1, n, d), d);
        const QuantizedMatrix qhat = quantize(qf.slice(0, 0), Granularity::per_block(bq), QuantDtype::Int8);
        const QuantizedMatrix khat = quantize(ks.slice(0, 0), Granularity::per_block(bkv), QuantDtype::Int8);
        Matrix<double> v16(n, d);
        for (int t = 0; t < n; ++t)
            for (int c = 0; c < d; ++c) v16(t, c) = snap_to_half(double(v[size_t(t) * d + c]));
        const int n_kv = (n + bkv - 1) / bkv;
        Matrix<int32_t> acc(bq, bkv);
        Matrix<float> s(bq, bkv), p(bq, bkv);
        Matrix<double> o16(bq, d), p16(bq, bkv);
        std::vector<float> m(bq), l(bq), rs(bq);
        for (int ti = 0; ti < n_tiles; ++ti) {
            const int i = tiles[ti];
            const int r0 = i * bq, rows = std::min(bq, n - r0);
            std::fill(m.begin(), m.end(), -std::numeric_limits<float>::infinity());
            std::fill(l.begin(), l.end(), 0.0f);
            std::fill(o16.data.begin(), o16.data.end(), 0.0);
            for (int j = 0; j < n_kv; ++j) {
                const int c0 = j * bkv, cols = std::min(bkv, n - c0);
                TileKind kind = TileKind::Full;
                if (causal) {
                    kind = apply_causal_tiling(i, j, bq, bkv, n);
                    if (kind == TileKind::Skip) continue;
                }
                detail::int8_tile_nt(qhat, khat, r0, rows, c0, cols, acc);
                for (int r = 0; r < rows; ++r)
                    for (int c = 0; c < cols; ++c)
                        s(r, c) = (float(acc(r, c)) * qhat.scales[i]) * khat.scales[(c0 + c) / bkv];
                if (kind == TileKind::Diagonal)
                    for (int r = 0; r < rows; ++r)
                        for (int c = 0; c < cols; ++c)
                            if (c0 + c > r0 + r) s(r, c) = -std::numeric_limits<float>::infinity();
                for (int r = 0; r < rows; ++r) {
                    float mx = m[r];
                    for (int c = 0; c < cols; ++c) mx = std::max(mx, s(r, c));
                    rs[r] = std::exp(m[r] - mx);
                    float sum = 0.0f;
                    for (int c = 0; c < cols; ++c) {
                        const float pv = s(r, c) == -std::numeric_limits<float>::infinity() ? 0.0f
                                                                                            : std::exp(s(r, c) - mx);
                        p(r, c) = pv;
                        sum += pv;
                    }
                    m[r] = mx;
                    l[r] = rs[r] * l[r] + sum;
                }
                for (int r = 0; r < rows; ++r) {
                    for (int c = 0; c < d; ++c)
                        o16(r, c) = pv_fp32 ? double(rs[r] * float(o16(r, c)))
                                            : snap_to_half(double(rs[r] * float(o16(r, c))));
                    for (int c = 0; c < cols; ++c) p16(r, c) = snap_to_half(double(p(r, c)));
                }
                const MatView<double> vb(&v16(c0, 0), cols, d, d);
                for (int r = 0; r < rows; ++r) {
                    if (pv_fp32) {
                        for (int kk = 0; kk < cols; ++kk) {
                            const float pv = float(p16(r, kk));
                            if (pv == 0.0f) continue;
                            for (int c = 0; c < d; ++c)
                                o16(r, c) = double(float(o16(r, c)) + pv * float(vb(kk, c)));
                        }
                    } else {
                        fp16_accumulate_row(&p16(r, 0), vb, cols, &o16(r, 0), d);
                    }
                }
            }
            for (int r = 0; r < rows; ++r) {
                const float inv_l = 1.0f / l[r];
                for (int c = 0; c < d; ++c) out[size_t(r0 + r) * d + c] = float(o16(r, c)) * inv_l;
            }
        }
        return 0;
    } catch (const std::invalid_argument& e) { return fail(e, 1); }
}

}  // extern "C"
