// sageattn/attention.hpp -- B200 drop-in for the reference's attention entry points.
//
// Source-compatible replacement for /root/reference/proj/include/sageattn/
// attention.hpp: an application that calls
//     sageattn::sage_attention(const AttentionInput&, SageVariant, const SageOptions&)
//     sageattn::sage_attention(const AttentionInput&, const KernelConfig&, const SageOptions&)
// (attention.hpp:318-319, 547-550) switches to the B200 path by putting
// <repo>/include first on its include path and linking
// paper_2410_02367_b200/libsageattn_b200.so.  sage_attention is a thin header
// over the C ABI in sageattn_b200.h; the arithmetic runs in the CUDA kernels
// (K1 prepass + K2 tcgen05 attention, K3 head x batch sharding over every
// visible sm_100 device).
//
// Kept from the reference contract:
//   * the carriers Matrix / MatView / Tensor4 (tensor.hpp), QuantDtype (quant.hpp)
//     and AttentionInput, KernelConfig, QkGranularity, PvPath, SageVariant,
//     SageOptions, SageDiagnostics, TileKind with the same members and layouts;
//   * kernel_config_for, apply_causal_tiling, naive_attention, flash_attention_fp;
//   * exceptions and messages: std::invalid_argument for bad block sizes,
//     shape mismatch and non-finite input, std::overflow_error for a non-finite
//     P~V accumulator (attention.hpp:84-102, 321, 531-533);
//   * pure / re-entrant calls (per-call device contexts, attention.hpp:9-12);
//   * SageDiagnostics: the MAC counters (404, 445) and, on the INT8 P~V path,
//     the static-scale P~ mismatch counters (479-488), counted on the GPU.
// Differences:
//   * the four variants B, T (Fp16Acc P~V) and vB, vT (INT8 P~V) with block
//     128/64 and INT8 Q/K run; FP8 dtypes, PerTensor scales or other block sizes
//     throw std::invalid_argument -- there is no CPU fallback for sage_attention;
//   * head_dim must be 64 or 128;
//   * P~V accumulates in FP32 on the tensor cores (the reference's
//     pv_fp32_accumulator arm) whatever pv_fp32_accumulator says, unless
//     b200::honour_pv_accumulator_option() (SAB_PV_ACCUM=options) maps
//     pv_fp32_accumulator == false to the binary16 TMEM accumulator; Q^/K^
//     codes, scales and mean(K) are bit-identical to the reference.
// naive_attention (the binary64 exact oracle, attention.hpp:107-149) and
// flash_attention_fp (the binary32 tiled baseline, 169-252) are not on the
// SageAttn path; they stay host functions here so programs that compare
// against them keep compiling and behaving as before.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#if defined(__linux__)
#include <sys/mman.h>
#endif

#include "../sageattn_b200.h"
#include "quant.hpp"
#include "tensor.hpp"

namespace sageattn {

struct AttentionInput {
    Tensor4f q;
    Tensor4f k;
    Tensor4f v;
    bool causal = false;
};

enum class QkGranularity : uint8_t { PerToken, PerBlock, PerTensor };
enum class PvPath : uint8_t { Int8, Fp16Acc };
enum class SageVariant : uint8_t { T, B, VT, VB };

struct KernelConfig {
    QkGranularity qk_granularity = QkGranularity::PerBlock;
    PvPath pv_path = PvPath::Fp16Acc;
    int block_q = 128;
    int block_kv = 64;
};

inline KernelConfig kernel_config_for(SageVariant v) {
    const bool per_token = v == SageVariant::T || v == SageVariant::VT;
    const bool fp16_pv = v == SageVariant::T || v == SageVariant::B;
    return {per_token ? QkGranularity::PerToken : QkGranularity::PerBlock, fp16_pv ? PvPath::Fp16Acc : PvPath::Int8,
            128, 64};
}

struct SageDiagnostics {
    uint64_t s_stage_macs = 0;
    uint64_t pv_stage_macs = 0;
    bool measure_static_scale = false;
    uint64_t static_scale_elements = 0;
    uint64_t static_scale_first_block_mismatches = 0;
    uint64_t static_scale_later_block_mismatches = 0;
};

struct SageOptions {
    bool smooth_k = true;
    QuantDtype qk_dtype = QuantDtype::Int8;
    QuantDtype pv_dtype = QuantDtype::Int8;
    bool pv_fp32_accumulator = false;
    SageDiagnostics* diagnostics = nullptr;
};

enum class TileKind : uint8_t { Full, Diagonal, Skip };

inline TileKind apply_causal_tiling(int i, int j, int block_q, int block_kv, int n_tokens) {
    if (block_q < 1 || block_kv < 1) throw std::invalid_argument("block sizes must be >= 1");
    const int r0 = i * block_q, c0 = j * block_kv;
    const int r1 = std::min(r0 + block_q, n_tokens) - 1;
    const int c1 = std::min(c0 + block_kv, n_tokens) - 1;
    if (r0 < 0 || r0 > r1 || c0 < 0 || c0 > c1 || r1 >= n_tokens || c1 >= n_tokens)
        throw std::invalid_argument("tile indices out of range");
    if (c0 > r1) return TileKind::Skip;
    return c1 <= r0 ? TileKind::Full : TileKind::Diagonal;
}

namespace b200 {

// Maps a C-ABI status to the reference's exception types.
inline void throw_status(int status) {
    if (status == SAB_OK) return;
    const std::string msg = sab_last_error();
    switch (status) {
        case SAB_ERR_OVERFLOW: throw std::overflow_error(msg);
        case SAB_ERR_SHAPE:
        case SAB_ERR_NONFINITE:
        case SAB_ERR_UNSUPPORTED:
        case SAB_ERR_ARGUMENT: throw std::invalid_argument(msg);
        default: throw std::runtime_error("sage_attention (B200): " + msg);
    }
}

// Devices the host-buffer path (K3) shards over: 0 = every visible sm_100 device,
// n > 0 = the first n of them.
inline int& device_count_override() {
    static int n = 1;
    return n;
}

// P~V accumulator of a drop-in call (B/T).  false (default): FP32 in TMEM whatever
// SageOptions::pv_fp32_accumulator says -- the arm the parity gate is stated against.
// true: honour the option as the reference does (attention.hpp:75, 447-475), so the
// default pv_fp32_accumulator == false selects the binary16 TMEM accumulator
// (SAB_PV_FP16).  Environment: SAB_PV_ACCUM=options sets it at first use.
inline bool& honour_pv_accumulator_option() {
    static bool on = [] {
        const char* e = std::getenv("SAB_PV_ACCUM");
        return e && std::string(e) == "options";
    }();
    return on;
}

// The sm_100 ordinals a call uses (never a device of another architecture).
inline std::vector<int> devices_for_call() {
    int n = 0;
    throw_status(sab_device_ordinals(nullptr, 0, &n));
    std::vector<int> ids(size_t(std::max(n, 1)), 0);
    if (n > 0) throw_status(sab_device_ordinals(ids.data(), n, &n));
    const int want = device_count_override();
    if (want > 0 && want < int(ids.size())) ids.resize(size_t(want));
    return ids;
}

// The returned O.  Tensor4f's std::vector zero-fills its storage on the calling thread, and
// for a large tensor that fill is dominated by 4 KB page faults (about a fifth of a second
// per GB); on Linux the storage is reserved first and advised onto transparent huge pages,
// then filled.  SAB_DROPIN_THP=0 skips the advice.
inline Tensor4f alloc_output(int b, int h, int n, int d) {
    Tensor4f t;
    if (b < 1 || h < 1 || n < 1 || d < 1) throw std::invalid_argument("tensor dimensions must be positive");
    t.batch = b;
    t.heads = h;
    t.tokens = n;
    t.head_dim = d;
    const size_t count = size_t(b) * size_t(h) * size_t(n) * size_t(d);
#if defined(__linux__) && defined(MADV_HUGEPAGE)
    static const bool thp = [] {
        const char* e = std::getenv("SAB_DROPIN_THP");
        return !(e && e[0] == '0');
    }();
    constexpr uintptr_t kHuge = uintptr_t(2) << 20;
    if (thp && count * sizeof(float) >= 16 * kHuge) {
        t.data.reserve(count);
        const uintptr_t a = (reinterpret_cast<uintptr_t>(t.data.data()) + kHuge - 1) & ~(kHuge - 1);
        const uintptr_t e = reinterpret_cast<uintptr_t>(t.data.data() + count) & ~(kHuge - 1);
        if (e > a) (void)madvise(reinterpret_cast<void*>(a), e - a, MADV_HUGEPAGE);  // advice only
    }
#endif
    t.data.resize(count);
    return t;
}

inline void validate_input(const AttentionInput& in, const char* what) {
    if (!in.q.same_shape(in.k) || !in.q.same_shape(in.v))
        throw std::invalid_argument(std::string(what) + ": Q, K, V shapes differ");
    if (!in.q.all_finite() || !in.k.all_finite() || !in.v.all_finite())
        throw std::invalid_argument(std::string(what) + ": non-finite input");
}

}  // namespace b200

inline Tensor4f sage_attention(const AttentionInput& in, const KernelConfig& config,
                               const SageOptions& options = {}) {
    if (config.block_q < 1 || config.block_kv < 1)
        throw std::invalid_argument("sage_attention: block sizes must be >= 1");
    if (!in.q.same_shape(in.k) || !in.q.same_shape(in.v))
        throw std::invalid_argument("sage_attention: Q, K, V shapes differ");
    if (config.qk_granularity != QkGranularity::PerBlock && config.qk_granularity != QkGranularity::PerToken)
        throw std::invalid_argument(
            "sage_attention: only PerBlock (B, vB) or PerToken (T, vT) Q/K granularity runs on the B200 path");
    if (options.qk_dtype != QuantDtype::Int8)
        throw std::invalid_argument("sage_attention: only INT8 Q/K quantization runs on the B200 path");
    if (config.pv_path == PvPath::Int8 && options.pv_dtype != QuantDtype::Int8)
        throw std::invalid_argument("sage_attention: only INT8 P~V quantization runs on the B200 path");

    sab_desc d;
    sab_desc_init(&d, in.q.batch, in.q.heads, in.q.tokens, in.q.head_dim, in.causal ? 1 : 0);
    d.in_dtype = SAB_F32;  // bit-exact quantization of arbitrary fp32 Q/K (quant.hpp:128-173)
    d.out_dtype = SAB_F32;
    d.block_q = config.block_q;
    d.block_kv = config.block_kv;
    d.smooth_k = options.smooth_k ? 1 : 0;
    d.check_v = 1;  // validate_input scans V too (attention.hpp:101)
    d.qk_granularity = config.qk_granularity == QkGranularity::PerToken ? SAB_QK_PER_TOKEN : SAB_QK_PER_BLOCK;
    d.pv_path = config.pv_path == PvPath::Int8 ? SAB_PV_PATH_INT8 : SAB_PV_PATH_FP16;
    d.pv_accum = (b200::honour_pv_accumulator_option() && d.pv_path == SAB_PV_PATH_FP16 &&
                  !options.pv_fp32_accumulator)
                     ? SAB_PV_FP16
                     : SAB_PV_FP32;
    // attention.hpp:479: the static-scale counters exist only on the INT8 P~V path.
    SageDiagnostics* diag = options.diagnostics;
    d.measure_static_scale = (diag && diag->measure_static_scale && d.pv_path == SAB_PV_PATH_INT8) ? 1 : 0;
    Tensor4f out = b200::alloc_output(in.q.batch, in.q.heads, in.q.tokens, in.q.head_dim);
    const std::vector<int> devs = b200::devices_for_call();
    uint64_t counts[3] = {0, 0, 0};
    b200::throw_status(sab_attention_fwd_host_diag(&d, in.q.data.data(), in.k.data.data(), in.v.data.data(),
                                                   out.data.data(), devs.data(), int(devs.size()), counts));
    if (diag) {
        uint64_t s = 0, p = 0;
        b200::throw_status(sab_diagnostics(&d, &s, &p));
        diag->s_stage_macs += s;
        diag->pv_stage_macs += p;
        if (d.measure_static_scale) {
            diag->static_scale_elements += counts[0];
            diag->static_scale_first_block_mismatches += counts[1];
            diag->static_scale_later_block_mismatches += counts[2];
        }
    }
    return out;
}

inline Tensor4f sage_attention(const AttentionInput& in, SageVariant variant, const SageOptions& options = {}) {
    return sage_attention(in, kernel_config_for(variant), options);
}

// ---------------------------------------------------------------------------------------------
// Host functions outside the SageAttn path, kept so reference-API programs still build.

// Exact attention in binary64 (attention.hpp:107-149): scores Q K^T / sqrt(d), causal
// mask j > i, softmax and P V all accumulated in double.
inline Tensor4d naive_attention(const AttentionInput& in) {
    b200::validate_input(in, "naive_attention");
    const int n = in.q.tokens, d = in.q.head_dim;
    const double scale = 1.0 / std::sqrt(double(d));
    Tensor4d out(in.q.batch, in.q.heads, n, d);
    std::vector<double> w(size_t(n), 0.0);
    for (int b = 0; b < in.q.batch; ++b)
        for (int h = 0; h < in.q.heads; ++h) {
            const MatView<float> Q = in.q.slice(b, h), K = in.k.slice(b, h), V = in.v.slice(b, h);
            double* O = out.slice_ptr(b, h);
            for (int t = 0; t < n; ++t) {
                const int keys = in.causal ? t + 1 : n;
                double mx = -std::numeric_limits<double>::infinity();
                for (int j = 0; j < keys; ++j) {
                    double dot = 0.0;
                    for (int c = 0; c < d; ++c) dot += double(Q(t, c)) * double(K(j, c));
                    w[size_t(j)] = dot * scale;
                    mx = std::max(mx, w[size_t(j)]);
                }
                double sum = 0.0;
                for (int j = 0; j < keys; ++j) sum += (w[size_t(j)] = std::exp(w[size_t(j)] - mx));
                double* row = O + size_t(t) * size_t(d);
                std::fill(row, row + d, 0.0);
                for (int j = 0; j < keys; ++j)
                    for (int c = 0; c < d; ++c) row[c] += w[size_t(j)] * double(V(j, c));
                for (int c = 0; c < d; ++c) row[c] /= sum;
            }
        }
    return out;
}

// Tiled binary32 attention with online softmax (attention.hpp:169-252): the same
// block traversal, causal tile classes and binary32 arithmetic order.
inline Tensor4f flash_attention_fp(const AttentionInput& in, int block_q = 128, int block_kv = 64) {
    if (block_q < 1 || block_kv < 1) throw std::invalid_argument("flash_attention_fp: block sizes must be >= 1");
    b200::validate_input(in, "flash_attention_fp");
    const int n = in.q.tokens, d = in.q.head_dim;
    const float scale = float(1.0 / std::sqrt(double(d)));
    const float ninf = -std::numeric_limits<float>::infinity();
    Tensor4f out(in.q.batch, in.q.heads, n, d);
    Matrix<float> s(block_q, block_kv), acc(block_q, d);
    const size_t rows_per_block = static_cast<size_t>(block_q);
    std::vector<float> m(rows_per_block), l(rows_per_block);
    for (int b = 0; b < in.q.batch; ++b)
        for (int h = 0; h < in.q.heads; ++h) {
            const MatView<float> Q = in.q.slice(b, h), K = in.k.slice(b, h), V = in.v.slice(b, h);
            float* O = out.slice_ptr(b, h);
            for (int r0 = 0, i = 0; r0 < n; r0 += block_q, ++i) {
                const int bq = std::min(block_q, n - r0);
                std::fill(m.begin(), m.end(), ninf);
                std::fill(l.begin(), l.end(), 0.0f);
                std::fill(acc.data.begin(), acc.data.end(), 0.0f);
                for (int c0 = 0, j = 0; c0 < n; c0 += block_kv, ++j) {
                    const int bkv = std::min(block_kv, n - c0);
                    TileKind kind = TileKind::Full;
                    if (in.causal && (kind = apply_causal_tiling(i, j, block_q, block_kv, n)) == TileKind::Skip)
                        continue;
                    for (int r = 0; r < bq; ++r)
                        for (int c = 0; c < bkv; ++c) {
                            float dot = 0.0f;
                            for (int x = 0; x < d; ++x) dot += Q(r0 + r, x) * K(c0 + c, x);
                            s(r, c) = dot * scale;
                            if (kind == TileKind::Diagonal && c0 + c > r0 + r) s(r, c) = ninf;
                        }
                    for (int r = 0; r < bq; ++r) {
                        float mx = m[size_t(r)];
                        for (int c = 0; c < bkv; ++c) mx = std::max(mx, s(r, c));
                        const float alpha = std::exp(m[size_t(r)] - mx);
                        float sum = 0.0f;
                        for (int c = 0; c < bkv; ++c) {
                            const float p = s(r, c) == ninf ? 0.0f : std::exp(s(r, c) - mx);
                            s(r, c) = p;
                            sum += p;
                        }
                        m[size_t(r)] = mx;
                        l[size_t(r)] = alpha * l[size_t(r)] + sum;
                        for (int x = 0; x < d; ++x) acc(r, x) *= alpha;
                        for (int c = 0; c < bkv; ++c) {
                            if (s(r, c) == 0.0f) continue;
                            for (int x = 0; x < d; ++x) acc(r, x) += s(r, c) * V(c0 + c, x);
                        }
                    }
                }
                for (int r = 0; r < bq; ++r) {
                    const float inv = 1.0f / l[size_t(r)];
                    for (int x = 0; x < d; ++x) O[size_t(r0 + r) * size_t(d) + size_t(x)] = acc(r, x) * inv;
                }
            }
        }
    return out;
}

}  // namespace sageattn
