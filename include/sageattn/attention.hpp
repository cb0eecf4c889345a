// sageattn/attention.hpp -- B200 drop-in for the reference's SAGEAttn-B / -T entry point.
//
// Source-compatible replacement for /root/reference/proj/include/sageattn/
// attention.hpp as far as the SAGEAttn-B hot path goes: an application that
// calls
//     sageattn::sage_attention(const AttentionInput&, SageVariant::B | SageVariant::T, const SageOptions&)
//     sageattn::sage_attention(const AttentionInput&, const KernelConfig&, const SageOptions&)
// (attention.hpp:318-319, 547-550) switches to the B200 path by putting
// <repo>/include first on its include path and linking
// paper_2410_02367_b200/libsageattn_b200.so.  Everything below is a thin
// header over the C ABI in sageattn_b200.h; the arithmetic runs in the CUDA
// kernels (K1 prepass + K2 tcgen05 attention, K3 head x batch sharding).
//
// Kept from the reference contract:
//   * the types AttentionInput, KernelConfig, QkGranularity, PvPath, SageVariant,
//     SageOptions, SageDiagnostics, QuantDtype, Tensor4f / Tensor4d, TileKind with
//     the same members and layouts (tensor.hpp:58-107 (B,H,N,d) row-major);
//   * kernel_config_for, apply_causal_tiling;
//   * exceptions and messages: std::invalid_argument for bad block sizes,
//     shape mismatch and non-finite input, std::overflow_error for a non-finite
//     P~V accumulator (attention.hpp:84-102, 321, 531-533);
//   * pure / re-entrant calls (per-call device contexts, attention.hpp:9-12).
// Differences (documented in INTEGRATION.md):
//   * the four variants B, T (Fp16Acc P~V) and vB, vT (INT8 P~V) with
//     block 128/64 and INT8 run; FP8 dtypes or other block sizes throw
//     std::invalid_argument -- there is no CPU fallback;
//   * head_dim must be 64 or 128;
//   * P~V accumulates in FP32 on the tensor cores (the reference's
//     pv_fp32_accumulator arm) whatever pv_fp32_accumulator says; Q^/K^ codes,
//     scales and mean(K) are bit-identical to the reference.
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "../sageattn_b200.h"

namespace sageattn {

enum class QuantDtype : uint8_t { Int8, FpE4M3, FpE5M2 };

// Dense (batch, heads, tokens, head_dim) container; each (b, h) slice is a
// contiguous tokens x head_dim block.
template <typename T>
struct Tensor4 {
    int batch = 0, heads = 0, tokens = 0, head_dim = 0;
    std::vector<T> data;

    Tensor4() = default;
    Tensor4(int b, int h, int n, int d, T fill = T{}) : batch(b), heads(h), tokens(n), head_dim(d) {
        if (b < 1 || h < 1 || n < 1 || d < 1) throw std::invalid_argument("tensor dimensions must be positive");
        data.assign(size_t(b) * size_t(h) * size_t(n) * size_t(d), fill);
    }
    size_t size() const { return data.size(); }
    size_t offset(int b, int h, int t, int c) const {
        return ((size_t(b) * size_t(heads) + size_t(h)) * size_t(tokens) + size_t(t)) * size_t(head_dim) + size_t(c);
    }
    T& at(int b, int h, int t, int c) { return data[offset(b, h, t, c)]; }
    const T& at(int b, int h, int t, int c) const { return data[offset(b, h, t, c)]; }
    T* slice_ptr(int b, int h) { return data.data() + offset(b, h, 0, 0); }
    const T* slice_ptr(int b, int h) const { return data.data() + offset(b, h, 0, 0); }
    std::span<const T> slice_span(int b, int h) const {
        return {slice_ptr(b, h), size_t(tokens) * size_t(head_dim)};
    }
    bool same_shape(const Tensor4& o) const {
        return batch == o.batch && heads == o.heads && tokens == o.tokens && head_dim == o.head_dim;
    }
    bool all_finite() const {
        for (const T& v : data)
            if (!std::isfinite(static_cast<double>(v))) return false;
        return true;
    }
};

using Tensor4f = Tensor4<float>;
using Tensor4d = Tensor4<double>;

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
    const int r1 = (r0 + block_q < n_tokens ? r0 + block_q : n_tokens) - 1;
    const int c1 = (c0 + block_kv < n_tokens ? c0 + block_kv : n_tokens) - 1;
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

// Devices used by the host-buffer path (K3 sharding); 0 = all visible.
inline int& device_count_override() {
    static int n = 1;
    return n;
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
    Tensor4f out(in.q.batch, in.q.heads, in.q.tokens, in.q.head_dim);
    int n_dev = b200::device_count_override();
    if (n_dev <= 0) sab_device_count(&n_dev);
    b200::throw_status(sab_attention_fwd_host(&d, in.q.data.data(), in.k.data.data(), in.v.data.data(),
                                              out.data.data(), nullptr, n_dev > 0 ? n_dev : 1));
    if (options.diagnostics) {
        uint64_t s = 0, p = 0;
        b200::throw_status(sab_diagnostics(&d, &s, &p));
        options.diagnostics->s_stage_macs += s;
        options.diagnostics->pv_stage_macs += p;
    }
    return out;
}

inline Tensor4f sage_attention(const AttentionInput& in, SageVariant variant, const SageOptions& options = {}) {
    return sage_attention(in, kernel_config_for(variant), options);
}

}  // namespace sageattn
