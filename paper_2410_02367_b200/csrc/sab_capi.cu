// sab_capi.cu -- the extern "C" boundary (include/sageattn_b200.h).
//
// Validation mirrors the reference entry (attention.hpp:320-322, 98-103;
// tensor.hpp:70-71); launches K1 (sab_prepass.cu) and K2 (sab_attention.cu);
// the host-buffer entry implements K3, the head x batch partition of
// attention.hpp:357-358 over 1..8 devices (one host thread per device, no
// collective: units are independent).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "sab_internal.h"

using namespace sab;

namespace {

thread_local std::string g_last_error;

int set_error(int status, const std::string& msg) {
    g_last_error = msg;
    return status;
}

int cuda_fail(cudaError_t e, const char* where) {
    return set_error(SAB_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

int64_t units_of(const sab_desc* d) { return int64_t(d->batch) * d->heads; }

int elem_size(int dtype) { return dtype == SAB_F32 ? 4 : 2; }

int layout_of(const sab_desc* d, sab_ws_layout* L) {
    const size_t units = size_t(units_of(d));
    const size_t n = size_t(d->tokens), hd = size_t(d->head_dim);
    const int depth = tree_depth(d->tokens);
    const int npc = nodes_per_cta(depth);
    const int n_partials = (1 << depth) / npc;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t at = off;
        off = align_up(off + bytes, 256);
        return uint64_t(at);
    };
    L->qcodes = take(units * n * hd);
    L->kcodes = take(units * n * hd);
    const bool pt = d->qk_granularity == SAB_QK_PER_TOKEN;
    const size_t npad = (n + kBlockKV - 1) / kBlockKV * kBlockKV;  // per-token rows padded to 64 tokens
    L->qscales = take(units * (pt ? npad : (n + kBlockQ - 1) / kBlockQ) * sizeof(float));
    L->kscales = take(units * (pt ? npad : (n + kBlockKV - 1) / kBlockKV) * sizeof(float));
    L->mean_k = take(units * hd * sizeof(float));
    L->partials = take(units * size_t(n_partials) * hd * sizeof(float));
    const bool pv8 = d->pv_path == SAB_PV_PATH_INT8;
    L->v16 = take(d->in_dtype == SAB_F32 && !pv8 ? units * n * hd * 2 : 0);
    int kv_chunk = 0, nchunk = 1;
    // The INT8 P~V path quantizes P~ against the running row max (quantize_p_static,
    // quant.hpp:258-279), so chunked maxima would change its codes: no split there.  The
    // binary16 accumulator arm keeps one accumulator per row over all keys: no split either.
    if (!pv8 && d->pv_accum == SAB_PV_FP32) kv_split_plan(int64_t(units), d->tokens, d->causal, &kv_chunk, &nchunk);
    const size_t npair = (size_t(d->tokens) + 2 * kBlockQ - 1) / (2 * kBlockQ);
    const size_t items = kv_chunk ? units * npair * size_t(nchunk) : 0;
    // Everything a call must find zeroed is contiguous (one memset per call, see
    // reset_bytes): status word + per-unit K1 counters, static-scale counters, split counters.
    // word, K2 scheduler [2], K1 per-unit counters [3 x units] (mean partials done, mean ready,
    // K chunks past the mean wait) and K1's ticket counter.
    L->status = take(sizeof(int32_t) * (4 + 3 * units));
    L->diag = take(2 * sizeof(unsigned long long));
    L->split_cnt = take(kv_chunk ? 2 * units * npair * sizeof(int32_t) : 0);
    L->vcodes = take(pv8 ? units * hd * npad : 0);
    L->vscales = take(pv8 ? 2 * units * hd * sizeof(float) : 0);
    L->split_o = take(items * 2 * kBlockQ * hd * sizeof(float));
    L->split_ml = take(items * 2 * kBlockQ * 2 * sizeof(float));
    L->kv_chunk = kv_chunk;
    L->kv_nchunk = kv_chunk ? nchunk : 0;
    L->total = off;
    L->n_partials = n_partials;
    L->tree_depth = depth;
    return SAB_OK;
}

template <typename T>
T* at(void* base, uint64_t off) {
    return reinterpret_cast<T*>(static_cast<uint8_t*>(base) + off);
}

PrepassParams prepass_params(const sab_desc* d, const sab_ws_layout& L, const void* q, const void* k, const void* v,
                             void* ws) {
    PrepassParams p{};
    p.q = q;
    p.k = k;
    p.v = v;
    p.qcodes = at<int8_t>(ws, L.qcodes);
    p.kcodes = at<int8_t>(ws, L.kcodes);
    p.qscales = at<float>(ws, L.qscales);
    p.kscales = at<float>(ws, L.kscales);
    p.mean = at<float>(ws, L.mean_k);
    p.partials = at<float>(ws, L.partials);
    const bool pv8 = d->pv_path == SAB_PV_PATH_INT8;
    p.v16 = d->in_dtype == SAB_F32 && !pv8 ? at<uint16_t>(ws, L.v16) : nullptr;
    if (pv8) {
        p.vcodes = at<int8_t>(ws, L.vcodes);
        p.vscales = at<float>(ws, L.vscales);
        p.vamax = reinterpret_cast<int*>(p.vscales + units_of(d) * d->head_dim);
        p.ldv = (d->tokens + kBlockKV - 1) / kBlockKV * kBlockKV;
    }
    p.status = at<int>(ws, L.status);
    p.counters = p.status + 3;
    p.ready = p.counters + units_of(d);
    p.kdone = p.ready + units_of(d);
    p.ticket = p.kdone + units_of(d);
    p.units = int(units_of(d));
    p.n = d->tokens;
    p.d = d->head_dim;
    p.depth = L.tree_depth;
    p.nodes_per_cta = nodes_per_cta(L.tree_depth);
    p.n_partials = L.n_partials;
    p.smooth = d->smooth_k != 0;
    p.per_token = d->qk_granularity == SAB_QK_PER_TOKEN;
    p.check_v = d->check_v != 0 && !pv8;  // the INT8 V pass scans V itself
    p.in_f32 = d->in_dtype == SAB_F32;
    p.inv_n = 1.0f / static_cast<float>(d->tokens);
    p.fold = static_cast<float>(1.0 / std::sqrt(static_cast<double>(d->head_dim)));
    return p;
}

AttnParams attn_params(const sab_desc* d, const sab_ws_layout& L, const void* ws, const void* v, void* o) {
    AttnParams a{};
    void* w = const_cast<void*>(ws);
    a.qcodes = at<int8_t>(w, L.qcodes);
    a.kcodes = at<int8_t>(w, L.kcodes);
    a.qscales = at<float>(w, L.qscales);
    a.kscales = at<float>(w, L.kscales);
    const bool pv8 = d->pv_path == SAB_PV_PATH_INT8;
    a.v16 = pv8 ? nullptr : d->in_dtype == SAB_F32 ? static_cast<const void*>(at<uint16_t>(w, L.v16)) : v;
    if (pv8) {
        a.vcodes = at<int8_t>(w, L.vcodes);
        a.vscales = at<float>(w, L.vscales);
        a.ldv = (d->tokens + kBlockKV - 1) / kBlockKV * kBlockKV;
    }
    a.o = o;
    a.o_v8 = (reinterpret_cast<uintptr_t>(o) & 31u) == 0;
    a.pv16 = !pv8 && d->pv_accum == SAB_PV_FP16;
    a.status = at<int>(w, L.status);
    a.sched = a.status + 1;
    a.units = int(units_of(d));
    a.n = d->tokens;
    a.d = d->head_dim;
    a.causal = d->causal != 0;
    a.out_f32 = d->out_dtype == SAB_F32;
    a.per_token = d->qk_granularity == SAB_QK_PER_TOKEN;
    a.diag = (pv8 && d->measure_static_scale) ? at<unsigned long long>(w, L.diag) : nullptr;
    a.kv_chunk = L.kv_chunk;
    a.nchunk = L.kv_chunk ? L.kv_nchunk : 1;
    a.part_o = L.kv_chunk ? at<float>(w, L.split_o) : nullptr;
    a.part_ml = L.kv_chunk ? at<float2>(w, L.split_ml) : nullptr;
    a.split_cnt = L.kv_chunk ? at<int>(w, L.split_cnt) : nullptr;
    return a;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Bytes from L.status that every call zeroes in one memset: the status word, K1's
// per-unit counters, the static-scale counters and the KV-split counters (the counters
// are self-resetting; zeroing them too means an aborted call leaves nothing stale).
size_t reset_bytes(const sab_ws_layout& L) {
    const size_t end = L.kv_chunk ? L.vcodes : L.split_cnt;  // split_cnt is empty without a split
    return size_t(end - L.status);
}

// K1's grid.y carries the unit index: one device call covers at most 65535 units (the
// host-buffer path splits larger shards into chunks).
constexpr int64_t kMaxUnitsPerLaunch = 65535;

int enqueue_prepass(const sab_desc* d, const sab_ws_layout& L, const void* q, const void* k, const void* v, void* ws,
                    cudaStream_t s, bool reset) {
    if (units_of(d) > kMaxUnitsPerLaunch)
        return set_error(SAB_ERR_UNSUPPORTED, "sab_prepass: batch*heads above 65535 per device call");
    if (reset) {
        cudaError_t e = cudaMemsetAsync(at<uint8_t>(ws, L.status), 0, reset_bytes(L), s);
        if (e != cudaSuccess) return cuda_fail(e, "sab_prepass: status reset");
    }
    cudaError_t e = launch_prepass(prepass_params(d, L, q, k, v, ws), s);
    if (e != cudaSuccess) return cuda_fail(e, "sab_prepass: launch");
    return SAB_OK;
}

int enqueue_attention(const sab_desc* d, const sab_ws_layout& L, void* ws, const void* v, void* o, cudaStream_t s) {
    cudaError_t e = launch_attention(attn_params(d, L, ws, v, o), s);
    if (e != cudaSuccess) return cuda_fail(e, "sab_attention: launch");
    return SAB_OK;
}

// Elements quantize_p_static sees (attention.hpp:485): bq * bkv per non-skipped tile,
// i.e. the S-stage MACs divided by head_dim.
uint64_t static_scale_elements(const sab_desc* d) {
    uint64_t s = 0, p = 0;
    if (sab_diagnostics(d, &s, &p) != SAB_OK) return 0;
    return s / uint64_t(d->head_dim);
}

int map_status_word(int word) {
    if (word & kStatusNonFinite) return set_error(SAB_ERR_NONFINITE, "sage_attention: non-finite input");
    if (word & kStatusOverflow)
        return set_error(SAB_ERR_OVERFLOW, "sage_attention: binary16 P~V accumulator overflowed");
    return SAB_OK;
}

}  // namespace

extern "C" {

const char* sab_status_string(int status) {
    switch (status) {
        case SAB_OK: return "ok";
        case SAB_ERR_SHAPE: return "bad shape or block sizes";
        case SAB_ERR_NONFINITE: return "sage_attention: non-finite input";
        case SAB_ERR_OVERFLOW: return "sage_attention: binary16 P~V accumulator overflowed";
        case SAB_ERR_CUDA: return "CUDA error";
        case SAB_ERR_UNSUPPORTED: return "option outside the SAGEAttn-B B200 path";
        case SAB_ERR_WORKSPACE: return "workspace missing or too small";
        case SAB_ERR_NO_DEVICE: return "no sm_100 device";
        case SAB_ERR_ARGUMENT: return "bad argument";
        default: return "unknown status";
    }
}

const char* sab_last_error(void) { return g_last_error.c_str(); }

int sab_abi_version(void) { return SAB_ABI_VERSION; }

void sab_desc_init(sab_desc* d, int32_t batch, int32_t heads, int32_t tokens, int32_t head_dim, int32_t causal) {
    if (!d) return;
    std::memset(d, 0, sizeof(*d));
    d->batch = batch;
    d->heads = heads;
    d->tokens = tokens;
    d->head_dim = head_dim;
    d->causal = causal;
    d->in_dtype = SAB_F16;
    d->out_dtype = SAB_F32;
    d->block_q = kBlockQ;
    d->block_kv = kBlockKV;
    d->smooth_k = 1;
    d->pv_accum = SAB_PV_FP32;
    d->check_v = 0;
    d->qk_granularity = SAB_QK_PER_BLOCK;
    d->pv_path = SAB_PV_PATH_FP16;
}

int sab_check_desc(const sab_desc* d) {
    if (!d) return set_error(SAB_ERR_ARGUMENT, "sab_desc is NULL");
    if (d->block_q < 1 || d->block_kv < 1)
        return set_error(SAB_ERR_SHAPE, "sage_attention: block sizes must be >= 1");
    if (d->batch < 1 || d->heads < 1 || d->tokens < 1 || d->head_dim < 1)
        return set_error(SAB_ERR_SHAPE, "tensor dimensions must be positive");
    if (d->head_dim != 64 && d->head_dim != 128)
        return set_error(SAB_ERR_UNSUPPORTED, "sage_attention: head_dim must be 64 or 128 on the B200 path");
    if (d->block_q != kBlockQ || d->block_kv != kBlockKV)
        return set_error(SAB_ERR_UNSUPPORTED,
                         "sage_attention: SAGEAttn-B/T use block_q=128, block_kv=64 (kernel_config_for(B|T))");
    if (d->qk_granularity != SAB_QK_PER_BLOCK && d->qk_granularity != SAB_QK_PER_TOKEN)
        return set_error(SAB_ERR_UNSUPPORTED, "sage_attention: Q/K granularity must be per-block (B) or per-token (T)");
    if (d->pv_path != SAB_PV_PATH_FP16 && d->pv_path != SAB_PV_PATH_INT8)
        return set_error(SAB_ERR_UNSUPPORTED, "sage_attention: P~V path must be FP16 (B/T) or INT8 (vB/vT)");
    if ((d->in_dtype != SAB_F16 && d->in_dtype != SAB_F32) || (d->out_dtype != SAB_F16 && d->out_dtype != SAB_F32))
        return set_error(SAB_ERR_ARGUMENT, "sab_desc: dtype must be SAB_F16 or SAB_F32");
    if (d->pv_accum != SAB_PV_FP32 && d->pv_accum != SAB_PV_FP16)
        return set_error(SAB_ERR_UNSUPPORTED, "sage_attention: P~V accumulator must be SAB_PV_FP32 or SAB_PV_FP16");
    if (d->pv_accum == SAB_PV_FP16 && d->pv_path != SAB_PV_PATH_FP16)
        return set_error(SAB_ERR_UNSUPPORTED,
                         "sage_attention: the binary16 P~V accumulator applies to the FP16 P~V path (B/T)");
    if (units_of(d) > (int64_t(1) << 24))
        return set_error(SAB_ERR_UNSUPPORTED, "sage_attention: batch*heads too large");
    // The INT8 P~V path accumulates P~^ V^ in one INT32 TMEM accumulator per row over all
    // keys: each key adds at most 127 * 127, so more than 2^31 / 16129 keys could wrap it.
    if (d->pv_path == SAB_PV_PATH_INT8 && d->tokens > kMaxTokensInt8Pv)
        return set_error(SAB_ERR_UNSUPPORTED,
                         "sage_attention: the INT8 P~V path (vB/vT) supports at most 133144 tokens "
                         "(INT32 P~V accumulator)");
    return SAB_OK;
}

int sab_workspace_layout(const sab_desc* d, sab_ws_layout* layout) {
    int st = sab_check_desc(d);
    if (st) return st;
    if (!layout) return set_error(SAB_ERR_ARGUMENT, "layout is NULL");
    return layout_of(d, layout);
}

int sab_workspace_size(const sab_desc* d, size_t* bytes) {
    sab_ws_layout L;
    int st = sab_workspace_layout(d, &L);
    if (st) return st;
    if (!bytes) return set_error(SAB_ERR_ARGUMENT, "bytes is NULL");
    *bytes = size_t(L.total);
    return SAB_OK;
}

int sab_prepass(const sab_desc* d, const void* q, const void* k, const void* v, void* ws, size_t ws_bytes,
                void* stream) {
    sab_ws_layout L;
    int st = sab_workspace_layout(d, &L);
    if (st) return st;
    if (!q || !k) return set_error(SAB_ERR_ARGUMENT, "sab_prepass: q/k is NULL");
    if ((d->in_dtype == SAB_F32 || d->check_v || d->pv_path == SAB_PV_PATH_INT8) && !v)
        return set_error(SAB_ERR_ARGUMENT, "sab_prepass: v is NULL");
    if (!ws || ws_bytes < L.total) return set_error(SAB_ERR_WORKSPACE, "sab_prepass: workspace too small");
    if (!aligned16(q) || !aligned16(k) || (v && !aligned16(v)) || !aligned16(ws))
        return set_error(SAB_ERR_ARGUMENT, "sab_prepass: pointers must be 16-byte aligned");
    return enqueue_prepass(d, L, q, k, v, ws, static_cast<cudaStream_t>(stream), true);
}

int sab_prepass_rope(const sab_desc* d, const void* q, const void* k, const void* v, const float* cos_table,
                     const float* sin_table, int rope_layout, void* ws, size_t ws_bytes, void* stream) {
    sab_ws_layout L;
    int st = sab_workspace_layout(d, &L);
    if (st) return st;
    if (!q || !k || !cos_table || !sin_table) return set_error(SAB_ERR_ARGUMENT, "sab_prepass_rope: NULL pointer");
    if (rope_layout != SAB_ROPE_INTERLEAVED && rope_layout != SAB_ROPE_HALF)
        return set_error(SAB_ERR_ARGUMENT, "sab_prepass_rope: rope_layout must be SAB_ROPE_INTERLEAVED or SAB_ROPE_HALF");
    if ((d->in_dtype == SAB_F32 || d->check_v || d->pv_path == SAB_PV_PATH_INT8) && !v)
        return set_error(SAB_ERR_ARGUMENT, "sab_prepass_rope: v is NULL");
    if (!ws || ws_bytes < L.total) return set_error(SAB_ERR_WORKSPACE, "sab_prepass_rope: workspace too small");
    if (!aligned16(q) || !aligned16(k) || (v && !aligned16(v)) || !aligned16(ws) || !aligned16(cos_table) ||
        !aligned16(sin_table))
        return set_error(SAB_ERR_ARGUMENT, "sab_prepass_rope: pointers must be 16-byte aligned");
    if (units_of(d) > kMaxUnitsPerLaunch)
        return set_error(SAB_ERR_UNSUPPORTED, "sab_prepass: batch*heads above 65535 per device call");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaMemsetAsync(at<uint8_t>(ws, L.status), 0, reset_bytes(L), s);
    if (e != cudaSuccess) return cuda_fail(e, "sab_prepass_rope: status reset");
    PrepassParams pp = prepass_params(d, L, q, k, v, ws);
    pp.rope = rope_layout;
    pp.rope_cos = cos_table;
    pp.rope_sin = sin_table;
    e = launch_prepass(pp, s);
    if (e != cudaSuccess) return cuda_fail(e, "sab_prepass_rope: launch");
    return SAB_OK;
}

int sab_attention(const sab_desc* d, void* ws, size_t ws_bytes, const void* v, void* o, void* stream) {
    sab_ws_layout L;
    int st = sab_workspace_layout(d, &L);
    if (st) return st;
    if (!ws || ws_bytes < L.total) return set_error(SAB_ERR_WORKSPACE, "sab_attention: workspace too small");
    if (!o || (d->in_dtype == SAB_F16 && d->pv_path != SAB_PV_PATH_INT8 && !v)) return set_error(SAB_ERR_ARGUMENT, "sab_attention: v/o is NULL");
    if (!aligned16(o) || (v && !aligned16(v))) return set_error(SAB_ERR_ARGUMENT, "sab_attention: misaligned v/o");
    return enqueue_attention(d, L, ws, v, o, static_cast<cudaStream_t>(stream));
}

int sab_attention_fwd(const sab_desc* d, const void* q, const void* k, const void* v, void* o, void* ws,
                      size_t ws_bytes, void* stream) {
    int st = sab_prepass(d, q, k, v, ws, ws_bytes, stream);
    if (st) return st;
    return sab_attention(d, ws, ws_bytes, v, o, stream);
}

int sab_read_status(const sab_desc* d, const void* ws, void* stream, int* status) {
    sab_ws_layout L;
    int st = sab_workspace_layout(d, &L);
    if (st) return st;
    if (!ws || !status) return set_error(SAB_ERR_ARGUMENT, "sab_read_status: NULL argument");
    int word = 0;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaMemcpyAsync(&word, at<int>(const_cast<void*>(ws), L.status), sizeof(int),
                                    cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "sab_read_status");
    *status = map_status_word(word);
    return SAB_OK;
}

int sab_shard_plan(int units, int n_shards, int s, int* first, int* count) {
    if (units < 0 || n_shards < 1 || s < 0 || s >= n_shards || !first || !count)
        return set_error(SAB_ERR_ARGUMENT, "sab_shard_plan: bad argument");
    const int base = units / n_shards, rem = units % n_shards;
    *count = base + (s < rem ? 1 : 0);
    *first = s * base + std::min(s, rem);
    return SAB_OK;
}

int sab_diagnostics(const sab_desc* d, uint64_t* s_stage_macs, uint64_t* pv_stage_macs) {
    if (!d || !s_stage_macs || !pv_stage_macs) return set_error(SAB_ERR_ARGUMENT, "sab_diagnostics: NULL argument");
    if (d->block_q < 1 || d->block_kv < 1) return set_error(SAB_ERR_SHAPE, "sage_attention: block sizes must be >= 1");
    if (d->batch < 1 || d->heads < 1 || d->tokens < 1 || d->head_dim < 1)
        return set_error(SAB_ERR_SHAPE, "tensor dimensions must be positive");
    // attention.hpp:396-404: every non-skipped (i, j) tile adds bq * bkv * d.
    const int64_t n = d->tokens, bq = d->block_q, bkv = d->block_kv;
    uint64_t per_unit = 0;
    for (int64_t r0 = 0; r0 < n; r0 += bq) {
        const int64_t rows = std::min(bq, n - r0), r1 = r0 + rows - 1;
        if (!d->causal) {
            per_unit += uint64_t(rows) * uint64_t(n);
            continue;
        }
        for (int64_t c0 = 0; c0 < n && c0 <= r1; c0 += bkv) per_unit += uint64_t(rows) * uint64_t(std::min(bkv, n - c0));
    }
    const uint64_t macs = per_unit * uint64_t(d->head_dim) * uint64_t(units_of(d));
    *s_stage_macs = macs;
    *pv_stage_macs = macs;
    return SAB_OK;
}

int sab_device_ordinals(int* ordinals, int capacity, int* count) {
    if (!count || (capacity > 0 && !ordinals)) return set_error(SAB_ERR_ARGUMENT, "sab_device_ordinals: NULL argument");
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) n = 0;
    int c = 0;
    for (int i = 0; i < n; ++i) {
        int major = 0, minor = 0;
        if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, i) == cudaSuccess &&
            cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, i) == cudaSuccess && major == 10 &&
            minor == 0) {
            if (c < capacity) ordinals[c] = i;
            ++c;
        }
    }
    *count = c;
    return SAB_OK;
}

int sab_device_count(int* count) {
    if (!count) return set_error(SAB_ERR_ARGUMENT, "count is NULL");
    return sab_device_ordinals(nullptr, 0, count);
}

int sab_qk_int32_tiles(const sab_desc* d, const void* ws, int unit, int q_tile, int32_t* s_out, void* stream) {
    sab_ws_layout L;
    int st = sab_workspace_layout(d, &L);
    if (st) return st;
    const int ntq = (d->tokens + kBlockQ - 1) / kBlockQ;
    if (!ws || !s_out || unit < 0 || unit >= units_of(d) || q_tile < 0 || q_tile >= ntq)
        return set_error(SAB_ERR_ARGUMENT, "sab_qk_int32_tiles: bad argument");
    AttnParams a = attn_params(d, L, ws, nullptr, nullptr);
    if (d->in_dtype == SAB_F16) a.v16 = at<uint16_t>(const_cast<void*>(ws), L.qcodes);  // any valid mapping; V unused
    a.s_dump = s_out;
    a.dump_unit = unit;
    a.dump_qtile = q_tile;
    cudaError_t e = launch_qk_dump(a, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "sab_qk_int32_tiles");
    return SAB_OK;
}

// ----------------------------------------------------------------- K3 host path
namespace {

// Per-device execution context of the host-buffer path: three streams
// (H2D / compute / D2H), per-chunk events, grow-only device buffers and, for
// pageable caller buffers, two pinned staging slots per direction.  Contexts
// are pooled so repeated calls do not pay cudaMalloc / cudaHostAlloc / stream
// creation; a context is owned by one call at a time, so concurrent callers
// never share buffers (the reference entry is re-entrant, attention.hpp:9-12).
struct DevCtx {
    int device = -1;
    cudaStream_t s_in = nullptr, s_out = nullptr;
    cudaStream_t s_cmp[2] = {nullptr, nullptr};  // chunks alternate: adjacent chunks' kernels overlap
    std::vector<cudaEvent_t> ev_in, ev_cmp, ev_out;
    uint8_t* buf = nullptr;
    size_t buf_bytes = 0;
    uint8_t* pin_in[2] = {nullptr, nullptr};   // staging of Q, K, V chunks
    uint8_t* pin_out[2] = {nullptr, nullptr};  // staging of O chunks
    size_t pin_in_bytes = 0, pin_out_bytes = 0;
};

std::mutex g_pool_mu;
std::vector<DevCtx*> g_pool;

cudaError_t ctx_reserve(DevCtx* c, size_t bytes, int n_events) {
    cudaError_t e = cudaSuccess;
    if (!c->s_in) {
        if ((e = cudaStreamCreateWithFlags(&c->s_in, cudaStreamNonBlocking)) != cudaSuccess ||
            (e = cudaStreamCreateWithFlags(&c->s_cmp[0], cudaStreamNonBlocking)) != cudaSuccess ||
            (e = cudaStreamCreateWithFlags(&c->s_cmp[1], cudaStreamNonBlocking)) != cudaSuccess ||
            (e = cudaStreamCreateWithFlags(&c->s_out, cudaStreamNonBlocking)) != cudaSuccess)
            return e;
    }
    while (int(c->ev_in.size()) < n_events) {
        cudaEvent_t a, b, o;
        if ((e = cudaEventCreateWithFlags(&a, cudaEventDisableTiming)) != cudaSuccess) return e;
        if ((e = cudaEventCreateWithFlags(&b, cudaEventDisableTiming)) != cudaSuccess) return e;
        if ((e = cudaEventCreateWithFlags(&o, cudaEventDisableTiming)) != cudaSuccess) return e;
        c->ev_in.push_back(a);
        c->ev_cmp.push_back(b);
        c->ev_out.push_back(o);
    }
    if (c->buf_bytes < bytes) {
        if (c->buf) cudaFree(c->buf);
        c->buf = nullptr;
        c->buf_bytes = 0;
        if ((e = cudaMalloc(&c->buf, bytes)) != cudaSuccess) return e;
        c->buf_bytes = bytes;
    }
    return e;
}

cudaError_t ctx_reserve_pinned(DevCtx* c, size_t in_bytes, size_t out_bytes) {
    cudaError_t e = cudaSuccess;
    if (c->pin_in_bytes < in_bytes) {
        for (auto& p : c->pin_in) {
            if (p) cudaFreeHost(p);
            p = nullptr;
        }
        c->pin_in_bytes = 0;
        for (auto& p : c->pin_in)
            if ((e = cudaHostAlloc(reinterpret_cast<void**>(&p), in_bytes, cudaHostAllocPortable)) != cudaSuccess)
                return e;
        c->pin_in_bytes = in_bytes;
    }
    if (c->pin_out_bytes < out_bytes) {
        for (auto& p : c->pin_out) {
            if (p) cudaFreeHost(p);
            p = nullptr;
        }
        c->pin_out_bytes = 0;
        for (auto& p : c->pin_out)
            if ((e = cudaHostAlloc(reinterpret_cast<void**>(&p), out_bytes, cudaHostAllocPortable)) != cudaSuccess)
                return e;
        c->pin_out_bytes = out_bytes;
    }
    return e;
}

DevCtx* ctx_acquire(int device) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    for (size_t i = 0; i < g_pool.size(); ++i) {
        if (g_pool[i]->device == device) {
            DevCtx* c = g_pool[i];
            g_pool.erase(g_pool.begin() + i);
            return c;
        }
    }
    DevCtx* c = new DevCtx;
    c->device = device;
    return c;
}

void ctx_release(DevCtx* c) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    g_pool.push_back(c);
}

// True when `p` is ordinary pageable host memory (not cudaHostAlloc'ed or
// registered): copies from it would serialise behind the driver's own bounce
// buffer, so the host path stages it through pinned slots instead.
bool is_pageable(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();  // clear the sticky-free error of an unknown pointer
        return true;
    }
    return a.type == cudaMemoryTypeUnregistered;
}

// memcpy split over `threads` host threads (host memory bandwidth needs several
// cores; one core copies at roughly a third of PCIe Gen5 speed).
void par_copy(void* dst, const void* src, size_t bytes, int threads) {
    constexpr size_t kMinPiece = size_t(4) << 20;
    threads = int(std::max<size_t>(1, std::min<size_t>(size_t(threads), bytes / kMinPiece)));
    if (threads <= 1) {
        std::memcpy(dst, src, bytes);
        return;
    }
    const size_t piece = (bytes + threads - 1) / threads;
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) {
        const size_t a = size_t(t) * piece, b = std::min(bytes, a + piece);
        if (a < b)
            pool.emplace_back([=] { std::memcpy(static_cast<uint8_t*>(dst) + a, static_cast<const uint8_t*>(src) + a, b - a); });
    }
    std::memcpy(dst, src, std::min(bytes, piece));
    for (auto& t : pool) t.join();
}

struct ShardJob {
    const sab_desc* desc;
    const uint8_t *q, *k, *v;
    uint8_t* o;
    int device;
    int first, count;
    int copy_threads;  // host threads per staging copy
    int status;
    std::string error;
    unsigned long long mismatches[2] = {0, 0};  // static-scale P~ diagnostics of this shard
};

// Test / tuning knobs of the host-buffer path (read once): SAB_HOST_CHUNK_UNITS forces
// the units per (full) chunk, SAB_HOST_RAMP=0 turns the size ramp off, SAB_HOST_STREAMS=1
// keeps every chunk on one compute stream.
int host_chunk_units() {
    static const int v = [] {
        const char* e = std::getenv("SAB_HOST_CHUNK_UNITS");
        return e ? std::atoi(e) : 0;
    }();
    return v;
}
// Host threads per staging copy of a shard: SAB_HOST_COPY_THREADS, else up to 8 per device.
int host_copy_threads(int n_devices) {
    static const int forced = [] {
        const char* e = std::getenv("SAB_HOST_COPY_THREADS");
        return e ? std::atoi(e) : 0;
    }();
    if (forced > 0) return forced;
    return std::max(1, std::min(8, int(std::thread::hardware_concurrency()) / std::max(1, n_devices)));
}
int host_ramp() {
    static const int v = [] {
        const char* e = std::getenv("SAB_HOST_RAMP");
        return e ? std::atoi(e) : 1;
    }();
    return v;
}
int host_compute_streams() {
    static const int v = [] {
        const char* e = std::getenv("SAB_HOST_STREAMS");
        return e ? std::max(1, std::atoi(e)) : 2;
    }();
    return v;
}

int run_shard_on(ShardJob* job, DevCtx* ctx) {
    const sab_desc* D = job->desc;
    const size_t in_e = elem_size(D->in_dtype), out_e = elem_size(D->out_dtype);
    const size_t unit_elems = size_t(D->tokens) * D->head_dim;
    // Chunks of whole units (up to ~128 MB of inputs, and at least ~4 full chunks when
    // the shard allows) so that H2D of chunk c+1, compute of chunk c and D2H of chunk
    // c-1 overlap on the three streams.  The sizes ramp 1, 2, 4, ... units up to that
    // and back down at the end: the un-overlapped first H2D and last compute + D2H
    // are one unit's worth, while the middle chunks are large enough that per-copy
    // overheads and partial K2 waves stay small.
    const size_t unit_in_bytes = 3 * unit_elems * in_e;
    const size_t by_bytes = std::max<size_t>(1, (128u << 20) / unit_in_bytes);
    const size_t by_count = std::max<size_t>(1, size_t(job->count) / 4);
    int chunk = int(std::max<size_t>(
        1, std::min<size_t>(std::min<size_t>(job->count, size_t(kMaxUnitsPerLaunch)), std::min(by_bytes, by_count))));
    if (const int forced = host_chunk_units(); forced > 0)
        chunk = std::min(std::min(forced, job->count), int(kMaxUnitsPerLaunch));
    std::vector<int> starts{0};
    {
        std::vector<int> up;
        int ramp = 0;
        if (host_ramp())
            for (int sz = 1; sz < chunk && 2 * (ramp + sz) + chunk <= job->count; sz *= 2) up.push_back(sz), ramp += sz;
        auto push = [&](int sz) { starts.push_back(starts.back() + sz); };
        for (int sz : up) push(sz);
        for (int rem = job->count - 2 * ramp; rem > 0; rem -= std::min(chunk, rem)) push(std::min(chunk, rem));
        for (auto it = up.rbegin(); it != up.rend(); ++it) push(*it);
    }
    const int n_chunks = int(starts.size()) - 1;
    // Chunks alternate between two compute streams, each with its own workspace, so the
    // tail wave of chunk c's K2 overlaps chunk c+1's K1 and first wave.
    const int ncs = (n_chunks > 1 && host_compute_streams() > 1) ? 2 : 1;

    sab_desc cd = *D;
    cd.batch = 1;
    cd.heads = chunk;
    sab_ws_layout L;
    layout_of(&cd, &L);

    const size_t in_bytes = align_up(size_t(job->count) * unit_elems * in_e, 256);
    const size_t out_bytes = align_up(size_t(job->count) * unit_elems * out_e, 256);
    const size_t ws_bytes = align_up(L.total, 256);
    cudaError_t e = ctx_reserve(ctx, 3 * in_bytes + out_bytes + ncs * ws_bytes, n_chunks);
    if (e != cudaSuccess) return cuda_fail(e, "sab_attention_fwd_host: device buffers");
    // Pageable caller buffers go through two pinned slots per direction: the host
    // thread copies chunk c into slot c % 2 while the GPU reads chunk c - 1 from the
    // other slot (and the same, reversed, for O).
    const uint8_t* src_in[3] = {job->q, job->k, job->v};
    bool stage_in[3], stage_out = is_pageable(job->o);
    bool any_in = false;
    for (int t = 0; t < 3; ++t) any_in |= (stage_in[t] = is_pageable(src_in[t]));
    const size_t chunk_in = size_t(chunk) * unit_elems * in_e, chunk_out = size_t(chunk) * unit_elems * out_e;
    if (any_in || stage_out) {
        e = ctx_reserve_pinned(ctx, any_in ? 3 * chunk_in : 0, stage_out ? chunk_out : 0);
        if (e != cudaSuccess) return cuda_fail(e, "sab_attention_fwd_host: pinned staging buffers");
    }
    uint8_t* dev_in[3] = {ctx->buf, ctx->buf + in_bytes, ctx->buf + 2 * in_bytes};
    uint8_t* dout = ctx->buf + 3 * in_bytes;
    uint8_t* wss[2] = {dout + out_bytes, dout + out_bytes + ws_bytes};

    for (int i = 0; i < ncs; ++i)
        if ((e = cudaMemsetAsync(wss[i] + L.status, 0, reset_bytes(L), ctx->s_cmp[i])) != cudaSuccess)
            return cuda_fail(e, "sab_attention_fwd_host: memset");
    // Copies the finished O of chunk c out of its pinned slot into the caller's buffer.
    auto drain_out = [&](int c) -> cudaError_t {
        const int u0 = starts[c], cu = starts[c + 1] - starts[c];
        cudaError_t x = cudaEventSynchronize(ctx->ev_out[c]);
        if (x == cudaSuccess)
            par_copy(job->o + size_t(u0) * unit_elems * out_e, ctx->pin_out[c % 2], size_t(cu) * unit_elems * out_e,
                     job->copy_threads);
        return x;
    };
    int st = SAB_OK;
    for (int c = 0; c < n_chunks && st == SAB_OK; ++c) {
        const int u0 = starts[c], cu = starts[c + 1] - starts[c];
        const size_t ioff = size_t(u0) * unit_elems * in_e, ibytes = size_t(cu) * unit_elems * in_e;
        const size_t ooff = size_t(u0) * unit_elems * out_e, obytes = size_t(cu) * unit_elems * out_e;
        const int slot = c % 2;
        cudaStream_t scmp = ctx->s_cmp[c % ncs];
        uint8_t* ws = wss[c % ncs];
        // The slot was last read by the H2D of chunk c - 2.
        if (any_in && c >= 2 && (e = cudaEventSynchronize(ctx->ev_in[c - 2])) != cudaSuccess) {
            st = cuda_fail(e, "sab_attention_fwd_host: staging");
            break;
        }
        for (int t = 0; t < 3 && e == cudaSuccess; ++t) {
            const uint8_t* from = src_in[t] + ioff;
            if (stage_in[t]) {
                uint8_t* pinned = ctx->pin_in[slot] + size_t(t) * chunk_in;
                par_copy(pinned, from, ibytes, job->copy_threads);
                from = pinned;
            }
            e = cudaMemcpyAsync(dev_in[t] + ioff, from, ibytes, cudaMemcpyHostToDevice, ctx->s_in);
        }
        if (e != cudaSuccess || (e = cudaEventRecord(ctx->ev_in[c], ctx->s_in)) != cudaSuccess ||
            (e = cudaStreamWaitEvent(scmp, ctx->ev_in[c], 0)) != cudaSuccess) {
            st = cuda_fail(e, "sab_attention_fwd_host: H2D");
            break;
        }
        // A short last chunk keeps the full-chunk layout L (every region is sized for
        // `chunk` units, so `cu` units fit): only the unit count changes.  A layout
        // recomputed for `cu` units would move the regions after the status word
        // (V^ / delta_V of the INT8 P~V path) on top of it.
        sab_desc xd = cd;
        xd.heads = cu;
        if ((st = enqueue_prepass(&xd, L, dev_in[0] + ioff, dev_in[1] + ioff, dev_in[2] + ioff, ws, scmp, false)) !=
            SAB_OK)
            break;
        if ((st = enqueue_attention(&xd, L, ws, dev_in[2] + ioff, dout + ooff, scmp)) != SAB_OK) break;
        // The O slot of chunk c was last filled by chunk c - 2, drained below at step c - 1.
        if ((e = cudaEventRecord(ctx->ev_cmp[c], scmp)) != cudaSuccess ||
            (e = cudaStreamWaitEvent(ctx->s_out, ctx->ev_cmp[c], 0)) != cudaSuccess ||
            (e = cudaMemcpyAsync(stage_out ? ctx->pin_out[slot] : job->o + ooff, dout + ooff, obytes,
                                 cudaMemcpyDeviceToHost, ctx->s_out)) != cudaSuccess ||
            (e = cudaEventRecord(ctx->ev_out[c], ctx->s_out)) != cudaSuccess) {
            st = cuda_fail(e, "sab_attention_fwd_host: D2H");
            break;
        }
        if (stage_out && c >= 1 && (e = drain_out(c - 1)) != cudaSuccess) {
            st = cuda_fail(e, "sab_attention_fwd_host: D2H staging");
            break;
        }
    }
    if (st == SAB_OK && stage_out && (e = drain_out(n_chunks - 1)) != cudaSuccess)
        st = cuda_fail(e, "sab_attention_fwd_host: D2H staging");
    int word[2] = {0, 0};
    unsigned long long mism[2][2] = {{0, 0}, {0, 0}};
    for (int i = 0; i < ncs && st == SAB_OK; ++i) {
        if ((e = cudaMemcpyAsync(&word[i], wss[i] + L.status, sizeof(int), cudaMemcpyDeviceToHost, ctx->s_cmp[i])) !=
            cudaSuccess)
            st = cuda_fail(e, "sab_attention_fwd_host: status");
        else if (D->measure_static_scale &&
                 (e = cudaMemcpyAsync(mism[i], wss[i] + L.diag, sizeof(mism[i]), cudaMemcpyDeviceToHost,
                                      ctx->s_cmp[i])) != cudaSuccess)
            st = cuda_fail(e, "sab_attention_fwd_host: diagnostics");
    }
    // Always drain every stream before the context is reused.
    cudaError_t es[4] = {cudaStreamSynchronize(ctx->s_in), cudaStreamSynchronize(ctx->s_cmp[0]),
                         cudaStreamSynchronize(ctx->s_cmp[1]), cudaStreamSynchronize(ctx->s_out)};
    if (st == SAB_OK) {
        for (cudaError_t x : es)
            if (x != cudaSuccess) return cuda_fail(x, "sab_attention_fwd_host: sync");
        job->mismatches[0] = mism[0][0] + mism[1][0];
        job->mismatches[1] = mism[0][1] + mism[1][1];
        st = map_status_word(word[0]);
        if (st == SAB_OK) st = map_status_word(word[1]);
    }
    return st;
}

// Restores the calling thread's current device on scope exit: the single-device
// call runs its shard on the caller's thread and must not leave it switched.
struct DeviceGuard {
    int saved = -1;
    DeviceGuard() {
        if (cudaGetDevice(&saved) != cudaSuccess) saved = -1;
    }
    ~DeviceGuard() {
        if (saved >= 0) cudaSetDevice(saved);
    }
};

void run_shard(ShardJob* job) {
    DeviceGuard guard;
    cudaError_t e = cudaSetDevice(job->device);
    int st;
    if (e != cudaSuccess) {
        st = cuda_fail(e, "cudaSetDevice");
    } else {
        DevCtx* ctx = ctx_acquire(job->device);
        st = run_shard_on(job, ctx);
        ctx_release(ctx);
    }
    job->status = st;
    if (st != SAB_OK) job->error = g_last_error;
}

}  // namespace

int sab_attention_fwd_host(const sab_desc* d, const void* q, const void* k, const void* v, void* o,
                           const int* devices, int n_devices) {
    return sab_attention_fwd_host_diag(d, q, k, v, o, devices, n_devices, nullptr);
}

int sab_attention_fwd_host_diag(const sab_desc* d, const void* q, const void* k, const void* v, void* o,
                                const int* devices, int n_devices, uint64_t counts[3]) {
    if (counts) counts[0] = counts[1] = counts[2] = 0;
    int st = sab_check_desc(d);
    if (st) return st;
    if (!q || !k || !v || !o) return set_error(SAB_ERR_ARGUMENT, "sab_attention_fwd_host: NULL buffer");
    int avail = 0;
    if (cudaGetDeviceCount(&avail) != cudaSuccess || avail < 1)
        return set_error(SAB_ERR_NO_DEVICE, "sab_attention_fwd_host: no CUDA device");
    if (n_devices < 1) n_devices = 1;
    std::vector<int> devs(n_devices);
    for (int i = 0; i < n_devices; ++i) {
        devs[i] = devices ? devices[i] : i;
        if (devs[i] < 0 || devs[i] >= avail)
            return set_error(SAB_ERR_NO_DEVICE, "sab_attention_fwd_host: device ordinal out of range");
    }
    const int units = int(units_of(d));
    const size_t in_unit = size_t(d->tokens) * d->head_dim * elem_size(d->in_dtype);
    const size_t out_unit = size_t(d->tokens) * d->head_dim * elem_size(d->out_dtype);
    std::vector<ShardJob> jobs(n_devices);
    for (int s = 0; s < n_devices; ++s) {
        ShardJob& j = jobs[s];
        j.desc = d;
        j.device = devs[s];
        sab_shard_plan(units, n_devices, s, &j.first, &j.count);
        j.q = static_cast<const uint8_t*>(q) + j.first * in_unit;
        j.k = static_cast<const uint8_t*>(k) + j.first * in_unit;
        j.v = static_cast<const uint8_t*>(v) + j.first * in_unit;
        j.o = static_cast<uint8_t*>(o) + j.first * out_unit;
        j.copy_threads = host_copy_threads(n_devices);
        j.status = SAB_OK;
    }
    if (n_devices == 1) {
        if (jobs[0].count > 0) run_shard(&jobs[0]);
    } else {
        std::vector<std::thread> pool;
        for (auto& j : jobs)
            if (j.count > 0) pool.emplace_back(run_shard, &j);
        for (auto& t : pool) t.join();
    }
    // Same precedence as the reference: validation errors before overflow.
    int worst = SAB_OK;
    std::string msg;
    for (auto& j : jobs) {
        if (j.status == SAB_OK) continue;
        if (worst == SAB_OK || j.status == SAB_ERR_NONFINITE || (worst == SAB_ERR_OVERFLOW)) {
            worst = j.status;
            msg = j.error;
        }
    }
    if (worst != SAB_OK) return set_error(worst, msg);
    if (counts && d->measure_static_scale && d->pv_path == SAB_PV_PATH_INT8) {
        counts[0] = static_scale_elements(d);
        for (auto& j : jobs) {
            counts[1] += j.mismatches[0];
            counts[2] += j.mismatches[1];
        }
    }
    return SAB_OK;
}

int sab_read_static_scale_counts(const sab_desc* d, const void* ws, void* stream, uint64_t counts[3]) {
    sab_ws_layout L;
    int st = sab_workspace_layout(d, &L);
    if (st) return st;
    if (!ws || !counts) return set_error(SAB_ERR_ARGUMENT, "sab_read_static_scale_counts: NULL argument");
    unsigned long long m[2] = {0, 0};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaMemcpyAsync(m, at<uint8_t>(const_cast<void*>(ws), L.diag), sizeof(m), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "sab_read_static_scale_counts");
    const bool on = d->measure_static_scale && d->pv_path == SAB_PV_PATH_INT8;
    counts[0] = on ? static_scale_elements(d) : 0;
    counts[1] = on ? m[0] : 0;
    counts[2] = on ? m[1] : 0;
    return SAB_OK;
}

}  // extern "C"
