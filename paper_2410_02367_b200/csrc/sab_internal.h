// sab_internal.h -- launch parameters shared by the C-ABI layer and kernels.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <utility>
#include <cuda_runtime.h>

#include "../../include/sageattn_b200.h"

namespace sab {

constexpr int kBlockQ = 128;    // query tile = Q quantization group (attention.hpp:51, 344)
constexpr int kBlockKV = 64;    // K quantization group (attention.hpp:51, 345)
constexpr int kTileN = 64;      // keys per K2 KV tile (one K group)
// vB/vT: INT32 P~^V^ accumulator bound, floor((2^31 - 1) / (127 * 127)) keys.
constexpr int kMaxTokensInt8Pv = 133144;

// Device status word bits (mapped to sab_status by sab_read_status).
constexpr int kStatusNonFinite = 1;
constexpr int kStatusOverflow = 2;

struct PrepassParams {
    const void* q;
    const void* k;
    const void* v;
    int8_t* qcodes;
    int8_t* kcodes;
    float* qscales;
    float* kscales;
    float* mean;
    float* partials;
    uint16_t* v16;
    int* status;
    int* counters;      // per unit: mean-partial CTAs done (self-resetting, zeroed with status)
    int* ready;         // per unit: mean(K) written (k1_fused; self-resetting)
    int* kdone;         // per unit: K chunks past their mean(K) wait (k1_fused; self-resetting)
    int* ticket;        // k1_fused: next work-item ticket (self-resetting)
    int lag;            // k1_fused: K chunks of unit u are issued in stage u + lag
    int units, n, d;
    int depth;          // tree depth of the 4..9-token node level
    int nodes_per_cta;  // nodes summed per mean-partial CTA (power of two)
    int n_partials;     // 2^depth / nodes_per_cta
    int smooth;
    int per_token;      // SAGEAttn-T: one scale per token (qscales/kscales [units][n])
    int8_t* vcodes;     // vB: per-channel INT8 V^, transposed [units][d][ldv] (NULL: FP16 P~V path)
    float* vscales;     // vB: delta_V [units][d]
    int* vamax;         // vB: channel max |v| as float bits [units][d] (zeroed by launch_prepass)
    int ldv;            // vB: tokens padded to 64
    int check_v;
    int in_f32;
    float inv_n;        // 1.0f / float(N)          (quant.hpp:228)
    float fold;         // float(1/sqrt(double(d)))  (quant.hpp:249)
    // RoPE fused into the quantizer (sab_prepass_rope): Q and K are rotated
    // in binary32 on load, before the smooth / fold / quantize.  0 = off.
    int rope;           // SAB_ROPE_INTERLEAVED / SAB_ROPE_HALF
    const float* rope_cos;  // [n][d/2] per token position and channel pair
    const float* rope_sin;
};

// Mean-tree geometry for N tokens (quant.hpp:203-213): the smallest depth at
// which every node holds <= 9 tokens (floor(N/2^depth) < 9).
int tree_depth(int n);
int nodes_per_cta(int depth);

cudaError_t launch_prepass(const PrepassParams& p, cudaStream_t s);

struct AttnParams {
    const int8_t* qcodes;
    const int8_t* kcodes;
    const float* qscales;
    const float* kscales;
    const void* v16;
    const int8_t* vcodes;  // vB: INT8 V^ [units][d][ldv] (P~V kind::i8), else NULL
    const float* vscales;  // vB: delta_V [units][d]
    int ldv;
    void* o;
    int* status;
    int32_t* s_dump;  // debug: INT32 S tiles of one (unit, q-tile)
    int units, n, d, causal, out_f32, per_token;
    int dump_unit, dump_qtile;
    int group_units;  // K2 raster: units per L2-resident group (set by launch_attention)
    unsigned long long* diag;  // vB/vT static-scale P~ mismatches [first block, later blocks], or NULL
    // KV split (sab_ws_layout::kv_chunk): chunk c of a pair covers KV tiles
    // [c * kv_chunk, (c + 1) * kv_chunk); grid.y = nchunk.
    int kv_chunk, nchunk;
    // Persistent K2 (set by launch_attention): `items` work items over min(items, SMs)
    // CTAs, taken from the self-resetting counters sched[0] (next item) / sched[1] (CTAs
    // done) in the status block; persist == 0: one CTA per item.
    int items, persist;
    int o_v8;  // O is 32-byte aligned: the epilogue writes with 32-byte stores
    int pv16;  // SAB_PV_FP16: P~V accumulates in a binary16 TMEM accumulator (never KV-split)
    int* sched;
    float* part_o;          // [units][npair][nchunk][d/4][256] float4 groups of unnormalised partial O
    float2* part_ml;        // [units][npair][nchunk][256] (m, l)
    int* split_cnt;         // [units][npair][2] chunks finished / partials written (self-resetting)
};

// KV-split plan of one call (sab_ws_layout::kv_chunk / kv_nchunk): 0 / 1 when the
// (unit, pair) items already spread evenly over the SMs.
void kv_split_plan(int64_t units, int n, int causal, int* kv_chunk, int* nchunk);

cudaError_t launch_attention(const AttnParams& p, cudaStream_t s);
cudaError_t launch_qk_dump(const AttnParams& p, cudaStream_t s);

// PDL between K1a -> K1b -> K2 on the fast path (SAB_PDL=0 turns it off).
inline bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("SAB_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

// Launches `kern` on `s`, with the programmatic-stream-serialization attribute when
// PDL is enabled (the kernel must call griddep_wait before reading its producer's output).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace sab
