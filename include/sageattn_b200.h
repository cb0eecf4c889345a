/*
 * sageattn_b200.h -- C ABI of the B200-native SageAttn-B forward path.
 *
 * This is the drop-in boundary: plain C, plain pointers and sizes, no torch
 * or C++ types.  The C++ entry point of the reference,
 *     sageattn::sage_attention(const AttentionInput&, const KernelConfig&,
 *                              const SageOptions&)      (attention.hpp:318-319)
 *     sageattn::sage_attention(const AttentionInput&, SageVariant,
 *                              const SageOptions&)      (attention.hpp:547-550)
 * is re-provided source-compatibly by include/sageattn/attention.hpp, which
 * is a thin header over the functions below.  Each function names the
 * reference interface it replaces.
 *
 * SAGEAttn-vB (INT8 P~V) shares K1 and K2 through sab_desc.pv_path.
 *
 * Tensor layout everywhere: contiguous (batch, heads, tokens, head_dim),
 * i.e. units = batch*heads independent (tokens x head_dim) slices, the
 * layout of Tensor4::at (tensor.hpp:76-81).
 *
 * Library: paper_2410_02367_b200/libsageattn_b200.so (sm_100a only).
 */
#ifndef SAGEATTN_B200_H
#define SAGEATTN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SAB_ABI_VERSION 7

/* Status codes.  The C++ shim maps them back to the reference's exceptions:
 * SAB_ERR_SHAPE / SAB_ERR_NONFINITE / SAB_ERR_UNSUPPORTED -> std::invalid_argument,
 * SAB_ERR_OVERFLOW -> std::overflow_error (attention.hpp:100-102, 321, 531-533). */
enum sab_status {
    SAB_OK = 0,
    SAB_ERR_SHAPE = 1,        /* bad shape or block sizes                        */
    SAB_ERR_NONFINITE = 2,    /* non-finite Q, K or V element                    */
    SAB_ERR_OVERFLOW = 3,     /* non-finite P~V accumulator at finalize          */
    SAB_ERR_CUDA = 4,         /* CUDA runtime / driver failure                   */
    SAB_ERR_UNSUPPORTED = 5,  /* option outside the SAGEAttn-B hot path          */
    SAB_ERR_WORKSPACE = 6,    /* workspace missing or too small                  */
    SAB_ERR_NO_DEVICE = 7,    /* no sm_100 device visible                        */
    SAB_ERR_ARGUMENT = 8      /* NULL pointer or bad scalar argument             */
};

enum sab_dtype { SAB_F16 = 0, SAB_F32 = 1 };

/* P~V accumulation (FP16 P~V path, variants B/T):
 *   SAB_PV_FP32 -- FP32 accumulator in TMEM: the arm of SageOptions::pv_fp32_accumulator
 *                  (attention.hpp:75, 454-471).  The default; the parity gate.
 *   SAB_PV_FP16 -- one persistent binary16 accumulator per row in TMEM (tcgen05.mma
 *                  kind::f16 with an F16 D, the paper's mma f16.f16.f16), rescaled with a
 *                  binary16 rounding: the semantics of the reference's default arm
 *                  (attention.hpp:447-475, matmul.hpp:63-73).  The tensor core rounds once
 *                  per 16 products instead of after every addition, so it lands as far from
 *                  that arm as the arm is from its own FP32 arm (4e-3..1.6e-2 rel-L1, SURVEY
 *                  F3) and about 4x closer to the FP32 arm; a non-finite accumulator raises
 *                  SAB_ERR_OVERFLOW as in the reference.  Never KV-split.  ABI 7. */
enum sab_pv_accum { SAB_PV_FP32 = 0, SAB_PV_FP16 = 1 };

/* Q/K scale granularity: KernelConfig::qk_granularity (attention.hpp:34, 41-46).
 * PER_BLOCK = SAGEAttn-B (128-token Q groups, 64-token K groups); PER_TOKEN =
 * SAGEAttn-T (one scale per token; kernel_config_for(T), attention.hpp:50). */
enum sab_qk_granularity { SAB_QK_PER_BLOCK = 0, SAB_QK_PER_TOKEN = 1 };

/* P~V path: KernelConfig::pv_path (attention.hpp:35, 41-46).  FP16 = SAGEAttn-B/T
 * (binary16 P~ and V); INT8 = SAGEAttn-vB (static-scale INT8 P~, per-channel INT8 V,
 * INT32 products; kernel_config_for(VB), attention.hpp:53, 476-505).  ABI 3. */
enum sab_pv_path { SAB_PV_PATH_FP16 = 0, SAB_PV_PATH_INT8 = 1 };

/* Call descriptor: the shape of AttentionInput (attention.hpp:27-32) plus the
 * KernelConfig/SageOptions fields the B/T paths read (attention.hpp:41-46, 71-77). */
typedef struct sab_desc {
    int32_t batch, heads, tokens, head_dim;
    int32_t causal;       /* AttentionInput::causal                                */
    int32_t in_dtype;     /* sab_dtype of Q, K, V                                  */
    int32_t out_dtype;    /* sab_dtype of O                                        */
    int32_t block_q;      /* KernelConfig::block_q  (must be 128 on this path)     */
    int32_t block_kv;     /* KernelConfig::block_kv (must be 64 on this path)      */
    int32_t smooth_k;     /* SageOptions::smooth_k                                 */
    int32_t pv_accum;     /* sab_pv_accum                                          */
    int32_t check_v;      /* 1: scan V for non-finite values (validate_input)      */
    int32_t qk_granularity; /* sab_qk_granularity (ABI 2)                            */
    int32_t pv_path;      /* sab_pv_path (ABI 3)                                   */
    int32_t measure_static_scale; /* SageDiagnostics::measure_static_scale (ABI 4): INT8 P~V
                                     path only; K2 counts static- vs per-token-scale P~ code
                                     mismatches (attention.hpp:479-488) into the workspace */
} sab_desc;

/* Fills *d with the SAGEAttn-B defaults (kernel_config_for(B), attention.hpp:51;
 * SageOptions{} attention.hpp:71-77) for the given shape. */
void sab_desc_init(sab_desc* d, int32_t batch, int32_t heads, int32_t tokens, int32_t head_dim, int32_t causal);

/* Byte offsets of the prepass outputs inside the workspace. */
typedef struct sab_ws_layout {
    uint64_t qcodes;    /* int8  [units][tokens][head_dim]  Q^ (quant.hpp:128-173)   */
    uint64_t kcodes;    /* int8  [units][tokens][head_dim]  K^                        */
    uint64_t qscales;   /* float [units][ceil(tokens/128)]  delta_Q  (per token: [units][npad],    */
    uint64_t kscales;   /* float [units][ceil(tokens/64)]   delta_K   npad = 64*ceil(tokens/64))   */
    uint64_t mean_k;    /* float [units][head_dim]          SmoothState::mean_k        */
    uint64_t partials;  /* float [units][n_partials][head_dim] mean tree partial sums  */
    uint64_t v16;       /* fp16  [units][tokens][head_dim]  V on the fp16 grid (F32 in)*/
    uint64_t status;    /* int32 device status word, two int32 K2 scheduler counters,
                           then three int32 counters per unit (K1's mean tree; the
                           opt-in single-launch K1's mean-ready flags and K-chunk
                           counts) and its ticket counter; all zero between calls     */
    uint64_t total;     /* workspace bytes                                            */
    int32_t n_partials; /* subtree sums per unit of the pairwise mean tree            */
    int32_t tree_depth; /* depth of the 4..9-token leaf level (quant.hpp:203-213)     */
    uint64_t vcodes;    /* int8  [units][head_dim][64*ceil(tokens/64)] V^ transposed (INT8
                           P~V path only; quantize(V, per_channel), quant.hpp:128-173) */
    uint64_t vscales;   /* float [units][head_dim] delta_V, then float [units][head_dim]
                           channel max |v| scratch (INT8 P~V path only)              */
    uint64_t diag;      /* uint64 [2] static-scale mismatches (first KV block, later
                           blocks); zeroed by sab_prepass (ABI 4)                     */
    /* KV-split plan (ABI 5): when the call has too few (unit, query-tile pair) items to
     * fill the 148 SMs evenly (few heads per device under K3 sharding, long causal rows),
     * K2 splits each pair's KV range into chunks of kv_chunk 64-key tiles; each chunk
     * writes an unnormalised partial and the last chunk of a pair to finish merges them
     * (the reference's q-block independence, attention.hpp:383).  kv_chunk == 0: no split
     * and the three regions below are empty. */
    uint64_t split_o;   /* float4 [units][pairs][kv_nchunk][head_dim/4][256] partial O  */
    uint64_t split_ml;  /* float2 [units][pairs][kv_nchunk][256] (row max m, row sum l) */
    uint64_t split_cnt; /* int32 [units][pairs][2] chunks finished / partials written
                           (self-resetting)                                           */
    int32_t kv_chunk;   /* 64-key tiles per chunk, 0 = no split                         */
    int32_t kv_nchunk;  /* chunks of the longest pair (K2's grid.y)                      */
} sab_ws_layout;

const char* sab_status_string(int status);
/* Detailed message of the last failing call on this host thread. */
const char* sab_last_error(void);
int sab_abi_version(void);

/* Validates *d exactly like the reference entry (attention.hpp:320-322,
 * tensor.hpp:70-71) and rejects options outside the B path. */
int sab_check_desc(const sab_desc* d);

/* Workspace size / layout for one call on one device. */
int sab_workspace_size(const sab_desc* d, size_t* bytes);
int sab_workspace_layout(const sab_desc* d, sab_ws_layout* layout);

/* K1 -- replaces smooth_k (quant.hpp:220-242) + fold_scale_into_q (quant.hpp:246-252)
 * + quantize(per_block 128 / 64, Int8) (quant.hpp:128-173) as called at
 * attention.hpp:336-360.  Device pointers; asynchronous on `stream`
 * (a cudaStream_t, NULL = legacy default).  v may be NULL when in_dtype is
 * F16 and check_v is 0.  Resets and then sets the device status word. */
int sab_prepass(const sab_desc* d, const void* q, const void* k, const void* v, void* ws, size_t ws_bytes,
                void* stream);

/* RoPE layouts of sab_prepass_rope: which channels form the rotated pairs. */
enum sab_rope_layout {
    SAB_ROPE_INTERLEAVED = 1, /* pairs (2i, 2i+1): GPT-J / the complex form          */
    SAB_ROPE_HALF = 2         /* pairs (i, i + d/2): GPT-NeoX / rotate_half          */
};

/* K1 with the rotary position embedding fused into the quantizer -- the paper's
 * "quantization fused into the RoPE kernel".  q and k are the
 * PRE-rotation tensors; token t of every unit is rotated by cos/sin[t][i] (float
 * [tokens][head_dim/2], device, 16-byte aligned) in binary32 with every product and
 * sum rounded (no contraction):
 *   x_a' = x_a*c - x_b*s,   x_b' = x_a*s + x_b*c     ((a, b) = the layout's pair i)
 * and the result is exactly what sab_prepass would produce for the rotated tensors
 * given as F32 inputs (mean(K) of the rotated K, fold, per-block / per-token codes).
 * Same workspace and status contract as sab_prepass; K2 (sab_attention) is unchanged.
 * ABI 6. */
int sab_prepass_rope(const sab_desc* d, const void* q, const void* k, const void* v, const float* cos_table,
                     const float* sin_table, int rope_layout, void* ws, size_t ws_bytes, void* stream);

/* K2 -- replaces the q-block/kv-block engine of attention.hpp:383-541
 * (detail::int8_tile_nt, online softmax, P~V, normalize).  Reads Q^/K^/scales
 * from the workspace; v is the fp16 V (ignored when in_dtype is F32: the
 * prepass wrote V on the fp16 grid into the workspace).  Asynchronous. */
int sab_attention(const sab_desc* d, void* ws, size_t ws_bytes, const void* v, void* o, void* stream);

/* K1 + K2 on device pointers, asynchronous.  The data-dependent status
 * (non-finite input, overflow) is left in the workspace status word; read it
 * with sab_read_status after the stream has been synchronised. */
int sab_attention_fwd(const sab_desc* d, const void* q, const void* k, const void* v, void* o, void* ws,
                      size_t ws_bytes, void* stream);

/* Copies the device status word to *status (synchronous on `stream`). */
int sab_read_status(const sab_desc* d, const void* ws, void* stream, int* status);

/* Host-buffer forward, synchronous -- the full replacement of
 * sage_attention(in, SageVariant::B, opts) (attention.hpp:318-319, 547-550).
 * q/k/v/o are HOST pointers in (B,H,N,d) layout of in_dtype/out_dtype.
 * K3: the B*H units are split into contiguous shards over `n_devices`
 * devices (devices==NULL -> ordinals 0..n_devices-1; n_devices<=0 -> 1
 * device), one host thread per device, no collective.  Host buffers that are
 * not page-locked are staged through pinned chunks. */
int sab_attention_fwd_host(const sab_desc* d, const void* q, const void* k, const void* v, void* o,
                           const int* devices, int n_devices);

/* sab_attention_fwd_host plus the static-scale P~ diagnostics of the INT8 P~V path
 * (SageDiagnostics, attention.hpp:58-69, 479-488): when d->measure_static_scale is set,
 * counts[0] = P~ elements quantized (static_scale_elements), counts[1] / counts[2] =
 * static-scale codes that differ from per-token-scale codes in the first / later KV
 * blocks of each query block.  counts may be NULL; it is zeroed otherwise. */
int sab_attention_fwd_host_diag(const sab_desc* d, const void* q, const void* k, const void* v, void* o,
                                const int* devices, int n_devices, uint64_t counts[3]);

/* Device path: reads the static-scale counters of the last K2 call on `ws` into
 * counts[3] (same meaning as above); synchronous on `stream`. */
int sab_read_static_scale_counts(const sab_desc* d, const void* ws, void* stream, uint64_t counts[3]);

/* Contiguous K3 shard of `units` over `n_shards`: first unit and count of shard `s`. */
int sab_shard_plan(int units, int n_shards, int s, int* first, int* count);

/* Debug/parity: runs K2's tcgen05 kind::i8 QK^T for query tile `q_tile` of
 * unit `unit` and writes the exact INT32 S tiles (what detail::int8_tile_nt
 * computes, attention.hpp:265-279) for every 64-key KV tile K2 visits, as
 * int32 [n_kv_tiles][128 rows][64 keys] into device buffer `s_out`
 * (n_kv_tiles = ceil(tokens/64), or min(2*q_tile+2, ceil(tokens/64)) when
 * causal).  Async. */
int sab_qk_int32_tiles(const sab_desc* d, const void* ws, int unit, int q_tile, int32_t* s_out, void* stream);

/* SageDiagnostics MAC counters (attention.hpp:58-69, 404, 445) for the
 * reference's own 128x64 tiling, computed analytically. */
int sab_diagnostics(const sab_desc* d, uint64_t* s_stage_macs, uint64_t* pv_stage_macs);

/* Number of visible sm_100 devices. */
int sab_device_count(int* count);

/* Ordinals of the visible sm_100 devices, ascending: writes min(count, capacity)
 * of them to ordinals[] and the total to *count.  The drop-in passes this list
 * to sab_attention_fwd_host so mixed-GPU hosts never place a shard on another
 * architecture. */
int sab_device_ordinals(int* ordinals, int capacity, int* count);

#ifdef __cplusplus
}
#endif

#endif /* SAGEATTN_B200_H */
