"""ctypes binding of libsageattn_b200.so (the C ABI in include/sageattn_b200.h).

The library is the only compute path: there is no CPU or PyTorch fallback.
If it is missing, loading raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsageattn_b200.so")

SAB_OK = 0
SAB_ERR_SHAPE = 1
SAB_ERR_NONFINITE = 2
SAB_ERR_OVERFLOW = 3
SAB_ERR_CUDA = 4
SAB_ERR_UNSUPPORTED = 5
SAB_ERR_WORKSPACE = 6
SAB_ERR_NO_DEVICE = 7
SAB_ERR_ARGUMENT = 8

SAB_F16 = 0
SAB_F32 = 1
SAB_PV_FP32 = 0
SAB_PV_FP16 = 1  # binary16 P~V accumulator (the paper's mma f16.f16.f16)
SAB_QK_PER_BLOCK = 0  # SAGEAttn-B
SAB_QK_PER_TOKEN = 1  # SAGEAttn-T
SAB_PV_PATH_FP16 = 0  # B / T
SAB_PV_PATH_INT8 = 1  # vB
SAB_ROPE_INTERLEAVED = 1  # pairs (2i, 2i+1)
SAB_ROPE_HALF = 2  # pairs (i, i + d/2)

# Every symbol include/sageattn_b200.h declares (checked by tests/test_capi.py).
EXPORTS = (
    "sab_desc_init", "sab_status_string", "sab_last_error", "sab_abi_version", "sab_check_desc",
    "sab_workspace_size", "sab_workspace_layout", "sab_prepass", "sab_attention", "sab_attention_fwd",
    "sab_read_status", "sab_attention_fwd_host", "sab_shard_plan", "sab_qk_int32_tiles", "sab_diagnostics",
    "sab_device_count", "sab_device_ordinals", "sab_attention_fwd_host_diag", "sab_read_static_scale_counts",
    "sab_prepass_rope",
)


class SabDesc(C.Structure):
    _fields_ = [(name, C.c_int32) for name in (
        "batch", "heads", "tokens", "head_dim", "causal", "in_dtype", "out_dtype", "block_q", "block_kv",
        "smooth_k", "pv_accum", "check_v", "qk_granularity", "pv_path", "measure_static_scale")]


class SabWsLayout(C.Structure):
    _fields_ = [(name, C.c_uint64) for name in (
        "qcodes", "kcodes", "qscales", "kscales", "mean_k", "partials", "v16", "status", "total")] + [
        ("n_partials", C.c_int32), ("tree_depth", C.c_int32), ("vcodes", C.c_uint64), ("vscales", C.c_uint64),
        ("diag", C.c_uint64), ("split_o", C.c_uint64), ("split_ml", C.c_uint64), ("split_cnt", C.c_uint64),
        ("kv_chunk", C.c_int32), ("kv_nchunk", C.c_int32)]


class SabError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status


_lib = None


def load():
    """Loads the CUDA library (cached); raises if it was never built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_2410_02367_b200.build` "
                           "(there is no CPU fallback for the SageAttn-B path)")
    lib = C.CDLL(LIB_PATH)
    P = C.POINTER
    vp, sz = C.c_void_p, C.c_size_t
    lib.sab_desc_init.restype = None
    lib.sab_desc_init.argtypes = [P(SabDesc)] + [C.c_int32] * 5
    lib.sab_status_string.restype = C.c_char_p
    lib.sab_status_string.argtypes = [C.c_int]
    lib.sab_last_error.restype = C.c_char_p
    lib.sab_last_error.argtypes = []
    lib.sab_abi_version.restype = C.c_int
    lib.sab_check_desc.argtypes = [P(SabDesc)]
    lib.sab_workspace_size.argtypes = [P(SabDesc), P(sz)]
    lib.sab_workspace_layout.argtypes = [P(SabDesc), P(SabWsLayout)]
    lib.sab_prepass.argtypes = [P(SabDesc), vp, vp, vp, vp, sz, vp]
    lib.sab_attention.argtypes = [P(SabDesc), vp, sz, vp, vp, vp]
    lib.sab_attention_fwd.argtypes = [P(SabDesc), vp, vp, vp, vp, vp, sz, vp]
    lib.sab_read_status.argtypes = [P(SabDesc), vp, vp, P(C.c_int)]
    lib.sab_attention_fwd_host.argtypes = [P(SabDesc), vp, vp, vp, vp, P(C.c_int), C.c_int]
    lib.sab_shard_plan.argtypes = [C.c_int, C.c_int, C.c_int, P(C.c_int), P(C.c_int)]
    lib.sab_qk_int32_tiles.argtypes = [P(SabDesc), vp, C.c_int, C.c_int, vp, vp]
    lib.sab_diagnostics.argtypes = [P(SabDesc), P(C.c_uint64), P(C.c_uint64)]
    lib.sab_device_count.argtypes = [P(C.c_int)]
    lib.sab_device_ordinals.argtypes = [P(C.c_int), C.c_int, P(C.c_int)]
    lib.sab_attention_fwd_host_diag.argtypes = [P(SabDesc), vp, vp, vp, vp, P(C.c_int), C.c_int, P(C.c_uint64)]
    lib.sab_read_static_scale_counts.argtypes = [P(SabDesc), vp, vp, P(C.c_uint64)]
    lib.sab_prepass_rope.argtypes = [P(SabDesc), vp, vp, vp, vp, vp, C.c_int, vp, sz, vp]
    for name in EXPORTS:
        if name not in ("sab_desc_init", "sab_status_string", "sab_last_error"):
            getattr(lib, name).restype = C.c_int
    _lib = lib
    return lib


def check(status: int):
    """Raises SabError carrying the library's last message on a non-zero status."""
    if status != SAB_OK:
        lib = load()
        msg = lib.sab_last_error().decode() or lib.sab_status_string(status).decode()
        raise SabError(status, msg)


def desc(batch, heads, tokens, head_dim, causal=False, in_dtype=SAB_F16, out_dtype=SAB_F32, block_q=128,
         block_kv=64, smooth_k=True, pv_accum=SAB_PV_FP32, check_v=False, per_token=False,
         pv_int8=False) -> SabDesc:
    d = SabDesc()
    load().sab_desc_init(C.byref(d), batch, heads, tokens, head_dim, int(causal))
    d.in_dtype, d.out_dtype = in_dtype, out_dtype
    d.block_q, d.block_kv = block_q, block_kv
    d.smooth_k, d.pv_accum, d.check_v = int(smooth_k), pv_accum, int(check_v)
    d.qk_granularity = SAB_QK_PER_TOKEN if per_token else SAB_QK_PER_BLOCK
    d.pv_path = SAB_PV_PATH_INT8 if pv_int8 else SAB_PV_PATH_FP16
    return d


def workspace_layout(d: SabDesc) -> SabWsLayout:
    L = SabWsLayout()
    check(load().sab_workspace_layout(C.byref(d), C.byref(L)))
    return L


def shard_plan(units: int, n_shards: int, s: int):
    first, count = C.c_int(), C.c_int()
    check(load().sab_shard_plan(units, n_shards, s, C.byref(first), C.byref(count)))
    return first.value, count.value


def device_ordinals():
    """Ordinals of the visible sm_100 devices (sab_device_ordinals)."""
    n = C.c_int()
    check(load().sab_device_ordinals(None, 0, C.byref(n)))
    arr = (C.c_int * max(1, n.value))()
    check(load().sab_device_ordinals(arr, n.value, C.byref(n)))
    return list(arr[:n.value])


def diagnostics(d: SabDesc):
    a, b = C.c_uint64(), C.c_uint64()
    check(load().sab_diagnostics(C.byref(d), C.byref(a), C.byref(b)))
    return a.value, b.value
