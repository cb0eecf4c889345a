"""Python mirror of the reference's SageAttn-B entry point, over the C ABI.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/sageattn/attention.hpp:

* ``AttentionInput`` (27-32), ``QkGranularity``/``PvPath``/``SageVariant``
  (34-36), ``KernelConfig`` (41-46), ``kernel_config_for`` (48-56),
  ``SageDiagnostics`` (58-69), ``SageOptions`` (71-77), ``QuantDtype``
  (quant.hpp:22), ``apply_causal_tiling`` (83-94).
* ``sage_attention(inp, config_or_variant, options)`` (318-319, 547-550)
  runs on B200 through ``sab_attention_fwd_host``: ValueError stands for
  std::invalid_argument and OverflowError for std::overflow_error, with the
  reference's messages.  All four variants (B, T, vB, vT) run; options outside
  them (FP8 dtypes, PerTensor scales, other block sizes, head_dim not 64/128)
  raise ValueError -- there is no CPU fallback.

``sage_attention_cuda`` is the device-resident path for torch CUDA tensors
(fp16 in, fp16/fp32 out) used by bench.py; ``prepass_cuda`` and
``qk_int32_tiles_cuda`` expose K1 outputs and K2's INT32 S tiles for the
bit-exact parity tests.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Optional, Sequence, Union

import numpy as np

from . import _lib


class QkGranularity(IntEnum):
    PerToken = 0
    PerBlock = 1
    PerTensor = 2


class PvPath(IntEnum):
    Int8 = 0
    Fp16Acc = 1


class SageVariant(IntEnum):
    T = 0
    B = 1
    VT = 2
    VB = 3


class QuantDtype(IntEnum):
    Int8 = 0
    FpE4M3 = 1
    FpE5M2 = 2


class TileKind(IntEnum):
    Full = 0
    Diagonal = 1
    Skip = 2


@dataclass
class KernelConfig:
    qk_granularity: QkGranularity = QkGranularity.PerBlock
    pv_path: PvPath = PvPath.Fp16Acc
    block_q: int = 128
    block_kv: int = 64


def kernel_config_for(v: SageVariant) -> KernelConfig:
    g = QkGranularity.PerToken if v in (SageVariant.T, SageVariant.VT) else QkGranularity.PerBlock
    p = PvPath.Fp16Acc if v in (SageVariant.T, SageVariant.B) else PvPath.Int8
    return KernelConfig(g, p, 128, 64)


@dataclass
class SageDiagnostics:
    s_stage_macs: int = 0
    pv_stage_macs: int = 0
    measure_static_scale: bool = False
    static_scale_elements: int = 0
    static_scale_first_block_mismatches: int = 0
    static_scale_later_block_mismatches: int = 0


@dataclass
class SageOptions:
    smooth_k: bool = True
    qk_dtype: QuantDtype = QuantDtype.Int8
    pv_dtype: QuantDtype = QuantDtype.Int8
    pv_fp32_accumulator: bool = False
    diagnostics: Optional[SageDiagnostics] = None


@dataclass
class AttentionInput:
    q: np.ndarray
    k: np.ndarray
    v: np.ndarray
    causal: bool = False


def apply_causal_tiling(i: int, j: int, block_q: int, block_kv: int, n_tokens: int) -> TileKind:
    if block_q < 1 or block_kv < 1:
        raise ValueError("block sizes must be >= 1")
    r0 = i * block_q
    r1 = min(r0 + block_q, n_tokens) - 1
    c0 = j * block_kv
    c1 = min(c0 + block_kv, n_tokens) - 1
    if r0 < 0 or r0 > r1 or c0 < 0 or c0 > c1 or r1 >= n_tokens or c1 >= n_tokens:
        raise ValueError("tile indices out of range")
    if c0 > r1:
        return TileKind.Skip
    if c1 <= r0:
        return TileKind.Full
    return TileKind.Diagonal


def _raise_for(err: _lib.SabError):
    if err.status in (_lib.SAB_ERR_SHAPE, _lib.SAB_ERR_NONFINITE, _lib.SAB_ERR_UNSUPPORTED, _lib.SAB_ERR_ARGUMENT):
        raise ValueError(str(err)) from None
    if err.status == _lib.SAB_ERR_OVERFLOW:
        raise OverflowError(str(err)) from None
    raise err


def _check_b_path(config: KernelConfig, options: SageOptions):
    if config.block_q < 1 or config.block_kv < 1:
        raise ValueError("sage_attention: block sizes must be >= 1")
    if config.qk_granularity not in (QkGranularity.PerBlock, QkGranularity.PerToken):
        raise ValueError("sage_attention: only PerBlock (B, vB) or PerToken (T, vT) Q/K granularity runs on the "
                         "B200 path")
    if options.qk_dtype != QuantDtype.Int8:
        raise ValueError("sage_attention: only INT8 Q/K quantization runs on the B200 path")
    if config.pv_path == PvPath.Int8 and options.pv_dtype != QuantDtype.Int8:
        raise ValueError("sage_attention: only INT8 P~V quantization runs on the B200 path")


PV_ACCUM = {"fp32": _lib.SAB_PV_FP32, "fp16": _lib.SAB_PV_FP16}


def _pv_accum(pv_accum: str) -> int:
    if pv_accum not in PV_ACCUM:
        raise ValueError("pv_accum must be 'fp32' or 'fp16'")
    return PV_ACCUM[pv_accum]


def sage_attention(inp: AttentionInput, config: Union[KernelConfig, SageVariant],
                   options: Optional[SageOptions] = None, devices: Optional[Sequence[int]] = None,
                   pv_accum: str = "fp32") -> np.ndarray:
    """SAGEAttn-B / -T / -vB / -vT forward on host arrays (B, H, N, d); returns float32 (B, H, N, d).

    Q/K/V may be float32 (bit-exact prepass for any finite float32 input) or
    float16.  pv_accum (B/T): "fp32" -- P~V accumulates in FP32 on B200 whatever
    ``options.pv_fp32_accumulator`` says (the reference's FP32 arm,
    attention.hpp:454-471; the parity gate); "fp16" -- a persistent binary16 TMEM
    accumulator (the reference's default arm's semantics, attention.hpp:447-475);
    "options" -- follow ``options.pv_fp32_accumulator`` as the reference does."""
    options = options or SageOptions()
    if pv_accum == "options":
        pv_accum = "fp32" if options.pv_fp32_accumulator else "fp16"
    acc = _pv_accum(pv_accum)
    if isinstance(config, SageVariant):
        config = kernel_config_for(config)
    _check_b_path(config, options)
    q, k, v = (np.asarray(t) for t in (inp.q, inp.k, inp.v))
    if q.shape != k.shape or q.shape != v.shape:
        raise ValueError("sage_attention: Q, K, V shapes differ")
    if q.ndim != 4:
        raise ValueError("tensor dimensions must be positive")
    b, h, n, d = q.shape
    f16 = q.dtype == np.float16 and k.dtype == np.float16 and v.dtype == np.float16
    dt = np.float16 if f16 else np.float32
    q, k, v = (np.ascontiguousarray(t, dtype=dt) for t in (q, k, v))
    out = np.empty((b, h, n, d), np.float32)
    try:
        desc = _lib.desc(b, h, n, d, inp.causal, in_dtype=_lib.SAB_F16 if f16 else _lib.SAB_F32,
                         out_dtype=_lib.SAB_F32, block_q=config.block_q, block_kv=config.block_kv,
                         smooth_k=options.smooth_k, check_v=True,
                         per_token=config.qk_granularity == QkGranularity.PerToken,
                         pv_int8=config.pv_path == PvPath.Int8,
                         pv_accum=acc if config.pv_path == PvPath.Fp16Acc else _lib.SAB_PV_FP32)
        diag = options.diagnostics
        desc.measure_static_scale = int(diag is not None and diag.measure_static_scale
                                        and config.pv_path == PvPath.Int8)
        devs = list(devices) if devices else [0]
        arr = (C.c_int * len(devs))(*devs)
        counts = (C.c_uint64 * 3)()
        _lib.check(_lib.load().sab_attention_fwd_host_diag(C.byref(desc), q.ctypes.data, k.ctypes.data,
                                                           v.ctypes.data, out.ctypes.data, arr, len(devs), counts))
        if diag is not None:
            s, p = _lib.diagnostics(desc)
            diag.s_stage_macs += s
            diag.pv_stage_macs += p
            if desc.measure_static_scale:  # attention.hpp:479-488, counted by K2 on the GPU
                diag.static_scale_elements += counts[0]
                diag.static_scale_first_block_mismatches += counts[1]
                diag.static_scale_later_block_mismatches += counts[2]
    except _lib.SabError as e:
        _raise_for(e)
    return out


# ---------------------------------------------------------------------------- device path (torch)

def _torch():
    import torch

    return torch


class Workspace:
    """Device workspace for one shape (K1 outputs + status word), torch-allocated."""

    def __init__(self, desc: _lib.SabDesc, device):
        torch = _torch()
        self.desc = desc
        self.layout = _lib.workspace_layout(desc)
        self.buf = torch.empty(int(self.layout.total), dtype=torch.uint8, device=device)

    @property
    def ptr(self) -> int:
        return self.buf.data_ptr()

    @property
    def nbytes(self) -> int:
        return int(self.layout.total)

    def view(self, name: str, dtype, shape):
        torch = _torch()
        off = int(getattr(self.layout, name))
        nbytes = int(np.prod(shape)) * torch.tensor([], dtype=dtype).element_size()
        return self.buf[off:off + nbytes].view(dtype).view(*shape)


def _stream_ptr(stream) -> int:
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def make_desc(q, causal: bool, out_dtype=None, smooth_k: bool = True, check_v: bool = False,
              per_token: bool = False, pv_int8: bool = False, pv_accum: str = "fp32") -> _lib.SabDesc:
    torch = _torch()
    b, h, n, d = q.shape
    in_dt = _lib.SAB_F16 if q.dtype == torch.float16 else _lib.SAB_F32
    out_dt = _lib.SAB_F32 if out_dtype == torch.float32 else _lib.SAB_F16
    return _lib.desc(b, h, n, d, causal, in_dtype=in_dt, out_dtype=out_dt, smooth_k=smooth_k, check_v=check_v,
                     per_token=per_token, pv_int8=pv_int8, pv_accum=_pv_accum(pv_accum))


ROPE_LAYOUTS = {"interleaved": _lib.SAB_ROPE_INTERLEAVED, "half": _lib.SAB_ROPE_HALF}


def _enqueue_prepass(desc, q, k, v, ws, stream, rope):
    """sab_prepass, or sab_prepass_rope when rope = (cos, sin, layout) is given: cos / sin float32
    CUDA tensors (N, d/2) and layout "interleaved" (pairs 2i, 2i+1) or "half" (pairs i, i+d/2)."""
    vptr = v.data_ptr() if v is not None else None
    lib = _lib.load()
    if rope is None:
        return lib.sab_prepass(C.byref(desc), q.data_ptr(), k.data_ptr(), vptr, ws.ptr, ws.nbytes, _stream_ptr(stream))
    cos, sin, layout = rope
    torch = _torch()
    n, d = q.shape[2], q.shape[3]
    for t in (cos, sin):
        if t.dtype != torch.float32 or tuple(t.shape) != (n, d // 2) or not t.is_contiguous() or t.device != q.device:
            raise ValueError("rope tables must be contiguous float32 (tokens, head_dim/2) on the inputs' device")
    if layout not in ROPE_LAYOUTS:
        raise ValueError(f"rope layout must be one of {sorted(ROPE_LAYOUTS)}")
    return lib.sab_prepass_rope(C.byref(desc), q.data_ptr(), k.data_ptr(), vptr, cos.data_ptr(), sin.data_ptr(),
                                ROPE_LAYOUTS[layout], ws.ptr, ws.nbytes, _stream_ptr(stream))


def prepass_cuda(q, k, v=None, smooth_k: bool = True, ws: Optional[Workspace] = None, stream=None,
                 per_token: bool = False, pv_int8: bool = False, rope=None) -> Workspace:
    """K1 on CUDA tensors (B,H,N,d) fp16/fp32; returns the workspace holding codes/scales/mean
    (and, with pv_int8, the per-channel V^ of SAGEAttn-vB).  rope = (cos, sin, layout) rotates
    Q and K inside K1 first (sab_prepass_rope)."""
    desc = make_desc(q, False, smooth_k=smooth_k, per_token=per_token, pv_int8=pv_int8)
    ws = ws or Workspace(desc, q.device)
    try:
        _lib.check(_enqueue_prepass(desc, q, k, v, ws, stream, rope))
    except _lib.SabError as e:
        _raise_for(e)
    return ws


def prepass_outputs(ws: Workspace):
    """Views of K1's outputs: dict(qcodes, kcodes (units,N,d) int8, qscales, kscales, mean)."""
    torch = _torch()
    dsc = ws.desc
    units, n, d = dsc.batch * dsc.heads, dsc.tokens, dsc.head_dim
    pt = dsc.qk_granularity == _lib.SAB_QK_PER_TOKEN
    npad = -(-n // 64) * 64  # per-token scale rows are padded to 64 tokens
    return dict(qcodes=ws.view("qcodes", torch.int8, (units, n, d)),
                kcodes=ws.view("kcodes", torch.int8, (units, n, d)),
                qscales=ws.view("qscales", torch.float32, (units, npad))[:, :n] if pt else
                ws.view("qscales", torch.float32, (units, -(-n // 128))),
                kscales=ws.view("kscales", torch.float32, (units, npad))[:, :n] if pt else
                ws.view("kscales", torch.float32, (units, -(-n // 64))),
                mean=ws.view("mean_k", torch.float32, (units, d)),
                **(dict(vcodes=ws.view("vcodes", torch.int8, (units, d, npad))[:, :, :n].transpose(1, 2),
                        vscales=ws.view("vscales", torch.float32, (units, d)))
                   if dsc.pv_path == _lib.SAB_PV_PATH_INT8 else {}))


def read_status(ws: Workspace, stream=None) -> int:
    st = C.c_int()
    _lib.check(_lib.load().sab_read_status(C.byref(ws.desc), ws.ptr, _stream_ptr(stream), C.byref(st)))
    return st.value


def sage_attention_cuda(q, k, v, causal: bool = False, out=None, out_dtype=None, smooth_k: bool = True,
                        ws: Optional[Workspace] = None, stream=None, check: bool = True, per_token: bool = False,
                        pv_int8: bool = False, rope=None, pv_accum: str = "fp32"):
    """K1 + K2 on device-resident CUDA tensors (B,H,N,d); returns O (fp16 by default).

    With check=True the stream is synchronised and data-dependent errors raise
    like the reference; with check=False the call stays fully asynchronous.
    rope = (cos, sin, layout): Q and K are the pre-rotation tensors, rotated inside K1."""
    torch = _torch()
    out_dtype = out_dtype or (out.dtype if out is not None else torch.float16)
    desc = make_desc(q, causal, out_dtype=out_dtype, smooth_k=smooth_k, per_token=per_token, pv_int8=pv_int8,
                     pv_accum=pv_accum)
    if ws is None or ws.nbytes < int(_lib.workspace_layout(desc).total):
        ws = Workspace(desc, q.device)
    ws.desc = desc
    if out is None:
        out = torch.empty(q.shape, dtype=out_dtype, device=q.device)
    try:
        if rope is None:
            _lib.check(_lib.load().sab_attention_fwd(C.byref(desc), q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                                     out.data_ptr(), ws.ptr, ws.nbytes, _stream_ptr(stream)))
        else:
            _lib.check(_enqueue_prepass(desc, q, k, v, ws, stream, rope))
            _lib.check(_lib.load().sab_attention(C.byref(desc), ws.ptr, ws.nbytes, v.data_ptr(), out.data_ptr(),
                                                 _stream_ptr(stream)))
        if check:
            _lib.check(read_status(ws, stream))
    except _lib.SabError as e:
        _raise_for(e)
    return out


def attention_only_cuda(ws: Workspace, v, out, stream=None):
    """K2 alone, from a workspace already filled by K1 (bench timing of the dominant kernel)."""
    _lib.check(_lib.load().sab_attention(C.byref(ws.desc), ws.ptr, ws.nbytes, v.data_ptr(), out.data_ptr(),
                                         _stream_ptr(stream)))


def qk_int32_tiles_cuda(ws: Workspace, unit: int, q_tile: int, stream=None):
    """INT32 S tiles K2 computes with tcgen05 kind::i8 for (unit, q_tile): int32 (n_kv_tiles, 128, 64)."""
    torch = _torch()
    dsc = ws.desc
    ntk = -(-dsc.tokens // 64)
    nkv = min(2 * q_tile + 2, ntk) if dsc.causal else ntk
    out = torch.zeros((nkv, 128, 64), dtype=torch.int32, device=ws.buf.device)
    _lib.check(_lib.load().sab_qk_int32_tiles(C.byref(dsc), ws.ptr, unit, q_tile, out.data_ptr(),
                                              _stream_ptr(stream)))
    return out


def attention_fwd_host(q: np.ndarray, k: np.ndarray, v: np.ndarray, causal: bool, out: np.ndarray,
                       devices: Sequence[int] = (0,), per_token: bool = False, pv_int8: bool = False,
                       pv_accum: str = "fp32"):
    """The C-ABI host-buffer call (sab_attention_fwd_host) on raw fp16/fp32 arrays; `out` receives O."""
    b, h, n, d = q.shape
    in_dt = _lib.SAB_F16 if q.dtype == np.float16 else _lib.SAB_F32
    out_dt = _lib.SAB_F16 if out.dtype == np.float16 else _lib.SAB_F32
    desc = _lib.desc(b, h, n, d, causal, in_dtype=in_dt, out_dtype=out_dt, per_token=per_token, pv_int8=pv_int8,
                     pv_accum=_pv_accum(pv_accum))
    arr = (C.c_int * len(devices))(*devices)
    try:
        _lib.check(_lib.load().sab_attention_fwd_host(C.byref(desc), q.ctypes.data, k.ctypes.data, v.ctypes.data,
                                                      out.ctypes.data, arr, len(devices)))
    except _lib.SabError as e:
        _raise_for(e)
    return out
