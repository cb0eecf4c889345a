"""Accuracy metrics and adaptive per-layer kernel selection.

The reference specifies this module ("metrics-adaptive"; PAPER
section 4.3 metrics, section 4.5 adaptive quantization) but ships no code for it.
The policy: run each layer's calibration batches through the candidate kernel
(SAGEAttn-vB), compare with full-precision attention, and assign the candidate
iff the aggregated cosine similarity exceeds the threshold (0.998), else the
fallback (SAGEAttn-B).

The candidate and fallback run on the B200 kernels through ``sage_attention_cuda``.
The full-precision comparison is exact attention in binary64, evaluated on the
device with torch matmuls in row chunks.  It is the calibration yardstick, not a
product path.  The metrics are binary64 over binary32 outputs
("Metrics computed in binary64").
"""
from __future__ import annotations

import warnings
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from .sageattn import KernelConfig, PvPath, QkGranularity, SageVariant, kernel_config_for

DEFAULT_THRESHOLD = 0.998  # PAPER 4.5, "bigger than 99.8%"


# ---------------------------------------------------------------------------- metrics

def _f64(a) -> np.ndarray:
    if hasattr(a, "detach"):
        a = a.detach().cpu().numpy()
    return np.asarray(a, np.float64).ravel()


def cosine_sim(o, o_ref) -> float:
    """sum(O O') / (sqrt(sum O^2) sqrt(sum O'^2)); 0 with a warning when a norm is 0."""
    a, b = _f64(o), _f64(o_ref)
    if a.shape != b.shape:
        raise ValueError("cosine_sim: shape mismatch")
    den = np.sqrt((a * a).sum()) * np.sqrt((b * b).sum())
    if den == 0.0:
        warnings.warn("cosine_sim: degenerate (all-zero) input")
        return 0.0
    return float((a * b).sum() / den)


def relative_l1(o, o_ref) -> float:
    """sum|O - O'| / sum|O| with O the reference (second argument)."""
    a, b = _f64(o), _f64(o_ref)
    if a.shape != b.shape:
        raise ValueError("relative_l1: shape mismatch")
    den = np.abs(b).sum()
    if den == 0.0:
        raise ValueError("relative_l1: all-zero reference")
    return float(np.abs(a - b).sum() / den)


def rmse(o, o_ref) -> float:
    a, b = _f64(o), _f64(o_ref)
    if a.shape != b.shape:
        raise ValueError("rmse: shape mismatch")
    return float(np.sqrt(np.mean((a - b) ** 2)))


@dataclass
class AccuracyReport:
    cos_sim: float
    relative_l1: float
    rmse: float


def accuracy(o, o_ref) -> AccuracyReport:
    return AccuracyReport(cosine_sim(o, o_ref), relative_l1(o, o_ref), rmse(o, o_ref))


# ---------------------------------------------------------------------------- plan

def _name(cfg: KernelConfig) -> str:
    for v in SageVariant:
        if kernel_config_for(v) == cfg:
            return {"T": "SAGEAttn-T", "B": "SAGEAttn-B", "VT": "SAGEAttn-vT", "VB": "SAGEAttn-vB"}[v.name]
    return repr(cfg)


@dataclass
class LayerPlan:
    """Per-layer kernel assignment."""
    assignments: List[KernelConfig]
    cos_sim: List[float]
    threshold: float = DEFAULT_THRESHOLD
    candidate: KernelConfig = field(default_factory=lambda: kernel_config_for(SageVariant.VB))
    fallback: KernelConfig = field(default_factory=lambda: kernel_config_for(SageVariant.B))

    def to_text(self) -> str:
        """Human-readable serialisation."""
        lines = [f"threshold {self.threshold!r}", f"candidate {_name(self.candidate)}",
                 f"fallback {_name(self.fallback)}"]
        for i, (cfg, c) in enumerate(zip(self.assignments, self.cos_sim)):
            lines.append(f"layer {i} {_name(cfg)} cos_sim {c:.9f}")
        return "\n".join(lines) + "\n"


def assign(cos_per_layer: Sequence[float], threshold: float = DEFAULT_THRESHOLD,
           candidate: Optional[KernelConfig] = None, fallback: Optional[KernelConfig] = None) -> LayerPlan:
    """The selection rule alone: candidate iff cos_sim > threshold."""
    if not 0.0 <= threshold <= 1.0:
        raise ValueError("calibrate: threshold must lie in [0, 1]")
    candidate = candidate or kernel_config_for(SageVariant.VB)
    fallback = fallback or kernel_config_for(SageVariant.B)
    cos = [float(c) for c in cos_per_layer]
    return LayerPlan([candidate if c > threshold else fallback for c in cos], cos, threshold, candidate, fallback)


# ---------------------------------------------------------------------------- calibration on the device

def exact_attention(q, k, v, causal: bool, rows_per_chunk: int = 1024):
    """Full-precision attention in binary64 on q's device: (B,H,N,d) -> float64 (B,H,N,d)."""
    import torch

    q64, k64, v64 = (t.to(torch.float64) for t in (q, k, v))
    n, d = q.shape[2], q.shape[3]
    out = torch.empty(q.shape, dtype=torch.float64, device=q.device)
    scale = 1.0 / np.sqrt(d)
    for r0 in range(0, n, rows_per_chunk):
        r1 = min(n, r0 + rows_per_chunk)
        s = torch.matmul(q64[:, :, r0:r1], k64.transpose(-1, -2)) * scale
        if causal:
            rows = torch.arange(r0, r1, device=q.device)[:, None]
            cols = torch.arange(n, device=q.device)[None, :]
            s = s.masked_fill(cols > rows, float("-inf"))
        out[:, :, r0:r1] = torch.matmul(torch.softmax(s, dim=-1), v64)
    return out


def _run(cfg: KernelConfig, q, k, v, causal: bool):
    import torch

    from .sageattn import sage_attention_cuda

    if cfg.block_q != 128 or cfg.block_kv != 64:
        raise ValueError("calibrate: only block_q=128, block_kv=64 kernels run on the B200 path")
    return sage_attention_cuda(q, k, v, causal=causal, out_dtype=torch.float32,
                               per_token=cfg.qk_granularity == QkGranularity.PerToken,
                               pv_int8=cfg.pv_path == PvPath.Int8)


def calibrate(layers: Sequence[Sequence[Tuple[object, object, object, bool]]],
              candidate: Optional[KernelConfig] = None, fallback: Optional[KernelConfig] = None,
              threshold: float = DEFAULT_THRESHOLD, aggregate: str = "mean") -> LayerPlan:
    """calibrate(layers, candidate, fallback, threshold) -> LayerPlan.

    ``layers[i]`` is layer i's calibration batches, each (q, k, v, causal) with q/k/v CUDA
    tensors (B,H,N,d) fp16/fp32.  Per layer, the candidate's cosine similarity to exact
    attention is aggregated over the batches ("mean", the SPEC default, or "min", the
    worst case); the layer gets the candidate iff the aggregate exceeds the threshold."""
    if not layers or any(len(b) == 0 for b in layers):
        raise ValueError("calibrate: empty calibration set")
    if aggregate not in ("mean", "min"):
        raise ValueError("calibrate: aggregate must be 'mean' or 'min'")
    candidate = candidate or kernel_config_for(SageVariant.VB)
    fallback = fallback or kernel_config_for(SageVariant.B)
    per_layer = []
    for batches in layers:
        cs = [cosine_sim(_run(candidate, q, k, v, causal), exact_attention(q, k, v, causal))
              for q, k, v, causal in batches]
        per_layer.append(float(np.mean(cs)) if aggregate == "mean" else float(np.min(cs)))
    return assign(per_layer, threshold, candidate, fallback)
