"""B200-native (sm_100a) SageAttn-B forward: K1 prepass + K2 tcgen05 attention + K3 head x batch sharding.

The compute path is libsageattn_b200.so behind the C ABI in
include/sageattn_b200.h; this package only mirrors the reference interface
(sageattn.py), binds the library (_lib.py) and adds the host-side adaptive
kernel selection of SPEC.md's metrics-adaptive module (calibrate.py).
"""
from .sageattn import (  # noqa: F401
    AttentionInput, KernelConfig, PvPath, QkGranularity, QuantDtype, SageDiagnostics, SageOptions, SageVariant,
    TileKind, apply_causal_tiling, kernel_config_for, sage_attention, sage_attention_cuda, prepass_cuda,
    prepass_outputs, qk_int32_tiles_cuda, attention_fwd_host, read_status, Workspace,
)

__all__ = [
    "AttentionInput", "KernelConfig", "PvPath", "QkGranularity", "QuantDtype", "SageDiagnostics", "SageOptions",
    "SageVariant", "TileKind", "apply_causal_tiling", "kernel_config_for", "sage_attention", "sage_attention_cuda",
    "prepass_cuda", "prepass_outputs", "qk_int32_tiles_cuda", "attention_fwd_host", "read_status", "Workspace",
]
