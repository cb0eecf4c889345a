"""Generates tests/golden/*.npz from the REFERENCE itself (oracle/_ref/libsageref.so,
compiled from /root/reference/proj/include by oracle/Makefile).

    python tests/golden/make_golden.py

Each fixture holds the fp16 inputs and the reference's outputs: mean_k,
Q^/K^ codes and per-block scales, O of sage_attention(B) for both P~V arms,
the SageDiagnostics MAC counters and naive_attention's exact O.

The t_*.npz fixtures (SAGEAttn-T) hold the per-token codes and
scales (quantize(..., Granularity::per_token())) and O of
sage_attention(in, SageVariant::T) for both arms:

    python tests/golden/make_golden.py --variant-t
The vb_*.npz fixtures (SAGEAttn-vB) hold the per-channel V^ codes and
scales (quantize(V, Granularity::per_channel())) and O of
sage_attention(in, SageVariant::VB) and of SageVariant::VT (o_vt):
    python tests/golden/make_golden.py --variant-vb
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Reference  # noqa: E402
from paper_2410_02367_b200 import synth  # noqa: E402

CASES = [
    ("c1_small", 1, 2, 300, 64, False, "normal"),
    ("causal_outlier_d128", 1, 1, 257, 128, True, "outlier"),
    ("tiny_17", 1, 1, 17, 64, False, "outlier"),
    ("ragged_causal", 2, 1, 197, 64, True, "normal"),
]


T_CASES = [
    ("t_small", 1, 2, 300, 64, False, "normal"),
    ("t_causal_outlier_d128", 1, 1, 257, 128, True, "outlier"),
]


VB_CASES = [
    ("vb_small", 1, 2, 300, 64, False, "normal"),
    ("vb_causal_outlier_d128", 1, 1, 257, 128, True, "outlier"),
    ("vb_ragged_causal", 2, 1, 197, 64, True, "normal"),
]


def main_vb():
    ref = Reference()
    for name, b, h, n, d, causal, dist in VB_CASES:
        q, k, v = (x.reshape(b, h, n, d) for x in synth.qkv(b * h, n, d, dtype=np.float16, dist=dist))
        q32, k32, v32 = (x.astype(np.float32) for x in (q, k, v))
        vc = np.empty((b * h, n, d), np.int8)
        vs = np.empty((b * h, d), np.float32)
        for u in range(b * h):
            vc[u], vs[u] = ref.quantize_per_channel(v32.reshape(b * h, n, d)[u])
        o = ref.sage_attention_variant(q32, k32, v32, "VB", causal)
        o_vt = ref.sage_attention_variant(q32, k32, v32, "VT", causal)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), q=q, k=k, v=v, causal=causal, vcodes=vc, vscales=vs,
                            o=o, o_vt=o_vt)
        print(name, "written")


def main_t():
    ref = Reference()
    for name, b, h, n, d, causal, dist in T_CASES:
        q, k, v = (x.reshape(b, h, n, d) for x in synth.qkv(b * h, n, d, dtype=np.float16, dist=dist))
        q32, k32, v32 = (x.astype(np.float32) for x in (q, k, v))
        qc, qs, kc, ks = ref.quantize_per_token(q32, k32)
        o16 = ref.sage_attention_variant(q32, k32, v32, "T", causal, pv_fp32=False)
        o32 = ref.sage_attention_variant(q32, k32, v32, "T", causal, pv_fp32=True)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), q=q, k=k, v=v, causal=causal, qcodes=qc, qscales=qs,
                            kcodes=kc, kscales=ks, o_fp16acc=o16, o_fp32acc=o32)
        print(name, "written")


def main():
    ref = Reference()
    for name, b, h, n, d, causal, dist in CASES:
        q, k, v = (x.reshape(b, h, n, d) for x in synth.qkv(b * h, n, d, dtype=np.float16, dist=dist))
        q32, k32, v32 = (x.astype(np.float32) for x in (q, k, v))
        ks, mean = ref.smooth_k(k32)
        qc, qs = ref.quantize_q(q32)
        kc, kss = ref.quantize_k(k32)
        o16, macs = ref.sage_attention(q32, k32, v32, causal, pv_fp32=False)
        o32, _ = ref.sage_attention(q32, k32, v32, causal, pv_fp32=True)
        exact = ref.naive_attention(q32, k32, v32, causal)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), q=q, k=k, v=v, causal=causal, mean=mean,
                            qcodes=qc, qscales=qs, kcodes=kc, kscales=kss, o_fp16acc=o16, o_fp32acc=o32,
                            macs=macs, exact=exact.astype(np.float32))
        print(name, "written")


if __name__ == "__main__":
    if "--variant-t" in sys.argv:
        main_t()
    elif "--variant-vb" in sys.argv:
        main_vb()
    else:
        main()
