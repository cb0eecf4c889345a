"""GPU parity of SAGEAttn-vB / -vT: static-scale INT8 P~, per-channel INT8 V,
INT32 P~V products on tcgen05 kind::i8, in the same K1/K2 (vT: with per-token Q/K scales).

Bit-exact: K1's per-channel V^ codes and scales (quantize(V, per_channel), quant.hpp:128-173)
against the oracle, which tests/test_oracle.py pins to the compiled reference
(sage_attention(in, SageVariant::VB)).  O within the north-star tolerance
(cos >= 0.9999, rel-L1 <= 2e-3) of the reference's own vB output.
"""
import glob
import os

import numpy as np
import pytest

from oracle.oracle import cosine_sim, relative_l1
from paper_2410_02367_b200 import synth

pytestmark = pytest.mark.gpu

COS_MIN = 0.9999
REL_L1_MAX = 2e-3


def _qkv(b, h, n, d, dist="normal"):
    return [x.reshape(b, h, n, d) for x in synth.qkv(b * h, n, d, dtype=np.float32, dist=dist)]


def _dev(arrs, dtype, dev):
    import torch

    return [torch.from_numpy(np.ascontiguousarray(a)).to(dev).to(dtype) for a in arrs]


@pytest.mark.parametrize("shape", [(1, 2, 1024, 64), (2, 1, 300, 128), (1, 1, 17, 64), (1, 1, 1, 128),
                                   (1, 1, 17776, 64), (1, 2, 8192, 128)])
@pytest.mark.parametrize("in_f32", [False, True])
def test_prepass_v_per_channel_bit_exact(cuda, oracle, shape, in_f32):
    import torch

    from paper_2410_02367_b200 import prepass_cuda, prepass_outputs

    b, h, n, d = shape
    q, k, v = _qkv(b, h, n, d, dist="outlier")
    if in_f32:
        v = v + np.random.default_rng(5).standard_normal(v.shape).astype(np.float32) * 1e-3
    dt = torch.float32 if in_f32 else torch.float16
    qd, kd, vd = _dev([q, k, v], dt, cuda)
    ws = prepass_cuda(qd, kd, vd, pv_int8=True)
    torch.cuda.synchronize()
    got = prepass_outputs(ws)
    vc, vs = got["vcodes"].cpu().numpy(), got["vscales"].cpu().numpy()
    vin = v.reshape(b * h, n, d) if in_f32 else v.reshape(b * h, n, d).astype(np.float16).astype(np.float32)
    for u in range(b * h):
        rc, rs = oracle.quantize_per_channel(vin[u])
        assert np.array_equal(vc[u], rc), f"unit {u}: codes differ at {np.argwhere(vc[u] != rc)[:5]}"
        assert np.array_equal(vs[u].view(np.uint32), rs.view(np.uint32)), f"unit {u}: scales differ"
    # The Q/K half of K1 is unchanged by the INT8 P~V path.
    ref = oracle.prepass(q.reshape(b * h, n, d), k.reshape(b * h, n, d)) if in_f32 else \
        oracle.prepass(*(x.reshape(b * h, n, d).astype(np.float16).astype(np.float32) for x in (q, k)))
    for key in ("qcodes", "kcodes"):
        assert np.array_equal(got[key].cpu().numpy(), ref[key]), key


VB_CASES = [
    ((1, 2, 1024, 64), False, "normal"),
    ((1, 2, 1024, 128), True, "normal"),
    ((1, 1, 1105, 64), True, "outlier"),
    ((1, 1, 300, 128), False, "outlier"),
    ((2, 2, 197, 64), False, "normal"),
    ((1, 1, 2048, 128), True, "outlier"),
    ((1, 1, 4096, 64), False, "normal"),
    ((1, 1, 1, 64), False, "normal"),
]


@pytest.mark.parametrize("per_token", [False, True], ids=["vB", "vT"])
@pytest.mark.parametrize("shape,causal,dist", VB_CASES)
def test_attention_vb_within_tolerance(cuda, oracle, shape, causal, dist, per_token):
    import torch

    from paper_2410_02367_b200 import sage_attention_cuda

    b, h, n, d = shape
    q, k, v = _qkv(b, h, n, d, dist=dist)
    qd, kd, vd = _dev([q, k, v], torch.float16, cuda)
    o = sage_attention_cuda(qd, kd, vd, causal=causal, out_dtype=torch.float32, pv_int8=True, per_token=per_token)
    o = o.cpu().numpy().reshape(-1, n, d)
    f16 = [x.reshape(-1, n, d).astype(np.float16).astype(np.float32) for x in (q, k, v)]
    ref, _ = oracle.sage(*f16, causal, pv_int8=True, per_token=per_token)
    cs, rl = cosine_sim(o, ref), relative_l1(o, ref)
    assert cs >= COS_MIN and rl <= REL_L1_MAX, (cs, rl)


def test_dropin_variant_vb(cuda, oracle):
    """sage_attention(in, SageVariant::VB / VT) through the host C ABI, fp32 inputs (V^ from fp32 V)."""
    from paper_2410_02367_b200.sageattn import AttentionInput, SageVariant, sage_attention

    b, h, n, d = 1, 2, 333, 64
    q, k, v = _qkv(b, h, n, d)
    v = v + np.random.default_rng(9).standard_normal(v.shape).astype(np.float32) * 1e-3
    o = sage_attention(AttentionInput(q, k, v, causal=True), SageVariant.VB)
    ref, _ = oracle.sage(q.reshape(-1, n, d), k.reshape(-1, n, d), v.reshape(-1, n, d), True, pv_int8=True)
    cs, rl = cosine_sim(o.reshape(-1, n, d), ref), relative_l1(o.reshape(-1, n, d), ref)
    assert cs >= COS_MIN and rl <= REL_L1_MAX, (cs, rl)
    o = sage_attention(AttentionInput(q, k, v, causal=True), SageVariant.VT)
    ref, _ = oracle.sage(q.reshape(-1, n, d), k.reshape(-1, n, d), v.reshape(-1, n, d), True, pv_int8=True,
                         per_token=True)
    cs, rl = cosine_sim(o.reshape(-1, n, d), ref), relative_l1(o.reshape(-1, n, d), ref)
    assert cs >= COS_MIN and rl <= REL_L1_MAX, (cs, rl)
    v[0, 1, 7, 3] = np.inf
    with pytest.raises(ValueError, match="non-finite"):
        sage_attention(AttentionInput(q, k, v), SageVariant.VB)


GOLDEN_VB = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "vb_*.npz")))


@pytest.mark.parametrize("path", GOLDEN_VB, ids=[os.path.basename(p) for p in GOLDEN_VB])
def test_vb_against_reference_fixtures(cuda, path):
    """V^ codes/scales bit-exact and O within tolerance against vectors the reference produced."""
    import torch

    from paper_2410_02367_b200 import prepass_cuda, prepass_outputs, sage_attention_cuda

    g = np.load(path)
    b, h, n, d = g["q"].shape
    qd, kd, vd = (torch.from_numpy(g[x]).to(cuda) for x in ("q", "k", "v"))
    ws = prepass_cuda(qd, kd, vd, pv_int8=True)
    got = prepass_outputs(ws)
    assert np.array_equal(got["vcodes"].cpu().numpy(), g["vcodes"])
    assert np.array_equal(got["vscales"].cpu().numpy().view(np.uint32), g["vscales"].view(np.uint32))
    o = sage_attention_cuda(qd, kd, vd, causal=bool(g["causal"]), out_dtype=torch.float32, pv_int8=True)
    o, ref = o.cpu().numpy().reshape(-1, n, d), g["o"].reshape(-1, n, d)
    cs, rl = cosine_sim(o, ref), relative_l1(o, ref)
    assert cs >= COS_MIN and rl <= REL_L1_MAX, (cs, rl)
    o = sage_attention_cuda(qd, kd, vd, causal=bool(g["causal"]), out_dtype=torch.float32, pv_int8=True,
                            per_token=True)
    o, ref = o.cpu().numpy().reshape(-1, n, d), g["o_vt"].reshape(-1, n, d)
    cs, rl = cosine_sim(o, ref), relative_l1(o, ref)
    assert cs >= COS_MIN and rl <= REL_L1_MAX, ("vT", cs, rl)


@pytest.mark.parametrize("per_token", [False, True])
@pytest.mark.parametrize("heads,n,d", [(35, 1024, 64), (79, 512, 128)])
def test_host_path_short_last_chunk_int8_pv(cuda, per_token, heads, n, d):
    """Host path with a short last unit chunk (35 units -> chunks of 4, last 3) on the INT8 P~V path:
    every chunk keeps the full-chunk workspace layout, so V^ / delta_V never overlay the status
    word -- the output equals the one-call device path bit for bit and no spurious error is raised."""
    import torch

    from paper_2410_02367_b200 import attention_fwd_host, sage_attention_cuda

    q, k, v = (x.astype(np.float16) for x in _qkv(1, heads, n, d))
    oh = attention_fwd_host(q, k, v, True, np.empty(q.shape, np.float32), devices=[0], per_token=per_token,
                            pv_int8=True)
    qd, kd, vd = (torch.from_numpy(x).to(cuda) for x in (q, k, v))
    od = sage_attention_cuda(qd, kd, vd, causal=True, out_dtype=torch.float32, per_token=per_token, pv_int8=True)
    assert np.array_equal(oh, od.cpu().numpy())


def test_int8_pv_token_limit(cuda):
    """The INT32 P~V accumulator bound: more than 133144 keys are refused on vB / vT (ValueError)."""
    from paper_2410_02367_b200 import _lib

    d = _lib.desc(1, 1, 133145, 64, pv_int8=True)
    with pytest.raises(_lib.SabError, match="133144"):
        _lib.check(_lib.load().sab_check_desc(d))
    _lib.check(_lib.load().sab_check_desc(_lib.desc(1, 1, 133144, 64, pv_int8=True)))


@pytest.mark.parametrize("causal,per_token", [(False, False), (True, False), (True, True)])
def test_static_scale_diagnostics(cuda, reference, causal, per_token):
    """SageDiagnostics::measure_static_scale on vB / vT (attention.hpp:479-488): the element count
    equals the reference's, the mismatch counts agree with it to 1 % (the GPU's P~ differs from the
    reference's by exponential ulps, which can move a code across a rounding boundary)."""
    from paper_2410_02367_b200.sageattn import (AttentionInput, SageDiagnostics, SageOptions, SageVariant,
                                                sage_attention)

    b, h, n, d = 1, 3, 700, 64
    q, k, v = _qkv(b, h, n, d)
    diag = SageDiagnostics(measure_static_scale=True)
    sage_attention(AttentionInput(q, k, v, causal), SageVariant.VT if per_token else SageVariant.VB,
                   SageOptions(diagnostics=diag))
    el, first, later = reference.static_scale_counts(q, k, v, causal, per_token)
    assert diag.static_scale_elements == el
    assert abs(diag.static_scale_first_block_mismatches - first) <= max(2, 0.01 * first)
    assert abs(diag.static_scale_later_block_mismatches - later) <= max(2, 0.01 * later)
    assert later > 0  # static scales do differ from per-token ones after the first block
