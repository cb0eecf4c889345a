"""GPU parity of SAGEAttn-T: per-token Q/K scales in the same K1/K2.

Bit-exact: K1's per-token codes and scales (Granularity::per_token, quant.hpp:37-63)
against the oracle, which tests/test_oracle.py pins to the compiled reference
(quantize(..., per_token) and sage_attention(in, SageVariant::T)).  The INT32 QK^T
tiles of the T codes are bit-exact.  O within the north-star tolerance of the
reference's FP32-accumulator arm of variant T.
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


def _qkv(b, h, n, d, dist="normal", f32_noise=False):
    q, k, v = synth.qkv(b * h, n, d, dtype=np.float32, dist=dist)
    if f32_noise:
        rng = np.random.default_rng(11)
        q = q + rng.standard_normal(q.shape).astype(np.float32) * 1e-3
        k = k + rng.standard_normal(k.shape).astype(np.float32) * 1e-3
    return [x.reshape(b, h, n, d) for x in (q, k, v)]


def _dev(arrs, dtype, dev):
    import torch

    return [torch.from_numpy(np.ascontiguousarray(a)).to(dev).to(dtype) for a in arrs]


@pytest.mark.parametrize("shape", [(1, 2, 1024, 64), (2, 1, 300, 128), (1, 1, 17, 64), (1, 1, 1, 128),
                                   (1, 1, 17776, 64), (1, 2, 8192, 128)])
@pytest.mark.parametrize("in_f32", [False, True])
def test_prepass_per_token_bit_exact(cuda, oracle, shape, in_f32):
    import torch

    from paper_2410_02367_b200 import prepass_cuda, prepass_outputs

    b, h, n, d = shape
    q, k, v = _qkv(b, h, n, d, dist="outlier", f32_noise=in_f32)
    dt = torch.float32 if in_f32 else torch.float16
    qd, kd, vd = _dev([q, k, v], dt, cuda)
    ws = prepass_cuda(qd, kd, vd if in_f32 else None, per_token=True)
    torch.cuda.synchronize()
    got = {key: t.cpu().numpy() for key, t in prepass_outputs(ws).items()}
    ref = oracle.prepass(q.reshape(b * h, n, d), k.reshape(b * h, n, d), per_token=True)
    for key in ("qcodes", "kcodes"):
        assert np.array_equal(got[key], ref[key]), f"{key} differ at {np.argwhere(got[key] != ref[key])[:5]}"
    for key in ("qscales", "kscales", "mean"):
        assert np.array_equal(np.ascontiguousarray(got[key]).view(np.uint32), ref[key].view(np.uint32)), key


def test_qk_int32_tiles_per_token_codes(cuda, oracle):
    import torch

    from paper_2410_02367_b200 import prepass_cuda, prepass_outputs, qk_int32_tiles_cuda

    n, d = 1105, 128
    q, k, _ = _qkv(1, 1, n, d)
    qd, kd = _dev([q, k], torch.float16, cuda)
    ws = prepass_cuda(qd, kd, per_token=True)
    pre = {key: t.cpu().numpy() for key, t in prepass_outputs(ws).items()}
    for qt in (0, 8):
        tiles = qk_int32_tiles_cuda(ws, 0, qt).cpu().numpy()
        r0, bq = qt * 128, min(128, n - qt * 128)
        for j in range(tiles.shape[0]):
            c0, bkv = j * 64, min(64, n - j * 64)
            ref = oracle.int8_tile(pre["qcodes"][0], pre["kcodes"][0], r0, bq, c0, bkv)
            assert np.array_equal(tiles[j, :bq, :bkv], ref), (qt, j)


T_CASES = [
    ((1, 2, 1024, 64), False, "normal"),
    ((1, 2, 1024, 128), True, "normal"),
    ((1, 1, 1105, 64), True, "outlier"),
    ((1, 1, 300, 128), False, "outlier"),
    ((2, 2, 197, 64), False, "normal"),
    ((1, 1, 2048, 128), True, "outlier"),
]


@pytest.mark.parametrize("shape,causal,dist", T_CASES)
def test_attention_per_token_within_tolerance(cuda, oracle, shape, causal, dist):
    import torch

    from paper_2410_02367_b200 import sage_attention_cuda

    b, h, n, d = shape
    q, k, v = _qkv(b, h, n, d, dist=dist)
    qd, kd, vd = _dev([q, k, v], torch.float16, cuda)
    o = sage_attention_cuda(qd, kd, vd, causal=causal, out_dtype=torch.float32, per_token=True)
    o = o.cpu().numpy().reshape(-1, n, d)
    ref, _ = oracle.sage(q.reshape(-1, n, d), k.reshape(-1, n, d), v.reshape(-1, n, d), causal, pv_fp32=True,
                         per_token=True)
    cs, rl = cosine_sim(o, ref), relative_l1(o, ref)
    assert cs >= COS_MIN and rl <= REL_L1_MAX, (cs, rl)


def test_attention_per_token_sampled_tiles_c2(cuda, oracle):
    import torch

    from paper_2410_02367_b200 import sage_attention_cuda

    n, d, tiles = 8192, 128, [0, 31, 63]
    q, k, v = _qkv(1, 1, n, d)
    qd, kd, vd = _dev([q, k, v], torch.float16, cuda)
    o = sage_attention_cuda(qd, kd, vd, causal=True, out_dtype=torch.float32, per_token=True).cpu().numpy()
    o = o.reshape(n, d)
    pre = oracle.prepass(q.reshape(1, n, d), k.reshape(1, n, d), per_token=True)
    ref = oracle.sage_tiles(pre, v.reshape(1, n, d), 0, tiles, True, pv_fp32=True, per_token=True)
    rows = np.concatenate([np.arange(t * 128, min(n, t * 128 + 128)) for t in tiles])
    cs, rl = cosine_sim(o[rows], ref[rows]), relative_l1(o[rows], ref[rows])
    assert cs >= COS_MIN and rl <= REL_L1_MAX, (cs, rl)


def test_dropin_variant_t(cuda, oracle):
    """sage_attention(in, SageVariant::T) through the host C ABI, fp32 inputs."""
    from paper_2410_02367_b200.sageattn import AttentionInput, SageVariant, sage_attention

    b, h, n, d = 1, 2, 333, 64
    q, k, v = _qkv(b, h, n, d, f32_noise=True)
    o = sage_attention(AttentionInput(q, k, v, causal=True), SageVariant.T)
    ref, _ = oracle.sage(q.reshape(-1, n, d), k.reshape(-1, n, d), v.reshape(-1, n, d), True, pv_fp32=True,
                         per_token=True)
    cs, rl = cosine_sim(o.reshape(-1, n, d), ref), relative_l1(o.reshape(-1, n, d), ref)
    assert cs >= COS_MIN and rl <= REL_L1_MAX, (cs, rl)


GOLDEN_T = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "t_*.npz")))


@pytest.mark.parametrize("path", GOLDEN_T, ids=[os.path.basename(p) for p in GOLDEN_T])
def test_per_token_against_reference_fixtures(cuda, path):
    """K1 per-token codes/scales bit-exact and O within tolerance against vectors the reference produced."""
    import torch

    from paper_2410_02367_b200 import prepass_cuda, prepass_outputs, sage_attention_cuda

    g = np.load(path)
    b, h, n, d = g["q"].shape
    qd, kd, vd = (torch.from_numpy(g[x]).to(cuda) for x in ("q", "k", "v"))
    ws = prepass_cuda(qd, kd, per_token=True)
    got = {key: t.cpu().numpy() for key, t in prepass_outputs(ws).items()}
    assert np.array_equal(got["qcodes"], g["qcodes"].reshape(b * h, n, d))
    assert np.array_equal(got["kcodes"], g["kcodes"].reshape(b * h, n, d))
    assert np.array_equal(np.ascontiguousarray(got["qscales"]).view(np.uint32), g["qscales"].view(np.uint32))
    assert np.array_equal(np.ascontiguousarray(got["kscales"]).view(np.uint32), g["kscales"].view(np.uint32))
    o = sage_attention_cuda(qd, kd, vd, causal=bool(g["causal"]), out_dtype=torch.float32, per_token=True)
    o, ref = o.cpu().numpy().reshape(-1, n, d), g["o_fp32acc"].reshape(-1, n, d)
    cs, rl = cosine_sim(o, ref), relative_l1(o, ref)
    assert cs >= COS_MIN and rl <= REL_L1_MAX, (cs, rl)
