"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bit-exact: mean_k, Q^/K^ codes, per-block scales (K1) and the INT32 QK^T tiles
(K2's tcgen05 kind::i8).  Tolerance (north star): cos >= 0.9999 and
relative L1 <= 2e-3 of O against the reference's FP32-accumulator arm
(SageOptions::pv_fp32_accumulator, attention.hpp:454-471); error against
the default FP16 arm and against exact attention is reported, not gated.
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


def _to_dev(arrs, dtype, dev):
    import torch

    return [torch.from_numpy(np.ascontiguousarray(a)).to(dev).to(dtype) for a in arrs]


def _qkv(b, h, n, d, dist="normal", f32_noise=False):
    q, k, v = synth.qkv(b * h, n, d, dtype=np.float32, dist=dist)
    if f32_noise:  # values that are not on the fp16 grid exercise the fp32 prepass path
        rng = np.random.default_rng(7)
        q = q + rng.standard_normal(q.shape).astype(np.float32) * 1e-3
        k = k + rng.standard_normal(k.shape).astype(np.float32) * 1e-3
    return [x.reshape(b, h, n, d) for x in (q, k, v)]


PREPASS_SHAPES = [
    (1, 2, 1024, 64), (2, 3, 300, 128), (1, 1, 17, 64), (1, 1, 8, 128), (1, 1, 1, 64), (1, 2, 1105, 64),
    (1, 2, 8192, 128), (1, 1, 17776, 64), (1, 1, 131072, 128), (1, 1, 100003, 64), (2, 2, 197, 64),
]


@pytest.mark.parametrize("shape", PREPASS_SHAPES)
@pytest.mark.parametrize("in_f32", [False, True])
def test_prepass_bit_exact(cuda, oracle, shape, in_f32):
    import torch

    from paper_2410_02367_b200 import prepass_cuda, prepass_outputs

    b, h, n, d = shape
    q, k, v = _qkv(b, h, n, d, dist="outlier", f32_noise=in_f32)
    dt = torch.float32 if in_f32 else torch.float16
    qd, kd, vd = _to_dev([q, k, v], dt, cuda)
    ws = prepass_cuda(qd, kd, vd if in_f32 else None)
    torch.cuda.synchronize()
    got = {key: t.cpu().numpy() for key, t in prepass_outputs(ws).items()}
    if in_f32:  # V on the binary16 grid (attention.hpp:371-375; RNE == round_to_half)
        v16 = ws.view("v16", torch.float16, (b * h, n, d)).cpu().numpy()
        assert np.array_equal(v16.view(np.uint16), v.reshape(b * h, n, d).astype(np.float16).view(np.uint16))
    ref = oracle.prepass(q.reshape(b * h, n, d), k.reshape(b * h, n, d))
    for key in ("qcodes", "kcodes"):
        assert np.array_equal(got[key], ref[key]), f"{key} differ at {np.argwhere(got[key] != ref[key])[:5]}"
    for key in ("qscales", "kscales", "mean"):
        assert np.array_equal(got[key].view(np.uint32), ref[key].view(np.uint32)), key


@pytest.mark.parametrize("shape,causal", [((1, 2, 1024, 64), False), ((1, 2, 1024, 128), True),
                                          ((1, 1, 1105, 64), True), ((1, 1, 300, 128), False),
                                          ((1, 1, 8192, 128), True)])
def test_qk_int32_tiles_bit_exact(cuda, oracle, shape, causal):
    import torch

    from paper_2410_02367_b200 import prepass_cuda, prepass_outputs, qk_int32_tiles_cuda, sageattn

    b, h, n, d = shape
    q, k, v = _qkv(b, h, n, d)
    qd, kd = _to_dev([q, k], torch.float16, cuda)
    ws = prepass_cuda(qd, kd)
    ws.desc.causal = int(causal)
    pre = {key: t.cpu().numpy() for key, t in prepass_outputs(ws).items()}
    ntq = -(-n // 128)
    for unit in range(b * h):
        for qt in sorted({0, ntq // 2, ntq - 1}):
            tiles = qk_int32_tiles_cuda(ws, unit, qt).cpu().numpy()
            r0, bq = qt * 128, min(128, n - qt * 128)
            for j in range(tiles.shape[0]):
                c0, bkv = j * 64, min(64, n - j * 64)
                ref = oracle.int8_tile(pre["qcodes"][unit], pre["kcodes"][unit], r0, bq, c0, bkv)
                assert np.array_equal(tiles[j, :bq, :bkv], ref), (unit, qt, j)


ATTN_CASES = [
    ((1, 2, 1024, 64), False, "normal"),      # C1
    ((1, 2, 1024, 64), True, "normal"),
    ((1, 2, 1024, 128), False, "outlier"),
    ((1, 2, 1024, 128), True, "normal"),
    ((1, 1, 1105, 64), True, "outlier"),      # ragged 81-row last Q tile, 17-key last K group
    ((1, 1, 300, 128), False, "normal"),
    ((2, 2, 197, 64), False, "normal"),       # TIMM-like: one ragged Q tile
    ((1, 1, 64, 128), True, "normal"),
    ((1, 1, 2048, 128), True, "outlier"),
]


@pytest.mark.parametrize("shape,causal,dist", ATTN_CASES)
def test_attention_within_tolerance(cuda, oracle, shape, causal, dist):
    import torch

    from paper_2410_02367_b200 import sage_attention_cuda

    b, h, n, d = shape
    q, k, v = _qkv(b, h, n, d, dist=dist)
    qd, kd, vd = _to_dev([q, k, v], torch.float16, cuda)
    o = sage_attention_cuda(qd, kd, vd, causal=causal, out_dtype=torch.float32).cpu().numpy()
    ref32, _ = oracle.sage_b(q.reshape(-1, n, d), k.reshape(-1, n, d), v.reshape(-1, n, d), causal, pv_fp32=True)
    o = o.reshape(-1, n, d)
    cs, rl = cosine_sim(o, ref32), relative_l1(o, ref32)
    assert cs >= COS_MIN and rl <= REL_L1_MAX, (cs, rl)


@pytest.mark.parametrize("shape,causal,tiles", [((1, 1, 8192, 128), True, [0, 31, 63]),
                                                ((1, 1, 17776, 64), False, [0, 70, 138]),
                                                ((1, 1, 16384, 128), False, [5, 127]),
                                                ((1, 1, 131072, 128), True, [0, 3, 40])])  # C5 unit
def test_attention_sampled_tiles_large(cuda, oracle, shape, causal, tiles):
    """C2 / C3 / C4 / C5 shapes: compare sampled query tiles (units and q-tiles are independent)."""
    import torch

    from paper_2410_02367_b200 import sage_attention_cuda

    b, h, n, d = shape
    q, k, v = _qkv(b, h, n, d)
    qd, kd, vd = _to_dev([q, k, v], torch.float16, cuda)
    o = sage_attention_cuda(qd, kd, vd, causal=causal, out_dtype=torch.float32).cpu().numpy().reshape(n, d)
    pre = oracle.prepass(q.reshape(1, n, d), k.reshape(1, n, d))
    ref = oracle.sage_b_tiles(pre, v.reshape(1, n, d), 0, tiles, causal, pv_fp32=True)
    rows = np.concatenate([np.arange(t * 128, min(n, t * 128 + 128)) for t in tiles])
    cs, rl = cosine_sim(o[rows], ref[rows]), relative_l1(o[rows], ref[rows])
    assert cs >= COS_MIN and rl <= REL_L1_MAX, (cs, rl)


def test_fp16_output_and_host_path_agree(cuda, oracle):
    import torch

    from paper_2410_02367_b200 import AttentionInput, SageVariant, sage_attention, sage_attention_cuda

    b, h, n, d = 1, 4, 640, 128
    q, k, v = _qkv(b, h, n, d, dist="outlier")
    qd, kd, vd = _to_dev([q, k, v], torch.float16, cuda)
    o16 = sage_attention_cuda(qd, kd, vd, causal=True).float().cpu().numpy()
    o_host = sage_attention(AttentionInput(q.astype(np.float16), k.astype(np.float16), v.astype(np.float16), True),
                            SageVariant.B)
    o_host32 = sage_attention(AttentionInput(q, k, v, True), SageVariant.B)  # fp32 inputs: same values
    assert np.array_equal(o_host, o_host32)
    assert np.abs(o16 - o_host).max() <= 1e-3
    ref32, _ = oracle.sage_b(q.reshape(-1, n, d), k.reshape(-1, n, d), v.reshape(-1, n, d), True, pv_fp32=True)
    assert cosine_sim(o_host.reshape(-1, n, d), ref32) >= COS_MIN


def test_error_paths(cuda):
    from paper_2410_02367_b200 import (AttentionInput, KernelConfig, SageOptions, SageVariant, QuantDtype,
                                       sage_attention)

    q, k, v = _qkv(1, 1, 256, 64)
    with pytest.raises(ValueError, match="Q, K, V shapes differ"):
        sage_attention(AttentionInput(q, k[:, :, :128], v), SageVariant.B)
    with pytest.raises(ValueError, match="block sizes must be >= 1"):
        sage_attention(AttentionInput(q, k, v), KernelConfig(block_q=0))
    bad = q.copy()
    bad[0, 0, 100, 3] = np.inf
    with pytest.raises(ValueError, match="non-finite input"):
        sage_attention(AttentionInput(bad, k, v), SageVariant.B)
    badv = v.copy()
    badv[0, 0, 7, 1] = np.nan
    with pytest.raises(ValueError, match="non-finite input"):
        sage_attention(AttentionInput(q, k, badv), SageVariant.B)
    with pytest.raises(ValueError):
        sage_attention(AttentionInput(q, k, v), SageVariant.B, SageOptions(qk_dtype=QuantDtype.FpE4M3))


def test_multi_shard_host_path_equals_single(cuda):
    """K3 on the host path: shards are bit-identical to the unsharded call (same device twice here)."""
    from paper_2410_02367_b200 import attention_fwd_host

    q, k, v = (x.astype(np.float16) for x in _qkv(2, 3, 384, 64))
    o1 = attention_fwd_host(q, k, v, True, np.empty(q.shape, np.float32), devices=[0])
    o2 = attention_fwd_host(q, k, v, True, np.empty(q.shape, np.float32), devices=[0, 0, 0, 0])
    assert np.array_equal(o1, o2)


def test_host_path_many_chunks_equals_device_path(cuda):
    """Host path with many unit chunks (per-chunk K1 counters and status words) equals the device call."""
    import torch

    from paper_2410_02367_b200 import attention_fwd_host, sage_attention_cuda

    q, k, v = (x.astype(np.float16) for x in _qkv(2, 40, 200, 64))
    oh = attention_fwd_host(q, k, v, False, np.empty(q.shape, np.float32), devices=[0])
    qd, kd, vd = (torch.from_numpy(x).cuda() for x in (q, k, v))
    od = sage_attention_cuda(qd, kd, vd, causal=False, out_dtype=torch.float32).cpu().numpy()
    assert np.array_equal(oh, od)


GOLDEN_B = sorted(p for p in glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz"))
                  if not os.path.basename(p).startswith(("t_", "vb_")))


@pytest.mark.parametrize("path", GOLDEN_B, ids=[os.path.basename(p) for p in GOLDEN_B])
def test_against_reference_fixtures(cuda, path):
    """K1 bit-exact and O within tolerance against vectors produced by the reference itself."""
    import torch

    from paper_2410_02367_b200 import prepass_cuda, prepass_outputs, sage_attention_cuda

    g = np.load(path)
    b, h, n, d = g["q"].shape
    qd, kd, vd = (torch.from_numpy(g[x]).to(cuda) for x in ("q", "k", "v"))
    got = {key: t.cpu().numpy() for key, t in prepass_outputs(prepass_cuda(qd, kd)).items()}
    assert np.array_equal(got["qcodes"], g["qcodes"].reshape(b * h, n, d))
    assert np.array_equal(got["kcodes"], g["kcodes"].reshape(b * h, n, d))
    assert np.array_equal(got["qscales"].view(np.uint32), g["qscales"].view(np.uint32))
    assert np.array_equal(got["kscales"].view(np.uint32), g["kscales"].view(np.uint32))
    assert np.array_equal(got["mean"].view(np.uint32), g["mean"].reshape(b * h, d).view(np.uint32))
    o = sage_attention_cuda(qd, kd, vd, causal=bool(g["causal"]), out_dtype=torch.float32).cpu().numpy()
    o, ref = o.reshape(-1, n, d), g["o_fp32acc"].reshape(-1, n, d)
    cs, rl = cosine_sim(o, ref), relative_l1(o, ref)
    assert cs >= COS_MIN and rl <= REL_L1_MAX, (cs, rl)


def test_many_units_host_path_and_device_limit(cuda, oracle):
    """B*H above K1's 65535-unit grid: the host path chunks it, a single device call refuses it."""
    import torch

    from paper_2410_02367_b200 import attention_fwd_host, sage_attention_cuda

    b, h, n, d = 1, 70000, 3, 64
    q, k, v = (x.astype(np.float16) for x in _qkv(b, h, n, d))
    o = attention_fwd_host(q, k, v, False, np.empty(q.shape, np.float32), devices=[0]).reshape(-1, n, d)
    sel = np.array([0, 65534, 65535, 69999])
    ref, _ = oracle.sage_b(q.reshape(-1, n, d)[sel].astype(np.float32), k.reshape(-1, n, d)[sel].astype(np.float32),
                           v.reshape(-1, n, d)[sel].astype(np.float32), False, pv_fp32=True)
    assert cosine_sim(o[sel], ref) >= COS_MIN and relative_l1(o[sel], ref) <= REL_L1_MAX
    qd, kd, vd = _to_dev([q, k, v], torch.float16, cuda)
    with pytest.raises(ValueError, match="65535"):
        sage_attention_cuda(qd, kd, vd)


def test_host_path_pageable_and_pinned_agree(cuda):
    """Pageable caller buffers are staged through pinned chunks (sab_capi.cu); pinned ones go
    straight to cudaMemcpyAsync: both give the device path's output bit for bit."""
    import torch

    from paper_2410_02367_b200 import attention_fwd_host

    q, k, v = (x.astype(np.float16) for x in _qkv(2, 24, 1000, 128))
    o_page = attention_fwd_host(q, k, v, True, np.empty(q.shape, np.float32), devices=[0])
    pq, pk, pv = (torch.from_numpy(x).pin_memory().numpy() for x in (q, k, v))
    po = torch.empty(q.shape, dtype=torch.float32).pin_memory().numpy()
    attention_fwd_host(pq, pk, pv, True, po, devices=[0])
    assert np.array_equal(o_page, po)
