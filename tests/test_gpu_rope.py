"""GPU parity of the RoPE-fused K1 (sab_prepass_rope): Q^/K^ codes, scales and mean(K) bit-exact
against the oracle's prepass of the rotated tensors (quant.hpp:95-252 on rope(q), rope(k);
oracle/sage_oracle.c orc_rope), and O within the north-star tolerance of the oracle's
FP32-accumulator arm on the rotated inputs.

Tolerance (north star): cos >= 0.9999 and rel-L1 <= 2e-3 of O.
"""
import numpy as np
import pytest

from oracle.oracle import cosine_sim, relative_l1
from test_rope import rope_tables

pytestmark = pytest.mark.gpu
COS_MIN, REL_L1_MAX = 0.9999, 2e-3

CASES = [((1, 2, 300, 64), "half"), ((2, 1, 1105, 128), "interleaved"), ((1, 3, 128, 128), "half"),
         ((1, 1, 17, 64), "interleaved"), ((1, 2, 2048, 128), "half")]


@pytest.mark.parametrize("shape,layout", CASES)
@pytest.mark.parametrize("in_f32", [False, True])
@pytest.mark.parametrize("per_token", [False, True])
def test_rope_prepass_bit_exact(cuda, oracle, shape, layout, in_f32, per_token):
    import torch

    from paper_2410_02367_b200 import prepass_outputs, sageattn

    b, h, n, d = shape
    rng = np.random.default_rng(n * 7 + d)
    q, k = (rng.standard_normal(shape).astype(np.float32) * 2 for _ in range(2))
    if not in_f32:
        q, k = (x.astype(np.float16).astype(np.float32) for x in (q, k))
    cos, sin = rope_tables(n, d)
    dt = torch.float32 if in_f32 else torch.float16
    qd, kd = (torch.from_numpy(x).to(cuda, dt) for x in (q, k))
    tabs = (torch.from_numpy(cos).to(cuda), torch.from_numpy(sin).to(cuda), layout)
    vd = torch.zeros_like(qd) if in_f32 else None
    ws = sageattn.prepass_cuda(qd, kd, vd, per_token=per_token, rope=tabs)
    torch.cuda.synchronize()
    got = {key: t.cpu().numpy() for key, t in prepass_outputs(ws).items()}
    qr = oracle.rope(q.reshape(b * h, n, d), cos, sin, layout)
    kr = oracle.rope(k.reshape(b * h, n, d), cos, sin, layout)
    ref = oracle.prepass(qr, kr, per_token=per_token)
    for key in ("qcodes", "kcodes", "qscales", "kscales", "mean"):
        assert np.array_equal(got[key], ref[key]), key


@pytest.mark.parametrize("shape,layout", CASES[:3])
@pytest.mark.parametrize("causal", [False, True])
def test_rope_attention_within_tolerance(cuda, oracle, shape, layout, causal):
    import torch

    from paper_2410_02367_b200 import sage_attention_cuda

    b, h, n, d = shape
    rng = np.random.default_rng(n + 3)
    q, k, v = (rng.standard_normal(shape).astype(np.float16) for _ in range(3))
    cos, sin = rope_tables(n, d)
    qd, kd, vd = (torch.from_numpy(x).to(cuda) for x in (q, k, v))
    tabs = (torch.from_numpy(cos).to(cuda), torch.from_numpy(sin).to(cuda), layout)
    o = sage_attention_cuda(qd, kd, vd, causal=causal, out_dtype=torch.float32, rope=tabs)
    got = o.cpu().numpy().reshape(-1, n, d)
    qr = oracle.rope(q.reshape(-1, n, d).astype(np.float32), cos, sin, layout)
    kr = oracle.rope(k.reshape(-1, n, d).astype(np.float32), cos, sin, layout)
    ref, _ = oracle.sage_b(qr, kr, v.reshape(-1, n, d).astype(np.float32), causal, pv_fp32=True)
    cs, rl = cosine_sim(got, ref), relative_l1(got, ref)
    assert cs >= COS_MIN and rl <= REL_L1_MAX, (cs, rl)


def test_rope_argument_errors(cuda):
    import torch

    from paper_2410_02367_b200 import sageattn

    q = torch.zeros((1, 1, 64, 64), dtype=torch.float16, device=cuda)
    cos = torch.zeros((64, 32), dtype=torch.float32, device=cuda)
    with pytest.raises(ValueError, match="layout"):
        sageattn.prepass_cuda(q, q, rope=(cos, cos, "diagonal"))
    with pytest.raises(ValueError, match="tables"):
        sageattn.prepass_cuda(q, q, rope=(cos[:, :16].contiguous(), cos, "half"))
    q[0, 0, 5, 7] = float("inf")
    from paper_2410_02367_b200 import _lib

    ws = sageattn.prepass_cuda(q, q, rope=(cos, cos, "half"))
    torch.cuda.synchronize()
    assert sageattn.read_status(ws) == _lib.SAB_ERR_NONFINITE
