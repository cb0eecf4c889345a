"""RoPE fused into K1 (sab_prepass_rope; "quantization fused into the RoPE kernel").

CPU: the oracle's rotation (oracle/sage_oracle.c orc_rope) against an independent numpy
binary32 restatement (numpy rounds every float32 op, no contraction) -- bit-exact -- and
against a binary64 rotation.  GPU (tests/test_gpu_rope.py): the fused K1 against
oracle.prepass(rope(q), rope(k)) bit for bit, O within the north-star tolerance.
"""
import numpy as np
import pytest


def rope_tables(n, d, base=10000.0):
    """Standard RoPE angles t * base^(-2i/d), cos/sin in binary64 rounded to float32."""
    inv = base ** (-np.arange(0, d // 2, dtype=np.float64) * 2.0 / d)
    ang = np.arange(n, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)


def rope_numpy(x, cos, sin, layout):
    x = x.astype(np.float32)
    d = x.shape[-1]
    h = d // 2
    if layout == "interleaved":
        a, b = x[..., 0::2], x[..., 1::2]
    else:
        a, b = x[..., :h], x[..., h:]
    ra = a * cos - b * sin
    rb = a * sin + b * cos
    out = np.empty_like(x)
    if layout == "interleaved":
        out[..., 0::2], out[..., 1::2] = ra, rb
    else:
        out[..., :h], out[..., h:] = ra, rb
    return out


@pytest.mark.parametrize("layout", ["interleaved", "half"])
@pytest.mark.parametrize("n,d", [(1, 64), (37, 64), (300, 128)])
def test_oracle_rope_bit_exact_vs_numpy(oracle, layout, n, d):
    rng = np.random.default_rng(n + d)
    x = rng.standard_normal((3, n, d)).astype(np.float32) * 3
    cos, sin = rope_tables(n, d)
    got = oracle.rope(x, cos, sin, layout)
    ref = rope_numpy(x, cos, sin, layout)
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))
    # and close to the binary64 rotation
    r64 = rope_numpy(x.astype(np.float64), cos.astype(np.float64), sin.astype(np.float64), layout)
    assert np.max(np.abs(got - r64)) <= 1e-5 * max(1.0, np.max(np.abs(r64)))


def test_oracle_rope_position_zero_is_identity(oracle):
    x = np.random.default_rng(1).standard_normal((2, 1, 128)).astype(np.float32)
    cos, sin = rope_tables(1, 128)
    for layout in ("interleaved", "half"):
        assert np.array_equal(oracle.rope(x, cos, sin, layout), x)
