"""Accuracy metrics and adaptive per-layer selection.

CPU: the metric examples and the selection rule's properties as SPEC states them.
GPU: the SPEC's synthetic suite -- layers with outlier-free inputs (vB passes the
0.998 cosine threshold) and layers whose P~ blocks put most of the softmax mass in
probabilities just above the INT8 step (vB fails) -- checked against the rule
evaluated by brute force with the CPU oracle.
"""
import numpy as np
import pytest

from paper_2410_02367_b200 import SageVariant, kernel_config_for
from paper_2410_02367_b200.calibrate import assign, cosine_sim, relative_l1, rmse

VB, B = kernel_config_for(SageVariant.VB), kernel_config_for(SageVariant.B)


def test_metric_examples():
    x = np.array([1.0, 2.0, -3.0])
    assert cosine_sim(x, x) == pytest.approx(1.0)
    assert cosine_sim([1, 0], [0, 1]) == 0.0
    assert cosine_sim([1, 0], [1, 1]) == pytest.approx(1 / np.sqrt(2))
    assert cosine_sim(3.5 * x, x) == pytest.approx(1.0)  # scale invariance
    with pytest.warns(UserWarning):
        assert cosine_sim([0.0, 0.0], [1.0, 2.0]) == 0.0
    assert relative_l1(x, x) == 0.0
    assert relative_l1([1.0], [2.0]) == 0.5
    assert relative_l1([0.0, 0.0], [1.0, -1.0]) == 1.0
    with pytest.raises(ValueError):
        relative_l1([1.0], [0.0])
    assert rmse(x, x) == 0.0
    assert rmse([3.0, 4.0], [0.0, 0.0]) == pytest.approx(np.sqrt(12.5))
    assert rmse([0.0], [1.0]) == 1.0
    with pytest.raises(ValueError):
        cosine_sim([1.0, 2.0], [1.0])


def test_selection_rule():
    plan = assign([0.999, 0.95, 0.998, 0.9981])
    assert plan.assignments == [VB, B, B, VB]  # strictly greater than the threshold
    text = plan.to_text()
    assert "layer 0 SAGEAttn-vB" in text and "layer 1 SAGEAttn-B" in text
    cos = np.random.default_rng(1).uniform(0.99, 1.0, 64)
    assert all(c == VB for c in assign(cos, 0.0).assignments)
    assert all(c == B for c in assign(cos, 1.0).assignments)
    prev = None
    for t in np.linspace(0.99, 1.0, 21):  # raising the threshold never turns B into vB
        cur = [c == VB for c in assign(cos, t).assignments]
        if prev is not None:
            assert all(p or not c for p, c in zip(prev, cur))
        prev = cur
    with pytest.raises(ValueError):
        assign([0.9], 1.5)


def _layer(kind, seed, n=2048, d=64, heads=2):
    rng = np.random.default_rng(seed)
    if kind == "normal":
        q, k, v = (rng.standard_normal((1, heads, n, d)).astype(np.float32) for _ in range(3))
        return q, k, v
    # Every query prefers one key in 97 by a score gap of 5: the other keys keep p = e^-5, just above
    # INT8 P~'s 1/254 step, so vB rounds ~97 % of the softmax mass up by ~17 %.  V is biased so that
    # the error survives the average.
    u = np.ones(d, np.float32) / np.sqrt(d)
    q = (u * 8 + rng.standard_normal((1, heads, n, d)) * 0.1).astype(np.float32)
    k = (rng.standard_normal((1, heads, n, d)) * 0.1).astype(np.float32)
    k[:, :, ::97] = u * 5
    v = (1 + rng.standard_normal((1, heads, n, d)) * 0.3).astype(np.float32)
    v[:, :, ::97] = -1 + rng.standard_normal((1, heads, (n + 96) // 97, d)).astype(np.float32) * 0.3
    return q, k, v


@pytest.mark.gpu
def test_calibrate_synthetic_suite(cuda, oracle):
    import torch

    from paper_2410_02367_b200.calibrate import calibrate

    kinds = ["normal", "extreme", "normal", "extreme"]
    host = [[_layer(kind, 10 * i + b) for b in range(2)] for i, kind in enumerate(kinds)]
    layers = [[tuple(torch.from_numpy(x).to(cuda) for x in qkv) + (False,) for qkv in batches] for batches in host]
    plan = calibrate(layers)
    # Brute force: the rule evaluated with the oracle's vB output against exact attention.
    expect = []
    for batches in host:
        cs = []
        for q, k, v in batches:
            n, d = q.shape[2], q.shape[3]
            q3, k3, v3 = (x.reshape(-1, n, d) for x in (q, k, v))
            o, _ = oracle.sage(q3, k3, v3, False, pv_int8=True)
            cs.append(cosine_sim(o, oracle.naive(q3, k3, v3, False)))
        expect.append(np.mean(cs))
    assert [c == VB for c in plan.assignments] == [e > 0.998 for e in expect]
    assert [c == VB for c in plan.assignments] == [True, False, True, False]
    assert np.allclose(plan.cos_sim, expect, atol=2e-4)
    assert calibrate(layers, aggregate="min").assignments == plan.assignments
    with pytest.raises(ValueError):
        calibrate([])
