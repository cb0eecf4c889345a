"""Persistent K2 (one CTA per SM walking the work items, the next item's loads and first MMAs
overlapping the current item's epilogue) computes every item exactly as the one-CTA-per-item
launch does: outputs are bit-identical, on B, T, vB, causal and not, a KV-split shape."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(mode, path):
    env = dict(os.environ, SAB_K2_PERSIST=mode)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "persist_check.py"), path], capture_output=True,
                       text=True, env=env, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout + r.stderr
    return np.load(path)


def test_persistent_equals_one_cta_per_item(cuda, tmp_path):
    a = _run("1", str(tmp_path / "persist.npz"))
    b = _run("0", str(tmp_path / "single.npz"))
    assert sorted(a.files) == sorted(b.files)
    for key in a.files:
        assert np.isfinite(a[key]).all(), key
        assert np.array_equal(a[key].view(np.uint32), b[key].view(np.uint32)), key


@pytest.mark.parametrize("out_f32", [False, True])
def test_output_alignment_paths_agree(cuda, out_f32):
    """O written with 32-byte stores (32-byte aligned O) and with 16-byte stores (O only 16-byte
    aligned, the C ABI's minimum) is bit-identical."""
    import torch

    from paper_2410_02367_b200 import sage_attention_cuda

    shape = (1, 3, 700, 128)
    g = torch.Generator(device=cuda).manual_seed(7)
    q, k, v = (torch.randn(shape, generator=g, device=cuda).half() for _ in range(3))
    dt = torch.float32 if out_f32 else torch.float16
    a = sage_attention_cuda(q, k, v, causal=True, out_dtype=dt)
    n = a.numel()
    shift = 16 // a.element_size()  # 16 bytes: aligned for the ABI, not for 32-byte stores
    buf = torch.empty(n + shift, dtype=dt, device=cuda)
    b = buf[shift:].view(shape)
    assert b.data_ptr() % 32 == 16
    sage_attention_cuda(q, k, v, causal=True, out=b, out_dtype=dt)
    assert torch.equal(a, b)
