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
