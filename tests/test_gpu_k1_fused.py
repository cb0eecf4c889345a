"""K1 in one ticketed launch (k1_fused: mean partials, Q chunks and K chunks as work items in
lagged stages, K chunks waiting on a per-unit mean-ready flag) produces exactly the codes,
scales and mean(K) of the two-launch path (k1_mean_and_q -> k1_k_fast / the few-unit
k1_mean_partials -> k1_quantize), for the default lag and both extremes (lag 1: K chunks right
behind their unit's partials; lag = units: every K chunk after every partial), on repeated calls
over one workspace (self-resetting counters) and through the host path's chunked workspace reuse."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(path, **env):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "k1_fused_check.py"), path], capture_output=True,
                       text=True, env=dict(os.environ, SAB_HOST_CHUNK_UNITS="4", **env), timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout + r.stderr
    return np.load(path)


@pytest.fixture(scope="module")
def legacy(tmp_path_factory):
    return _run(str(tmp_path_factory.mktemp("k1") / "legacy.npz"), SAB_K1_FUSED="0")


@pytest.mark.parametrize("lag_pct", ["150", "0", "1000000"])
def test_fused_k1_equals_two_launch_k1(cuda, legacy, tmp_path, lag_pct):
    a = _run(str(tmp_path / "fused.npz"), SAB_K1_FUSED="1", SAB_K1_LAG_PCT=lag_pct)
    assert sorted(a.files) == sorted(legacy.files)
    for key in a.files:
        assert np.array_equal(a[key].view(np.uint8), legacy[key].view(np.uint8)), key
