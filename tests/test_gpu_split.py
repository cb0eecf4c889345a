"""K2's KV split (sab_ws_layout::kv_chunk): pairs whose KV range is cut into chunks, each
chunk's unnormalised (O, m, l) merged by the pair's last chunk CTA.  The split is the
strong-scaling remedy for K3 shards with few units per device (C2 on 8 GPUs = 4 units per
GPU); its output must stay within the north-star tolerance of the oracle's FP32 arm
(attention.hpp:383-541) on every path, and the C2 4-unit shard must actually split.

Tolerance (north star): cos >= 0.9999 and rel-L1 <= 2e-3 of O.
"""
import ctypes
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from gpu_helpers import _inputs, _run_as_benched
from oracle.oracle import cosine_sim, relative_l1

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
COS_MIN, REL_L1_MAX = 0.9999, 2e-3


def _layout(units, n, d, causal):
    from paper_2410_02367_b200 import _lib

    desc = _lib.SabDesc()
    _lib.load().sab_desc_init(ctypes.byref(desc), 1, units, n, d, int(causal))
    lay = _lib.SabWsLayout()
    _lib.check(_lib.load().sab_workspace_layout(ctypes.byref(desc), ctypes.byref(lay)))
    return lay


def test_split_plan_shapes(cuda):
    """The plan splits the few-unit causal shards and leaves full-size configs alone."""
    c2_shard = _layout(4, 8192, 128, True)  # C2 on 8 GPUs: 4 units per device
    assert c2_shard.kv_chunk > 0 and c2_shard.kv_nchunk > 1
    assert c2_shard.kv_chunk * c2_shard.kv_nchunk >= 128
    for units, n, d, causal in ((32, 8192, 128, True), (128, 16384, 128, False), (60, 17776, 64, False)):
        assert _layout(units, n, d, causal).kv_chunk == 0, (units, n, d, causal)


def test_c2_shard_split_as_benched(cuda, oracle):
    """C2's 8-GPU shard (4 units of (8192, 128), causal) through bench.py's step: split pairs
    (the long causal ones) and unsplit pairs within tolerance, INT32 tiles unchanged."""
    q, k, v = _inputs(4, 8192, 128, cuda)
    o, ws = _run_as_benched(q, k, v, True)
    n = 8192
    for u in range(4):
        tiles = [0, 1, 30, 31, 62, 63] if u in (0, 3) else [40, 41]
        qu, ku, vu = (t[0, u].float().cpu().numpy() for t in (q, k, v))
        pre = oracle.prepass(qu[None], ku[None])
        ref = oracle.sage_b_tiles(pre, vu[None], 0, tiles, True, pv_fp32=True)
        rows = np.concatenate([np.arange(t * 128, min(n, t * 128 + 128)) for t in tiles])
        got = o[0, u].float().cpu().numpy()[rows]
        cs, rl = cosine_sim(got, ref[rows]), relative_l1(got, ref[rows])
        assert cs >= COS_MIN and rl <= REL_L1_MAX, (u, cs, rl)


def test_split_deterministic(cuda):
    """The merge runs in chunk order whichever CTA finishes last: repeated calls are bit-identical."""
    import torch

    q, k, v = _inputs(4, 4096, 128, cuda)
    o1, _ = _run_as_benched(q, k, v, True)
    o2, _ = _run_as_benched(q, k, v, True)
    assert torch.equal(o1, o2)


@pytest.mark.parametrize("chunk", [3, 8])
def test_forced_kv_split_subprocess(cuda, chunk):
    """SAB_KV_SPLIT=<tiles> forces the split on small shapes: B and T, causal (rows with no
    visible key in a chunk) and not, ragged N, both head dims; vB / vT stay unsplit."""
    env = dict(os.environ, SAB_KV_SPLIT=str(chunk))
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "split_check.py")], capture_output=True,
                       text=True, env=env, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout + r.stderr
    res = json.loads(r.stdout.strip().splitlines()[-1])
    for case in res["cases"]:
        if case["pv_int8"]:  # P~ codes depend on the running max: the INT8 P~V path never splits
            assert case["kv_chunk"] == 0, case
        else:
            assert case["kv_chunk"] == chunk and case["nchunk"] > 1, case
        assert case["cos"] >= COS_MIN and case["rel_l1"] <= REL_L1_MAX, case
