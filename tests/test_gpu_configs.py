"""GPU parity on every BASELINE config exactly as bench.py runs it.

Each test generates the config's full synthetic inputs on the device (bench.py's
generator), runs K1 + K2 through the same two C-ABI calls bench.py times
(sab_prepass + sab_attention, fp16 O, the same descriptor and hence the same
L2-raster grouping and query-tile pairing), and compares sampled (unit, query
tile) rows of that output with the oracle's FP32-accumulator arm -- the
reference's per-unit engine (attention.hpp:357-360, 383-541), bit-identical to
it (tests/test_oracle.py).  Units and query tiles are independent, so
sampled rows are exact stand-ins for the whole call.  INT32 QK^T tiles of the
same codes are compared bit-exactly (attention.hpp:265-279).

Tolerance (north star): cos >= 0.9999 and rel-L1 <= 2e-3 of O.
"""
import json
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from gpu_helpers import _inputs, _run_as_benched
from oracle.oracle import cosine_sim, relative_l1

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
COS_MIN, REL_L1_MAX = 0.9999, 2e-3
THREADS = max(2, min(32, os.cpu_count() or 2))


def _host_unit(t, u):
    return t[0, u].float().cpu().numpy()


def _check_units(oracle, q, k, v, o, causal, picks):
    """picks: {unit: [q-tiles]}; oracle FP32 arm per unit on a thread each."""
    n = q.shape[2]

    def one(item):
        u, tiles = item
        qu, ku, vu = _host_unit(q, u), _host_unit(k, u), _host_unit(v, u)
        pre = oracle.prepass(qu[None], ku[None])
        ref = oracle.sage_b_tiles(pre, vu[None], 0, tiles, causal, pv_fp32=True)
        rows = np.concatenate([np.arange(t * 128, min(n, t * 128 + 128)) for t in tiles])
        got = o[0, u].float().cpu().numpy()[rows]
        return u, cosine_sim(got, ref[rows]), relative_l1(got, ref[rows])

    with ThreadPoolExecutor(THREADS) as ex:
        res = list(ex.map(one, sorted(picks.items())))
    for u, cs, rl in res:
        assert cs >= COS_MIN and rl <= REL_L1_MAX, (u, cs, rl)
    return res


def _check_int32(oracle, ws, q, k, unit, q_tile, kv_sample=None):
    """K2's tcgen05 kind::i8 S tiles of (unit, q_tile) against int8_tile_nt on the same codes."""
    from paper_2410_02367_b200 import prepass_outputs, qk_int32_tiles_cuda

    n = q.shape[2]
    pre = prepass_outputs(ws)
    qc, kc = pre["qcodes"][unit].cpu().numpy(), pre["kcodes"][unit].cpu().numpy()
    tiles = qk_int32_tiles_cuda(ws, unit, q_tile).cpu().numpy()
    r0, bq = q_tile * 128, min(128, n - q_tile * 128)
    js = range(tiles.shape[0]) if kv_sample is None else sorted({j for j in kv_sample if j < tiles.shape[0]} |
                                                                 {tiles.shape[0] - 1})
    for j in js:
        c0, bkv = j * 64, min(64, n - j * 64)
        assert np.array_equal(tiles[j, :bq, :bkv], oracle.int8_tile(qc, kc, r0, bq, c0, bkv)), (unit, q_tile, j)


def _pair_tiles(n, which):
    """First / middle / last query-tile pair of K2's (2 tiles per CTA) pairing."""
    ntq = -(-n // 128)
    npair = (ntq + 1) // 2
    out = []
    for p in {"first": [0], "middle": [npair // 2], "last": [npair - 1]}[which] if isinstance(which, str) else which:
        out += [t for t in (2 * p, 2 * p + 1) if t < ntq]
    return out


def _all_pairs(n):
    return sorted(set(_pair_tiles(n, "first") + _pair_tiles(n, "middle") + _pair_tiles(n, "last")))


def test_c2_full_as_benched(cuda, oracle):
    """C2 (1,32,8192,128) causal: 32 units = 4 L2 raster groups of 8; one unit per group,
    first / middle / last query-tile pair; INT32 tiles of the last pair of one unit."""
    q, k, v = _inputs(32, 8192, 128, cuda)
    o, ws = _run_as_benched(q, k, v, True)
    tiles = _all_pairs(8192)
    _check_units(oracle, q, k, v, o, True, {u: tiles for u in (0, 9, 18, 31)})
    ws.desc.causal = 1
    _check_int32(oracle, ws, q, k, 31, 63)
    _check_int32(oracle, ws, q, k, 9, 32, kv_sample=range(0, 66, 5))


def test_c3_full_as_benched(cuda, oracle):
    """C3 (2,30,17776,64): units 0, 29, 30, 59 incl. the 112-row Q tail (tile 138) and the
    48-key K tail; INT32 tiles at N=17776, d=64."""
    q, k, v = _inputs(60, 17776, 64, cuda)
    o, ws = _run_as_benched(q, k, v, False)
    tiles = _all_pairs(17776)
    assert 138 in tiles
    _check_units(oracle, q, k, v, o, False, {u: tiles for u in (0, 29, 30, 59)})
    _check_int32(oracle, ws, q, k, 59, 138)
    _check_int32(oracle, ws, q, k, 30, 70, kv_sample=range(0, 278, 23))


C4_POINTS = [(d, n, c) for d in (64, 128) for n in (1024, 2048, 4096, 8192, 16384, 32768) for c in (True, False)]


@pytest.mark.parametrize("d,n,causal", C4_POINTS, ids=[f"C4-{d}-{n}-{'c' if c else 'nc'}" for d, n, c in C4_POINTS])
def test_c4_point_as_benched(cuda, oracle, d, n, causal):
    """Every C4 kernel-bench point (4,32,N,d): one unit from each end of the batch, first /
    middle / last tile pair, INT32 tiles of the middle pair."""
    q, k, v = _inputs(128, n, d, cuda)
    o, ws = _run_as_benched(q, k, v, causal)
    tiles = _all_pairs(n)
    _check_units(oracle, q, k, v, o, causal, {5: tiles, 127: _pair_tiles(n, "last")})
    ws.desc.causal = int(causal)
    mid = _pair_tiles(n, "middle")[0]
    _check_int32(oracle, ws, q, k, 77, mid, kv_sample=range(0, 2 * mid + 2, max(1, (2 * mid + 2) // 6)))


def test_c5_shard_boundary(cuda, oracle):
    """C5 (1,64,131072,128) causal as one call, and the 8-GPU shard of rank 1 (units 8-15)
    as its own call (bench.py under torchrun): bit-identical, and unit 8 -- the first unit
    past the shard boundary -- within tolerance on first / middle / last tiles."""
    import torch

    from paper_2410_02367_b200 import _lib

    q, k, v = _inputs(64, 131072, 128, cuda)
    o, ws = _run_as_benched(q, k, v, True)
    first, count = _lib.shard_plan(64, 8, 1)
    assert (first, count) == (8, 8)
    qs, ks, vs = (t[:, first:first + count].contiguous() for t in (q, k, v))
    o_shard, _ = _run_as_benched(qs, ks, vs, True)
    assert torch.equal(o_shard, o[:, first:first + count])
    _check_units(oracle, q, k, v, o, True, {8: [0, 511, 1023]})
    ws.desc.causal = 1
    _check_int32(oracle, ws, q, k, 8, 1023, kv_sample=[0, 1, 700, 2045])


def test_many_raster_groups_subprocess(cuda):
    """SAB_L2_GROUP_MB=1 (read once per process) forces many L2 groups with several query-tile
    pairs per unit: every unit and tile of the output against the oracle, in a fresh process."""
    env = dict(os.environ, SAB_L2_GROUP_MB="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "raster_check.py")], capture_output=True, text=True,
                       env=env, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout + r.stderr
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert res["groups_checked"] >= 3
    for case in res["cases"]:
        assert case["groups"] > 1 and case["npair"] > 1, case
        assert case["cos"] >= COS_MIN and case["rel_l1"] <= REL_L1_MAX, case


def test_two_rank_shards_equal_single_call(cuda):
    """bench.py's K3 sharding on the CUDA path: two torchrun ranks (both on cuda:0, gloo for the
    host collectives) each run their shard; the gathered outputs equal the one-call output."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", "--master-port", "29613", os.path.join(ROOT, "tests", "dist_shard_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "SHARDS EQUAL" in r.stdout, r.stdout + r.stderr
