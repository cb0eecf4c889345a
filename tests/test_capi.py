"""CPU: the C-ABI library loads, exports every symbol include/sageattn_b200.h
declares, and its host-side logic (validation, workspace layout, mean-tree
geometry, K3 shard plan, diagnostics) is right.  No kernel launches here."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2410_02367_b200 import _lib, sageattn

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sageattn_b200.h")


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    declared = set(re.findall(r"^\s*(?:const\s+)?\w+\**\s+\**(sab_\w+)\s*\(", open(HEADER).read(), re.M))
    assert declared == set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.sab_abi_version() == 7


def test_desc_validation_mirrors_reference():
    lib = _lib.load()
    d = _lib.desc(1, 2, 1024, 64)
    assert lib.sab_check_desc(C.byref(d)) == _lib.SAB_OK
    bad = _lib.desc(1, 2, 1024, 64, block_q=0)
    assert lib.sab_check_desc(C.byref(bad)) == _lib.SAB_ERR_SHAPE
    assert b"block sizes must be >= 1" in lib.sab_last_error()
    assert lib.sab_check_desc(C.byref(_lib.desc(1, 0, 1024, 64))) == _lib.SAB_ERR_SHAPE
    assert lib.sab_check_desc(C.byref(_lib.desc(1, 1, 1024, 96))) == _lib.SAB_ERR_UNSUPPORTED
    assert lib.sab_check_desc(C.byref(_lib.desc(1, 1, 1024, 64, block_q=64))) == _lib.SAB_ERR_UNSUPPORTED
    assert lib.sab_check_desc(C.byref(_lib.desc(1, 1, 1024, 64, pv_accum=_lib.SAB_PV_FP16))) == _lib.SAB_OK
    assert lib.sab_check_desc(C.byref(_lib.desc(1, 1, 1024, 64, pv_accum=2))) == _lib.SAB_ERR_UNSUPPORTED
    # the binary16 accumulator belongs to the FP16 P~V path (B/T), not to vB/vT
    assert lib.sab_check_desc(C.byref(_lib.desc(1, 1, 1024, 64, pv_accum=_lib.SAB_PV_FP16, pv_int8=True))) == \
        _lib.SAB_ERR_UNSUPPORTED
    # ... and never takes the KV split (one accumulator per row over all keys)
    few = _lib.desc(1, 1, 16384, 128, pv_accum=_lib.SAB_PV_FP16)
    assert _lib.workspace_layout(few).kv_chunk == 0
    assert _lib.workspace_layout(_lib.desc(1, 1, 16384, 128)).kv_chunk > 0
    assert lib.sab_check_desc(C.byref(_lib.desc(1, 1, 1024, 64, per_token=True))) == _lib.SAB_OK
    assert lib.sab_check_desc(C.byref(_lib.desc(2, 32768, 64, 64))) == _lib.SAB_OK  # host path chunks it
    bad_g = _lib.desc(1, 1, 1024, 64)
    bad_g.qk_granularity = 2  # per-tensor is not a SAGEAttn variant
    assert lib.sab_check_desc(C.byref(bad_g)) == _lib.SAB_ERR_UNSUPPORTED


def test_per_token_layout_pads_scale_rows():
    for n in (1, 63, 64, 1105):
        L = _lib.workspace_layout(_lib.desc(2, 1, n, 64, per_token=True))
        npad = -(-n // 64) * 64
        assert L.kscales - L.qscales >= 2 * npad * 4 and L.mean_k - L.kscales >= 2 * npad * 4


@pytest.mark.parametrize("n,depth", [(1, 0), (8, 0), (9, 1), (17, 1), (18, 2), (1024, 7), (8192, 10),
                                     (17776, 11), (131072, 14), (100003, 14)])
def test_mean_tree_geometry(n, depth):
    L = _lib.workspace_layout(_lib.desc(1, 1, n, 64))
    assert L.tree_depth == depth
    assert (n >> depth) < 9 and (depth == 0 or (n >> (depth - 1)) >= 9)
    assert L.n_partials * min(1 << depth, 32) == 1 << depth


def test_workspace_layout_is_disjoint_and_aligned():
    for n, d, f32 in [(8192, 128, False), (17776, 64, True), (1, 64, False)]:
        dsc = _lib.desc(2, 3, n, d, in_dtype=_lib.SAB_F32 if f32 else _lib.SAB_F16)
        L = _lib.workspace_layout(dsc)
        units = 6
        regions = [(L.qcodes, units * n * d), (L.kcodes, units * n * d), (L.qscales, units * -(-n // 128) * 4),
                   (L.kscales, units * -(-n // 64) * 4), (L.mean_k, units * d * 4),
                   (L.partials, units * L.n_partials * d * 4), (L.v16, units * n * d * 2 if f32 else 0),
                   (L.status, 4)]
        end = 0
        for off, size in regions:
            assert off % 256 == 0 and off >= end
            end = off + size
        assert L.total >= end
        size = C.c_size_t()
        assert _lib.load().sab_workspace_size(C.byref(dsc), C.byref(size)) == 0 and size.value == L.total


@pytest.mark.parametrize("units,shards", [(32, 1), (32, 8), (60, 8), (60, 7), (64, 8), (3, 8), (128, 4)])
def test_shard_plan_partitions_units(units, shards):
    seen = []
    counts = []
    for s in range(shards):
        first, count = _lib.shard_plan(units, shards, s)
        seen.extend(range(first, first + count))
        counts.append(count)
    assert seen == list(range(units))
    assert max(counts) - min(counts) <= 1


@pytest.mark.parametrize("n,causal", [(1000, True), (1000, False), (1024, True), (17776, False), (197, True)])
def test_diagnostics_match_reference_counters(oracle, n, causal):
    dsc = _lib.desc(1, 2, n, 64, causal)
    s, p = _lib.diagnostics(dsc)
    if not causal:
        assert s == p == 2 * n * n * 64
    if n <= 1024:
        from paper_2410_02367_b200 import synth

        q, k, v = synth.qkv(2, n, 64, dtype=np.float32)
        _, macs = oracle.sage_b(q, k, v, causal)
        assert (s, p) == tuple(int(x) for x in macs)
    if causal and n == 1000:  # causal counts diagonal tiles in full, 1.1255x of N^2/2
        assert s / (2 * 64 * n * n / 2) == pytest.approx(1.1255, abs=1e-3)


def test_python_mirror_validation_without_gpu():
    """Validation that precedes any device work raises like the reference."""
    q = np.zeros((1, 1, 4, 64), np.float32)
    with pytest.raises(ValueError, match="Q, K, V shapes differ"):
        sageattn.sage_attention(sageattn.AttentionInput(q, q[:, :, :2], q), sageattn.SageVariant.B)
    with pytest.raises(ValueError, match="block sizes must be >= 1"):
        sageattn.sage_attention(sageattn.AttentionInput(q, q, q), sageattn.KernelConfig(block_kv=0))
    with pytest.raises(ValueError, match="INT8 P~V"):
        sageattn.sage_attention(sageattn.AttentionInput(q, q, q), sageattn.SageVariant.VB,
                                sageattn.SageOptions(pv_dtype=sageattn.QuantDtype.FpE4M3))
    assert sageattn.kernel_config_for(sageattn.SageVariant.B) == sageattn.KernelConfig()
    assert sageattn.apply_causal_tiling(0, 2, 128, 64, 1000) == sageattn.TileKind.Skip


def test_product_path_does_not_touch_oracle():
    """The shipped package never imports, links or loads the CPU checkers."""
    pkg = os.path.join(ROOT, "paper_2410_02367_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                for needle in ("import oracle", "from oracle", "liboracle", "libsageref", "sage_oracle"):
                    assert needle not in src, (f, needle)
