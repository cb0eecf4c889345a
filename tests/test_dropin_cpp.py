"""The C++ drop-in (include/sageattn/attention.hpp): an application written
against the reference API compiles, links libsageattn_b200.so, and on a B200
returns the SAGEAttn-B (and -T) output within tolerance of the reference's FP32-acc arm,
with the reference's MAC counters and exceptions."""
import os
import subprocess

import numpy as np
import pytest

from oracle.oracle import cosine_sim, relative_l1
from paper_2410_02367_b200 import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2410_02367_b200")


def _build(tmp_path):
    exe = str(tmp_path / "dropin_test")
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp"), "-o", exe, "-L", PKG, "-lsageattn_b200",
           f"-Wl,-rpath,{PKG}", f"-Wl,--no-as-needed"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_dropin_header_compiles_and_links(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
@pytest.mark.parametrize("shape,causal", [((1, 2, 1024, 64), False), ((2, 1, 300, 128), True)])
def test_dropin_runs_on_b200(tmp_path, cuda, oracle, shape, causal):
    from oracle.oracle import Reference
    try:
        reference = Reference()
    except (FileNotFoundError, OSError):
        reference = None
    exe = _build(tmp_path)
    b, h, n, d = shape
    q, k, v = synth.qkv(b * h, n, d, dtype=np.float32, dist="outlier")
    rng = np.random.default_rng(5)  # fp32 values off the fp16 grid: the drop-in quantizes fp32 exactly
    q = q + rng.standard_normal(q.shape).astype(np.float32) * 1e-3
    paths = []
    for name, a in (("q", q), ("k", k), ("v", v)):
        pth = tmp_path / f"{name}.bin"
        np.ascontiguousarray(a, np.float32).tofile(pth)
        paths.append(str(pth))
    out = tmp_path / "o.bin"
    r = subprocess.run([exe, str(b), str(h), str(n), str(d), str(int(causal)), *paths, str(out)], capture_output=True,
                       text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ERRORS OK" in r.stdout
    o = np.fromfile(out, np.float32).reshape(b * h, n, d)
    ref, macs = oracle.sage_b(q, k, v, causal, pv_fp32=True)
    assert cosine_sim(o, ref) >= 0.9999 and relative_l1(o, ref) <= 2e-3
    s, p = (int(x) for x in r.stdout.split("MACS")[1].split()[:2])
    assert (s, p) == tuple(int(x) for x in macs)
    assert "CARRIERS OK" in r.stdout
    cos = float(r.stdout.split("EXACT cos")[1].split()[0])
    flash_err = float(r.stdout.split("flash_maxerr")[1].split()[0])
    assert cos >= 0.999 and flash_err < 1e-4, (cos, flash_err)
    # Static-scale diagnostics (attention.hpp:479-488): GPU counts vs the reference's.
    el, first, later = (int(x) for x in r.stdout.split("STATIC")[1].split()[:3])
    if reference is not None:
        r_el, r_first, r_later = reference.static_scale_counts(q.reshape(shape), k.reshape(shape), v.reshape(shape),
                                                               causal)
        assert el == r_el
        assert abs(first - r_first) <= max(2, 0.01 * r_first) and abs(later - r_later) <= max(2, 0.01 * r_later)
    # honour_pv_accumulator_option(): the default options select the binary16 accumulator
    # (tests/test_gpu_pv16.py's gate), pv_fp32_accumulator=true the FP32 arm above.
    assert "PV32 SAME 1" in r.stdout
    o_16 = np.fromfile(str(out) + ".f16", np.float32).reshape(b * h, n, d)
    ref16, _ = oracle.sage_b(q, k, v, causal, pv_fp32=False)
    drift = relative_l1(ref16, ref)
    assert relative_l1(o_16, ref) <= drift and relative_l1(o_16, ref16) <= 1.5 * drift
    o_t = np.fromfile(str(out) + ".t", np.float32).reshape(b * h, n, d)
    ref_t, _ = oracle.sage(q, k, v, causal, pv_fp32=True, per_token=True)
    assert cosine_sim(o_t, ref_t) >= 0.9999 and relative_l1(o_t, ref_t) <= 2e-3
    o_vb = np.fromfile(str(out) + ".vb", np.float32).reshape(b * h, n, d)
    ref_vb, _ = oracle.sage(q, k, v, causal, pv_int8=True)
    assert cosine_sim(o_vb, ref_vb) >= 0.9999 and relative_l1(o_vb, ref_vb) <= 2e-3
    o_vt = np.fromfile(str(out) + ".vt", np.float32).reshape(b * h, n, d)
    ref_vt, _ = oracle.sage(q, k, v, causal, pv_int8=True, per_token=True)
    assert cosine_sim(o_vt, ref_vt) >= 0.9999 and relative_l1(o_vt, ref_vt) <= 2e-3
