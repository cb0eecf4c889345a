"""bench.py's JSON contract on CPU: the reference arm (the reference's own CPU code,
oracle/_ref) prints one well-formed line; GPU arms are exercised on the B200 box."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libsageref.so")),
                    reason="reference library not built")
def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", "C1",
                        "--steps", "1", "--warmup", "0", "--cpu-threads", "2"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "TOPS" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["steps"] == 1 and d["warmup"] == 0
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] == 2 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": "TOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("C1")


def test_paper_ops_and_workloads():
    sys.path.insert(0, ROOT)
    import bench

    assert bench.paper_ops(32, 8192, 128, True) == pytest.approx(5.4976e11, rel=1e-4)  # C2
    assert bench.paper_ops(60, 17776, 64, False) == pytest.approx(4.854e12, rel=1e-3)  # C3
    w = bench.workload("C4-128-16384-nc")
    assert (w["batch"], w["heads"], w["tokens"], w["head_dim"], w["causal"]) == (4, 32, 16384, 128, False)
    assert bench.workload("C5")["tokens"] == 131072


def test_overlap_groups():
    sys.path.insert(0, ROOT)
    import bench

    assert bench.overlap_groups("auto", 32, 8192, 128) == [32]  # measured: one launch each is fastest
    assert bench.overlap_groups("off", 60, 17776, 64) == [60]
    assert bench.overlap_groups("8", 32, 8192, 128) == [8, 24]
    assert bench.overlap_groups("4,8,20", 32, 8192, 128) == [4, 8, 20]
    assert bench.overlap_groups("8,24", 1, 8192, 128) == [1]
    with pytest.raises(SystemExit):
        bench.overlap_groups("8,8", 32, 8192, 128)
