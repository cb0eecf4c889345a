"""Helper of tests/test_gpu_configs.py::test_many_raster_groups_subprocess (run with
SAB_L2_GROUP_MB=1 so K2's L2 raster splits even small shapes into many unit groups,
each with several query-tile pairs).  Compares every unit and query tile of the
as-benched output with the oracle's FP32-accumulator arm; prints one JSON line."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import torch

    from oracle.oracle import Oracle, cosine_sim, relative_l1
    from gpu_helpers import _inputs, _run_as_benched

    assert os.environ.get("SAB_L2_GROUP_MB") == "1"
    dev = torch.device("cuda:0")
    orc = Oracle()
    cases = []
    for units, n, d, causal in ((12, 2048, 128, True), (9, 1105, 64, False), (6, 700, 128, True)):
        q, k, v = _inputs(units, n, d, dev)
        o, _ = _run_as_benched(q, k, v, causal)
        qh, kh, vh = (t[0].float().cpu().numpy() for t in (q, k, v))
        ref, _ = orc.sage_b(qh, kh, vh, causal, pv_fp32=True)
        got = o[0].float().cpu().numpy()
        kv_unit = n * d * 3
        per_group = max(1, (1 << 20) // kv_unit)  # the host's raster_group_units with a 1 MB budget
        groups = -(-units // per_group)
        cases.append({"shape": [1, units, n, d], "causal": causal, "groups": groups,
                      "npair": (-(-n // 128) + 1) // 2, "cos": cosine_sim(got, ref), "rel_l1": relative_l1(got, ref)})
    print(json.dumps({"groups_checked": sum(c["groups"] for c in cases), "cases": cases}))


if __name__ == "__main__":
    main()
