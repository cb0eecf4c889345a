"""Helper of tests/test_gpu_split.py::test_forced_kv_split_subprocess, run with SAB_KV_SPLIT=<tiles>
(read once per process) so that every (unit, query-tile pair) of small shapes is cut into
KV chunks merged by the pair's last chunk CTA.  Compares whole outputs of the B, T, vB and
vT paths with the oracle (attention.hpp:383-541; the reference's q-block independence makes
the chunked reduction an exact restatement up to summation order); prints one JSON line."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import numpy as np
    import torch

    from oracle.oracle import Oracle, cosine_sim, relative_l1
    from paper_2410_02367_b200 import _lib, sage_attention_cuda, sageattn

    chunk = int(os.environ["SAB_KV_SPLIT"])
    dev = torch.device("cuda:0")
    orc = Oracle()
    rng = np.random.default_rng(11)
    cases = []
    for (b, h, n, d), causal, per_token, pv_int8 in (
            ((1, 3, 2048, 128), True, False, False),
            ((2, 2, 1500, 64), False, False, False),
            ((1, 2, 1105, 128), True, True, False),
            ((1, 2, 1300, 64), True, False, True),
            ((1, 2, 900, 128), False, True, True),
            ((1, 3, 777, 64), True, False, False)):
        q, k, v = (rng.standard_normal((b, h, n, d)).astype(np.float16) for _ in range(3))
        desc = sageattn.make_desc(torch.empty((b, h, n, d), dtype=torch.float16, device=dev), causal)
        desc.qk_granularity = _lib.SAB_QK_PER_TOKEN if per_token else _lib.SAB_QK_PER_BLOCK
        desc.pv_path = _lib.SAB_PV_PATH_INT8 if pv_int8 else _lib.SAB_PV_PATH_FP16
        lay = _lib.SabWsLayout()
        _lib.check(_lib.load().sab_workspace_layout(C_byref(desc), C_byref(lay)))
        qd, kd, vd = (torch.from_numpy(x).to(dev) for x in (q, k, v))
        o = sage_attention_cuda(qd, kd, vd, causal=causal, out_dtype=torch.float32, per_token=per_token,
                                pv_int8=pv_int8)
        got = o.cpu().numpy().reshape(-1, n, d)
        f32 = [x.reshape(-1, n, d).astype(np.float32) for x in (q, k, v)]
        if pv_int8:
            ref, _ = orc.sage(*f32, causal, pv_int8=True, per_token=per_token)
        else:
            ref, _ = orc.sage(*f32, causal, pv_fp32=True, per_token=per_token)
        cases.append({"shape": [b, h, n, d], "causal": causal, "per_token": per_token, "pv_int8": pv_int8,
                      "kv_chunk": lay.kv_chunk, "nchunk": lay.kv_nchunk,
                      "cos": cosine_sim(got, ref), "rel_l1": relative_l1(got, ref)})
    print(json.dumps({"chunk": chunk, "cases": cases}))


def C_byref(x):
    import ctypes

    return ctypes.byref(x)


if __name__ == "__main__":
    main()
