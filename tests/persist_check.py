"""Helper of tests/test_gpu_persist.py: runs K1 + K2 on fixed seeded shapes under the process's
SAB_K2_PERSIST setting (read once per process) and saves every output to one .npz."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CASES = [((1, 6, 1024, 128), True, False, False), ((2, 5, 700, 64), False, False, False),
         ((1, 4, 2048, 128), False, True, False), ((1, 3, 1500, 64), True, False, True),
         ((1, 4, 8192, 128), True, False, False)]  # the last one splits (few units, long causal rows)


def main(out):
    import numpy as np
    import torch

    from paper_2410_02367_b200 import sage_attention_cuda

    dev = torch.device("cuda:0")
    res = {}
    for i, (shape, causal, per_token, pv_int8) in enumerate(CASES):
        g = torch.Generator(device=dev).manual_seed(100 + i)
        q, k, v = (torch.randn(shape, generator=g, device=dev).half() for _ in range(3))
        o = sage_attention_cuda(q, k, v, causal=causal, out_dtype=torch.float32, per_token=per_token,
                                pv_int8=pv_int8)
        res[f"case{i}"] = o.cpu().numpy()
    np.savez(out, **res)
    print("saved", out)


if __name__ == "__main__":
    main(sys.argv[1])
