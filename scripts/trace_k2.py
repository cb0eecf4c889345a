"""Runs one K2 launch with the SAB_TRACE build and dumps one CTA's clock64 timeline.

    python scripts/trace_k2.py <workload> <cta> <out.npy> [units]   (libsageattn_b200.so must be a SAB_TRACE build)
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2410_02367_b200 import _lib, sageattn  # noqa: E402

wl = bench.workload(sys.argv[1])
cta = int(sys.argv[2])
b, h, n, d, causal = wl["batch"], wl["heads"], wl["tokens"], wl["head_dim"], wl["causal"]
if len(sys.argv) > 4:  # optional unit count (a K3 shard), as (1, units)
    b, h = 1, int(sys.argv[4])
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
q, k, v = (torch.randn((b, h, n, d), generator=g, device=dev).half() for _ in range(3))
o = torch.empty_like(q)
ws = sageattn.prepass_cuda(q, k)
desc = sageattn.make_desc(q, causal, out_dtype=torch.float16)
ws.desc = desc
trace = torch.zeros(19 * 256 * 8, dtype=torch.int64, device=dev)
lib = _lib.load()
lib.sab_debug_set_trace.argtypes = [C.c_void_p, C.c_int]
for it in range(3):
    lib.sab_debug_set_trace(trace.data_ptr(), cta)
    trace.zero_()
    sageattn.attention_only_cuda(ws, v, o)
    torch.cuda.synchronize()
np.save(sys.argv[3], trace.cpu().numpy().reshape(19, 256, 8))
print("trace saved", sys.argv[3])
