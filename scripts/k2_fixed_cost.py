"""K2 time vs KV tiles per CTA at one wave of ~148 CTAs (non-causal, d=128): the intercept
is K2's fixed per-CTA cost (launch, prologue, first-tile latency, epilogue, teardown)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_02367_b200 import sageattn  # noqa: E402

dev = torch.device("cuda:0")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
rows = []
for n, units, d in ((256, 148, 128), (512, 74, 128), (1024, 37, 128), (2048, 18, 128), (4096, 9, 128),
                    (8192, 4, 128), (256, 148, 64), (1024, 37, 64), (4096, 9, 64)):
    g = torch.Generator(device=dev).manual_seed(0)
    q, k, v = (torch.randn((1, units, n, d), generator=g, device=dev).half() for _ in range(3))
    o = torch.empty_like(q)
    ws = sageattn.prepass_cuda(q, k)
    ws.desc = sageattn.make_desc(q, False, out_dtype=torch.float16)
    for _ in range(3):
        sageattn.attention_only_cuda(ws, v, o)
    ts = []
    for _ in range(20):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        sageattn.attention_only_cuda(ws, v, o)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    ctas = units * ((n + 255) // 256)
    rows.append({"n": n, "units": units, "d": d, "ctas": ctas, "tiles_per_cta": n // 64, "k2_us": ts[len(ts) // 2]})
    print(json.dumps(rows[-1]))
