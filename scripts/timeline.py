"""Device timeline of bench.py's step (K1 + K2) for one workload, from the torch profiler
(CUPTI): per-op start/duration and the gaps between them, averaged over steps.

    python scripts/timeline.py <workload> [--shard-of N] [--steps K]
"""
import argparse
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2410_02367_b200 import _lib, sageattn  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload")
ap.add_argument("--shard-of", type=int, default=1)
ap.add_argument("--steps", type=int, default=5)
a = ap.parse_args()
wl = bench.workload(a.workload)
units = wl["batch"] * wl["heads"]
first, count = _lib.shard_plan(units, a.shard_of, 0)
n, d, causal = wl["tokens"], wl["head_dim"], wl["causal"]
dev = torch.device("cuda:0")
q, k, v = bench.device_inputs(count, n, d, first, dev)
o = torch.empty_like(q)
desc = sageattn.make_desc(q, causal, out_dtype=torch.float16)
ws = sageattn.Workspace(desc, dev)
lib = _lib.load()
sp = torch.cuda.current_stream(dev).cuda_stream


def step():
    _lib.check(lib.sab_prepass(ctypes.byref(desc), q.data_ptr(), k.data_ptr(), None, ws.ptr, ws.nbytes, sp))
    _lib.check(lib.sab_attention(ctypes.byref(desc), ws.ptr, ws.nbytes, v.data_ptr(), o.data_ptr(), sp))


for _ in range(5):
    step()
torch.cuda.synchronize()
marker = torch.empty(1, device=dev)
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(a.steps):
        marker.fill_(0)
        step()
    torch.cuda.synchronize()
path = "/tmp/trace.json"
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") in ("kernel", "gpu_memset", "gpu_memcpy")]
ev.sort(key=lambda e: e["ts"])
rows = []
prev_end = None
for e in ev:
    gap = None if prev_end is None else e["ts"] - prev_end
    rows.append((e["name"][:60], e["dur"], gap))
    prev_end = e["ts"] + e["dur"]
for r in rows[-12:]:
    print(f"{r[0]:60s} dur {r[1]:8.2f} us  gap-before {r[2] if r[2] is None else round(r[2], 2)}")
