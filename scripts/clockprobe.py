"""Times K2 back to back on one workload while sampling SM clock / power / throttle reasons via NVML.

    python scripts/clockprobe.py C4-128-16384-nc [iters]
"""
import ctypes as C
import os
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2410_02367_b200 import _lib, sageattn  # noqa: E402
import pynvml  # noqa: E402

wl = bench.workload(sys.argv[1])
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
b, h, n, d, causal = wl["batch"], wl["heads"], wl["tokens"], wl["head_dim"], wl["causal"]
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
q, k, v = (torch.randn((b, h, n, d), generator=g, device=dev).half() for _ in range(3))
o = torch.empty_like(q)
ws = sageattn.prepass_cuda(q, k)
ws.desc = sageattn.make_desc(q, causal, out_dtype=torch.float16)
pynvml.nvmlInit()
hd = pynvml.nvmlDeviceGetHandleByIndex(0)
samples = []
stop = threading.Event()


def run():
    while not stop.is_set():
        samples.append((pynvml.nvmlDeviceGetClockInfo(hd, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetPowerUsage(hd) / 1000.0,
                        pynvml.nvmlDeviceGetCurrentClocksEventReasons(hd)))
        time.sleep(0.005)


for _ in range(3):
    sageattn.attention_only_cuda(ws, v, o)
torch.cuda.synchronize()
t = threading.Thread(target=run)
t.start()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(iters + 1)]
ev[0].record()
for i in range(iters):
    sageattn.attention_only_cuda(ws, v, o)
    ev[i + 1].record()
torch.cuda.synchronize()
stop.set()
t.join()
ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(iters)]
ops = bench.paper_ops(b * h, n, d, causal)
print("ms per launch:", " ".join(f"{x:.3f}" for x in ms))
print("TOPS first/median/last: %.0f %.0f %.0f" % (ops / ms[0] / 1e9, ops / sorted(ms)[len(ms) // 2] / 1e9, ops / ms[-1] / 1e9))
mid = samples[len(samples) // 4: 3 * len(samples) // 4] or samples
print("clock MHz min/med/max:", min(x[0] for x in mid), sorted(x[0] for x in mid)[len(mid) // 2], max(x[0] for x in mid))
print("power W min/med/max: %.0f %.0f %.0f" % (min(x[1] for x in mid), sorted(x[1] for x in mid)[len(mid) // 2], max(x[1] for x in mid)))
print("reasons:", sorted({hex(x[2]) for x in samples}))
