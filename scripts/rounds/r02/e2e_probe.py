"""Host-buffer path (sab_attention_fwd_host) throughput on pinned fp16 buffers, plus the raw
pinned H2D / D2H copy rates of this box for the same byte counts (the e2e ceiling)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2410_02367_b200 import sageattn  # noqa: E402

WL = {"C4-128-16384-nc": (4, 32, 16384, 128, False), "C2": (1, 32, 8192, 128, True),
      "C3": (2, 30, 17776, 64, False), "C4-128-1024-c": (4, 32, 1024, 128, True)}
name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
b, h, n, d, causal = WL[name]
ops = 4.0 * b * h * n * n * d * (0.5 if causal else 1.0)
g = torch.Generator().manual_seed(0)
host = [torch.randn((b, h, n, d), generator=g).half().pin_memory() for _ in range(3)]
hq, hk, hv = (t.numpy() for t in host)
ho_t = torch.empty((b, h, n, d), dtype=torch.float16).pin_memory()
ho = ho_t.numpy()
sageattn.attention_fwd_host(hq, hk, hv, causal, ho, devices=[0])
ts = []
for _ in range(reps):
    t0 = time.perf_counter()
    sageattn.attention_fwd_host(hq, hk, hv, causal, ho, devices=[0])
    ts.append(time.perf_counter() - t0)
t = min(ts)
# raw copies: H2D of Q,K,V and D2H of O, alone and concurrently
dev = [torch.empty_like(x, device="cuda") for x in host]
do = torch.empty_like(ho_t, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def h2d():
    with torch.cuda.stream(s1):
        for x, y in zip(dev, host):
            x.copy_(y, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2):
        ho_t.copy_(do, non_blocking=True)
for f in (h2d, d2h):
    f()
torch.cuda.synchronize()
def timed(fs):
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for f in fs:
            f()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best
bi = sum(x.numel() * 2 for x in host)
bo = ho_t.numel() * 2
th, td, tb = timed([h2d]), timed([d2h]), timed([h2d, d2h])
print(f"{name}: e2e {ops / t / 1e12:.1f} TOPS ({t * 1e3:.2f} ms, all {[round(x * 1e3, 2) for x in ts]}); "
      f"H2D {bi / th / 1e9:.1f} GB/s ({th * 1e3:.2f} ms), D2H {bo / td / 1e9:.1f} GB/s, both {tb * 1e3:.2f} ms "
      f"-> copy-bound e2e {ops / tb / 1e12:.1f} TOPS")
