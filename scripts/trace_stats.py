"""Summarises a SAB_TRACE timeline (.npy from scripts/trace_k2.py): per-step phase durations."""
import sys

import numpy as np

t = np.load(sys.argv[1]).reshape(-1)[:5 * 512 * 8].reshape(5, 512, 8).astype(np.int64)
base = t[4, 0, 0]
nk = int((t[0, :, 1] > 0).sum())
lo, hi = 10, nk - 10
d = lambda r, a, b: (t[r, lo:hi, b] - t[r, lo:hi, a]).mean()
for r, name in ((0, "softmax A"), (1, "softmax B")):
    print(f"{name}: period {np.diff(t[r, :nk, 1])[lo:hi].mean():.0f}  wait_s {d(r,0,1):.0f}  softmax {d(r,1,2):.0f}  "
          f"st+rescale {d(r,2,3):.0f}  fence+arrive {d(r,3,4):.0f} | ld {d(r,1,5):.0f} max {d(r,5,6):.0f} exp {d(r,6,7):.0f} "
          f"st {d(r,7,2):.0f}")
for r, name in ((2, "mma A"), (3, "mma B")):
    print(f"{name}: ev0->1 {d(r,0,1):.0f}  ev1->2 {d(r,1,2):.0f}  pwait {d(r,3,4):.0f}  pv_issue {d(r,4,5):.0f}")
print("A/B softmax start offset", (t[1, lo:hi, 1] - t[0, lo:hi, 1]).mean())
if len(sys.argv) > 2:
    for j in range(100, 104):
        print(j, {n: (t[r, j] - base)[:6].tolist() for r, n in enumerate(("A", "B", "mA", "mB", "prod"))})
