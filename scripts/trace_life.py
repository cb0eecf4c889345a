"""CTA lifecycle from a SAB_TRACE timeline (.npy of scripts/trace_k2.py): entry, prologue done,
griddep_wait released, first S of tile A, epilogue start / end, teardown -- cycles from entry."""
import sys

import numpy as np

t = np.load(sys.argv[1]).reshape(-1)[:5 * 512 * 8].reshape(5, 512, 8).astype(np.int64)
life = t[4, 511]
e0 = life[0]
nk = int((t[0, :511, 1] > 0).sum())
first_s = t[0, 0, 1]
last_s = t[0, nk - 1, 2] if nk else 0
names = ["entry", "prologue (bias smem, barriers, TMEM alloc)", "griddep_wait released", "epilogue start (O final)",
         "epilogue stores done", "before teardown", "TMEM dealloc done"]
for i, nm in enumerate(names):
    print(f"{nm:45s} {life[i] - e0 if life[i] else -1:>9d}")
print(f"{'first S of tile A ready':45s} {first_s - e0 if first_s else -1:>9d}")
print(f"{'last softmax of tile A done':45s} {last_s - e0 if last_s else -1:>9d}   ({nk} KV tiles)")
if nk > 2:
    per = np.diff(t[0, :nk, 1])
    print(f"{'softmax period (median, cycles/tile)':45s} {int(np.median(per)):>9d}")
