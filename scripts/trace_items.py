"""Per-item timeline of one persistent K2 CTA (SAB_TRACE build, scripts/trace_k2.py output):
item taken, first S of tile A ready, epilogue start / end, item done -- cycles from kernel entry."""
import sys

import numpy as np

t = np.load(sys.argv[1]).reshape(-1)[:5 * 512 * 8].reshape(5, 512, 8).astype(np.int64)
e0 = t[4, 511, 0]
print("item  taken  firstS  epi_start  epi_end  done   (cycles from entry; deltas: wait-S  body  epilogue  gap-to-next)")
prev_done = None
for i in range(100):
    r = t[4, 400 + i]
    if r[0] == 0:
        break
    taken, first, es, ee, done = (r[k] - e0 if r[k] else -1 for k in (0, 1, 3, 4, 5))
    gap = taken - prev_done if prev_done is not None else 0
    print(f"{i:4d} {taken:7d} {first:7d} {es:9d} {ee:8d} {done:7d}   {first - taken:6d} {es - first:6d} {ee - es:6d} {gap:6d}")
    prev_done = done
