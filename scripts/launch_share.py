"""Per-kernel summary of an ncu --csv launch list: launches, mean duration and share.

    python scripts/launch_share.py profiles/<launches>.csv
"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
per = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows[h + 1:]:
    if len(r) > vi:
        name = r[ki].split("(")[0].replace("void <unnamed>::", "")
        per[name][r[mi]].append(float(r[vi].replace(",", "")))
tot = sum(sum(m.get("gpu__time_duration.sum", [])) for m in per.values())
for name, m in per.items():
    t = m.get("gpu__time_duration.sum", [])
    extra = "  ".join(f"{k}={sum(v) / len(v):.4g}" for k, v in m.items() if k != "gpu__time_duration.sum")
    print(f"{name:40s} n={len(t):3d} mean={sum(t) / len(t) / 1e3:9.2f} us share={sum(t) / tot:.3f}  {extra}")
