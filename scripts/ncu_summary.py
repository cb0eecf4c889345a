"""Writes a text summary of an ncu report (key raw metrics + SASS instruction mix + top stalls).

    python scripts/ncu_summary.py <report.ncu-rep> > profiles/<name>.txt
"""
import collections
import csv
import re
import subprocess
import sys

KEYS = re.compile(r"^(gpu__time_duration.sum|sm__cycles_elapsed.avg|dram__bytes_(read|write).sum|"
                  r"dram__throughput.avg.pct_of_peak_sustained_elapsed|sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active|"
                  r"sm__pipe_tensor_subpipe_(hmma|imma)_cycles_active.avg.pct_of_peak_sustained_active|"
                  r"sm__inst_executed_pipe_(alu|fma|xu).avg.pct_of_peak_sustained_active|smsp__issue_active.avg.pct_of_peak_sustained_active|"
                  r"smsp__inst_executed.sum|launch__registers_per_thread|launch__grid_size|launch__block_size|"
                  r"launch__shared_mem_per_block_dynamic|smsp__warps_active.avg.per_cycle_active|"
                  r"smsp__average_warps_issue_stalled_\w+_per_issue_active.ratio|sm__warps_active.avg.pct_of_peak_sustained_active)$")

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
for r in rows[2:]:
    print("kernel:", r[hdr.index("Kernel Name")])
    for h, u, v in zip(hdr, units, r):
        if KEYS.match(h):
            try:
                if "stalled" in h and float(v) < 0.05:
                    continue
            except ValueError:
                pass
            print(f"  {h} = {v} {u}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout.splitlines()
blocks, cur = [], []
for line in src:
    if line.startswith('"Kernel Name"'):
        if cur:
            blocks.append(cur)
        cur = []
    else:
        cur.append(line)
if cur:
    blocks.append(cur)
for b in blocks:
    rr = list(csv.reader(b))
    if len(rr) < 2:
        continue
    h = rr[0]
    try:
        iS, iE, iW = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    except ValueError:
        continue
    ops, st, tot, tst, data = collections.Counter(), collections.Counter(), 0, 0, []
    for r in rr[1:]:
        try:
            ex, w = int(r[iE]), int(r[iW])
        except (ValueError, IndexError):
            continue
        op = re.sub(r"^@!?U?P\w+\s+", "", r[iS].strip()).split(" ")[0].split(".")[0]
        ops[op] += ex
        st[op] += w
        tot += ex
        tst += w
        data.append((w, ex, r[iS].strip()))
    print(f"  SASS mix (warp instructions executed: {tot}):")
    for op, c in ops.most_common(18):
        print(f"    {op:10s} {c:12d} {100 * c / max(tot, 1):5.1f}%   stall samples {100 * st[op] / max(tst, 1):5.1f}%")
    print("  top stalled instructions (samples, executed, sass):")
    for w, ex, s in sorted(data, reverse=True)[:10]:
        print(f"    {w:6d} {ex:10d}  {s[:90]}")
