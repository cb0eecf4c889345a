"""Markdown table of a C4 sweep from bench.py JSON lines.

    python scripts/sweep_table.py <dir> <prefix>   (files <prefix>C4-<d>-<N>-<c|nc>.json)
"""
import json
import os
import sys

d_, pre = sys.argv[1], sys.argv[2]
print("| Point | Step TOPS | K2 TOPS | K2/P_mix | K1 ms | K1 / HBM | SM clock | K2 launch | e2e TOPS |")
print("|---|---|---|---|---|---|---|---|---|")
for d in (64, 128):
    for n in (1024, 2048, 4096, 8192, 16384, 32768):
        for c in ("c", "nc"):
            name = f"C4-{d}-{n}-{c}"
            path = os.path.join(d_, f"{pre}{name}.json")
            lines = [x for x in open(path) if x.startswith("{")] if os.path.exists(path) else []
            if not lines:
                print(f"| {name} | n/a | | | | | | | |")
                continue
            j = json.loads(lines[0])
            r, k1, ck = j["roofline"], j["roofline_k1"], j["clocks"]
            cap = " cap" if "sw_power_cap" in ck["reasons"] else ""
            launch = "persistent" if "persist" in j["config"].get("k2_launch", "") else "one CTA per item"
            print(f"| {name} | {j['value']:.0f} | {r['achieved']:.0f} | {r['frac']:.2f} | {k1['ms_per_step']:.3f} | "
                  f"{k1['frac']:.2f} | {ck['sm_mhz']:.0f}{cap} | {launch} | {j['e2e']['value']:.0f} |")
