"""Builds libsageattn_b200.so in-tree for sm_100a (nvcc, no torch involvement).

    python -m paper_2410_02367_b200.build [--verbose]
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SOURCES = ["sab_prepass.cu", "sab_attention.cu", "sab_capi.cu"]
OUT = os.path.join(HERE, "libsageattn_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
         "-shared", "--expt-relaxed-constexpr"]


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(HERE, "..", "include", "sageattn_b200.h")]
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


ROOT = os.path.dirname(HERE)
BENCH = os.path.join(ROOT, "bench_support")


def _older(out: str, deps) -> bool:
    return not os.path.exists(out) or any(os.path.getmtime(p) > os.path.getmtime(out) for p in deps if os.path.exists(p))


def build_bench_support(force: bool = False) -> None:
    """bench.py's measurement helpers (not part of the library): the tcgen05 peak probe and the
    C++ drop-in timing shim (compiled against include/sageattn/attention.hpp)."""
    peak, peak_src = os.path.join(BENCH, "libsab_peak.so"), os.path.join(BENCH, "sab_peak.cu")
    if force or _older(peak, [peak_src, os.path.join(CSRC, "sab_ptx.cuh")]):
        subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-Xcompiler", "-fPIC",
                        "-shared", "-o", peak, peak_src], check=True)
    dropin, dropin_src = os.path.join(BENCH, "libdropin_bench.so"), os.path.join(BENCH, "dropin_bench.cpp")
    inc = os.path.join(ROOT, "include")
    deps = [dropin_src, OUT] + [os.path.join(inc, "sageattn", f) for f in os.listdir(os.path.join(inc, "sageattn"))]
    if force or _older(dropin, deps):
        subprocess.run(["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-I", inc, dropin_src, "-o", dropin, "-L", HERE,
                        "-lsageattn_b200", "-Wl,-rpath,$ORIGIN/../paper_2410_02367_b200"], check=True)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or _stale():
        cmd = [NVCC, *FLAGS, *(["-Xptxas", "-v"] if verbose else []), "-o", OUT + ".tmp",
               *[os.path.join(CSRC, s) for s in SOURCES]]
        subprocess.run(cmd, check=True)
        os.replace(OUT + ".tmp", OUT)
    build_bench_support(force)
    return OUT


if __name__ == "__main__":
    print(build(force=True, verbose="--verbose" in sys.argv))
