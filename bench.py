#!/usr/bin/env python
"""SageAttn-B forward throughput on B200 (paper OPS = 4*B*H*N^2*d / t, halved for causal).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C4-128-16384-nc] [--impl ours|reference]

One step = the whole hot path on one batch of synthetic fp16 inputs already
resident in HBM: K1 (smooth-K + INT8 quantization, 2 launches) + K2 (tcgen05
attention, 1 launch).  Under torchrun (N>1) the B*H units are head-sharded
over the ranks (K3, no collective on the data path); time = max over ranks.

Default workload = the north-star point of BASELINE.json configs[3]: the C4
kernel-bench sweep at head_dim 128, non-causal, N=16K (B=4, H=32), where the
>= 50 % dense-INT8 target is stated.  `secondary` adds a short C2 (Llama-2-7B
prefill, configs[1]) device-time line.  Other workloads: --workload C1|C2|C3|C5|
C4-<d>-<N>-<c|nc>.  Scaling defaults to strong (the fixed workload head-sharded
over N GPUs, as the north star asks); --scaling weak grows the batch with N.

Keys beyond the driver contract:
  e2e          same metric through the C-ABI host-buffer call (sab_attention_fwd_host)
               with pinned host fp16 inputs; H2D of Q/K/V and D2H of O inside the timed region
  e2e_dropin   same metric through the C++ drop-in sageattn::sage_attention(in, SageVariant::B)
               on fp32 Tensor4f in pageable memory, fp32 O returned (N=1 only)
  roofline     K2 (dominant kernel): paper-OPS / K2 time vs the mixed INT8+FP16 tensor peak
               (MEASURED_PEAKS.json), plus the same fraction at K2's sampled clock against
               the tcgen05 M=128 N=256 rates measured in this run (bench_support/sab_peak.cu)
  roofline_k1  K1: algorithmic bytes / K1 time vs measured HBM copy bandwidth
  cpu_baseline the reference's own CPU code (oracle/_ref) on a bounded, work-balanced sample
               of query tiles, rank 0 at N=1 only
  parity       the timed step's own fp16 O on those sampled tiles against the reference's
               FP32-accumulator arm (gated: cos >= 0.9999, rel-L1 <= 2e-3), its default
               FP16-accumulator arm and exact binary64 attention (reported)
"""
from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    "C1": dict(batch=1, heads=2, tokens=1024, head_dim=64, causal=False, name="C1 oracle case (1,2,1024,64) non-causal"),
    "C2": dict(batch=1, heads=32, tokens=8192, head_dim=128, causal=True,
               name="C2 Llama-2-7B prefill attention (1,32,8192,128) causal"),
    "C3": dict(batch=2, heads=30, tokens=17776, head_dim=64, causal=False,
               name="C3 CogVideoX-2B attention (2,30,17776,64) non-causal"),
    "C5": dict(batch=1, heads=64, tokens=131072, head_dim=128, causal=True,
               name="C5 long-context prefill (1,64,131072,128) causal"),
}
DEFAULT_WORKLOAD = "C4-128-16384-nc"
METRIC = "attention TOPS (4*B*H*N^2*d/s, halved for causal), SageAttn-B forward (K1 prepass + K2 attention)"
UNIT = "TOPS"
L2_BYTES = 126 * 1024 * 1024
COS_MIN, REL_L1_MAX = 0.9999, 2e-3  # north-star tolerance vs the reference's quantized path


def workload(name: str):
    if name in WORKLOADS:
        return dict(WORKLOADS[name])
    if name.startswith("C4-"):  # C4-<d>-<N>-<c|nc>
        _, d, n, c = name.split("-")
        return dict(batch=4, heads=32, tokens=int(n), head_dim=int(d), causal=(c == "c"),
                    name=f"C4 kernel-bench point (4,32,{n},{d}) {'causal' if c == 'c' else 'non-causal'}")
    raise SystemExit(f"unknown workload {name}")


def paper_ops(units: int, n: int, d: int, causal: bool) -> float:
    ops = 4.0 * units * n * n * d
    return ops / 2 if causal else ops


def measured_peaks():
    """MEASURED_PEAKS.json (driver-written) or the profiling guide's fallback, key by key."""
    fallback = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
    except (OSError, ValueError):
        return fallback, "fallback"
    out = {k: float(p[k]) if isinstance(p.get(k), (int, float)) else v for k, v in fallback.items()}
    return out, "measured" if all(isinstance(p.get(k), (int, float)) for k in fallback) else "measured/fallback"


def p_mix(p_i8: float, p_f16: float) -> float:
    """Mixed roofline of paper-OPS: half the ops are INT8 QK^T, half FP16 PV."""
    return 4.0 / (2.0 / p_i8 + 2.0 / p_f16)


def tensor_peak_probe():
    """tcgen05 M=128 N=256 dense rates measured on this GPU (ops / clk / SM), or None."""
    path = os.path.join(ROOT, "bench_support", "libsab_peak.so")
    if not os.path.exists(path):
        return None
    lib = ctypes.CDLL(path)
    lib.sab_peak_probe.argtypes = [ctypes.c_int, ctypes.c_int] + [ctypes.POINTER(ctypes.c_double)] * 3
    out = {}
    for kind, name in ((0, "i8"), (1, "f16")):
        per_clk, per_s, mhz = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        if lib.sab_peak_probe(kind, 20000, ctypes.byref(per_clk), ctypes.byref(per_s), ctypes.byref(mhz)) != 0:
            return None
        out[name] = {"ops_per_clk_per_sm": per_clk.value, "tops": per_s.value / 1e12, "probe_mhz": mhz.value}
    return out


class ClockSampler:
    """NVML sampler (every 2 ms) of SM clock, power and throttle reasons during the timed region."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap",
               0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int):
        self.samples, self.power, self.reasons, self.max_mhz, self.limit_w = [], [], set(), None, None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            try:
                self.limit_w = pynvml.nvmlDeviceGetEnforcedPowerLimit(self.h) / 1000.0
            except Exception:  # noqa: BLE001
                self.limit_w = None
        except Exception:  # noqa: BLE001 - clocks are reported as unavailable
            self.nv = None
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                mhz = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append(mhz)
                self.power.append(self.nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv:
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.nv:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "sm_min_mhz": min(self.samples) if self.samples else None,
                "reasons": sorted(self.reasons), "samples": len(self.samples),
                "power_w_median": statistics.median(self.power) if self.power else None,
                "power_limit_w": self.limit_w}


# ----------------------------------------------------------------------------- CPU reference sample

def tile_ops(n: int, d: int, causal: bool, tiles):
    """Paper-OPS of query tiles: 4*d per (query, attended key) pair."""
    total = 0
    for t in tiles:
        r0, r1 = t * 128, min(n, t * 128 + 128)
        keys = sum(r + 1 for r in range(r0, r1)) if causal else (r1 - r0) * n
        total += 4 * keys * d
    return float(total)


def balanced_tile_lists(n: int, d: int, causal: bool, threads: int, target_s: float):
    """Query tiles of one unit for `threads` threads with equal work per thread.

    Causal tile i costs ~(i + 1) key tiles, so each thread takes pairs (i, ntq - 1 - i)
    (equal cost per pair); non-causal tiles all cost the same.  The per-thread count is
    sized for ~target_s of work at ~0.3 GOPS per core, at least one item each,
    and the chosen items are spread over the unit (first, middle and last tiles appear)."""
    ntq = -(-n // 128)
    if causal and ntq > 1:
        items = [(i, ntq - 1 - i) for i in range(ntq // 2)]
    else:
        items = [(i,) for i in range(ntq)]
    cost = max(tile_ops(n, d, causal, items[0]) / 0.3e9, 1e-3)
    per_thread = max(1, min(len(items) // threads or 1, int(target_s / cost)))
    k = min(len(items), per_thread * threads)
    chosen = sorted({int(round(i * (len(items) - 1) / max(1, k - 1))) for i in range(k)}) if k > 1 else [0]
    picked = [items[i] for i in chosen]
    lists = [[t for it in picked[i::threads] for t in it] for i in range(threads)]
    return [sorted(x) for x in lists if x]


def cpu_reference_sample(wl, threads: int, target_s: float = 12.0, q=None, k=None, v=None):
    """Runs the reference's own CPU code (oracle/_ref, kind "reference") on work-balanced query
    tiles of unit 0, one host thread per tile list.

    Returns dict(value TOPS, seconds, sample, cores, kind, tiles, outputs (N,d) with the
    sampled rows filled)."""
    import numpy as np

    from paper_2410_02367_b200 import synth

    n, d, causal = wl["tokens"], wl["head_dim"], wl["causal"]
    if q is None:
        q, k, v = (x[0] for x in synth.qkv(1, n, d, dtype=np.float32))
    kind = "reference"
    try:
        from oracle.oracle import Reference

        ref = Reference()
    except (FileNotFoundError, OSError):
        ref, kind = None, "port"
    lists = balanced_tile_lists(n, d, causal, threads, target_s)
    tiles_all = sorted(t for tl in lists for t in tl)
    t0 = time.perf_counter()
    if ref is not None:
        outs = ref.sage_b_tiles_parallel(q, k, v, lists, causal)
    else:
        from oracle.oracle import Oracle

        orc = Oracle()
        pre = orc.prepass(q[None], k[None])
        outs = [None] * len(lists)

        def work(i):
            outs[i] = orc.sage_b_tiles(pre, v[None], 0, lists[i], causal, False)

        ths = [threading.Thread(target=work, args=(i,)) for i in range(len(lists))]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
    dt = time.perf_counter() - t0
    out = np.zeros((n, d), np.float32)
    for tl, o in zip(lists, outs):
        for t in tl:
            out[t * 128:min(n, t * 128 + 128)] = o[t * 128:min(n, t * 128 + 128)]
    ops = tile_ops(n, d, causal, tiles_all)
    desc = (f"{len(tiles_all)} of {-(-n // 128)} query tiles (128 rows each) of unit 0 of {wl['name']}, "
            f"equal work per thread{' (causal tile pairs i, last-i)' if causal else ''}, SageAttn-B default "
            f"FP16-accumulator arm, {len(lists)} host threads, {ops:.3e} paper-OPS")
    return dict(value=ops / dt / 1e12, seconds=dt, sample=desc, cores=len(lists), kind=kind, tiles=tiles_all,
                outputs=out, lists=lists)


def parity_report(wl, q, k, v, o_gpu, sample, threads: int):
    """The timed step's own O (unit 0) on the sampled tiles against the reference's arms.

    fp16_default_arm: the reference outputs the cpu_baseline leg just timed (SageOptions{});
    fp32_acc_arm:     the oracle's FP32-accumulator arm (bit-identical to the reference's
                      pv_fp32_accumulator, tests/test_oracle.py) -- the gated comparison;
    exact:            binary64 naive attention (attention.hpp:107-149).
    The last two run on up to 3 tiles (first / middle / last of the sample), one thread each."""
    import numpy as np

    from oracle.oracle import Oracle, cosine_sim, relative_l1

    n, d, causal = wl["tokens"], wl["head_dim"], wl["causal"]
    tiles = sample["tiles"]
    sub = sorted({tiles[0], tiles[len(tiles) // 2], tiles[-1]})
    rows_all = np.concatenate([np.arange(t * 128, min(n, t * 128 + 128)) for t in tiles])
    rows_sub = np.concatenate([np.arange(t * 128, min(n, t * 128 + 128)) for t in sub])
    orc = Oracle()
    pre = orc.prepass(q[None], k[None])
    f32 = [None] * len(sub)
    exact = [None] * len(sub)

    def work(i):
        t = sub[i]
        f32[i] = orc.sage_b_tiles(pre, v[None], 0, [t], causal, pv_fp32=True)[t * 128:min(n, t * 128 + 128)]
        exact[i] = orc.naive_rows(q, k, v, causal, t * 128, min(n, t * 128 + 128))

    ths = [threading.Thread(target=work, args=(i,)) for i in range(len(sub))]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    ref32, ex = np.concatenate(f32), np.concatenate(exact)
    og = o_gpu.astype(np.float32)
    cs32, rl32 = cosine_sim(og[rows_sub], ref32), relative_l1(og[rows_sub], ref32)
    out = {
        "unit": 0, "tiles_vs_default_arm": len(tiles), "tiles_vs_fp32_arm_and_exact": sub,
        "o_dtype": "fp16 (the timed step's output)",
        "fp32_acc_arm": {"cos": cs32, "rel_l1": rl32, "gate": f"cos >= {COS_MIN}, rel_l1 <= {REL_L1_MAX}",
                         "pass": bool(cs32 >= COS_MIN and rl32 <= REL_L1_MAX)},
        "fp16_default_arm": {"cos": cosine_sim(og[rows_all], sample["outputs"][rows_all]),
                             "rel_l1": relative_l1(og[rows_all], sample["outputs"][rows_all])},
        "exact": {"cos": cosine_sim(og[rows_sub], ex), "rel_l1": relative_l1(og[rows_sub], ex)},
        "reference_fp16_arm_vs_exact": {"cos": cosine_sim(sample["outputs"][rows_sub], ex),
                                        "rel_l1": relative_l1(sample["outputs"][rows_sub], ex)},
    }
    return out


def overlap_groups(spec: str, count: int, n: int, d: int) -> list:
    """Unit-group sizes of the overlapped step ('off' -> one group)."""
    if spec == "off" or count < 2:
        return [count]
    if spec == "auto":
        # Measured slower than one launch each on C2 and C3 (profiles/r01_experiments.md:
        # K2's 576-thread CTAs leave no room for K1 CTAs until its last wave drains).
        return [count]
    sizes = [int(x) for x in spec.split(",") if x]
    if len(sizes) == 1:
        sizes.append(count - sizes[0])
    if sum(sizes) != count or min(sizes) < 1:
        raise SystemExit(f"--groups {spec}: sizes must be positive and sum to the shard's {count} units")
    return sizes


def dropin_e2e(hq, hk, hv, wl, batch, iters: int):
    """e2e through the C++ drop-in (bench_support/libdropin_bench.so over include/sageattn/attention.hpp)."""
    import numpy as np

    path = os.path.join(ROOT, "bench_support", "libdropin_bench.so")
    if not os.path.exists(path):
        return None
    lib = ctypes.CDLL(path)
    fp = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
    lib.sab_dropin_bench.argtypes = [fp, fp, fp] + [ctypes.c_int] * 6 + [ctypes.POINTER(ctypes.c_double),
                                                                         ctypes.c_void_p]
    q32, k32, v32 = (np.ascontiguousarray(x, dtype=np.float32) for x in (hq, hk, hv))
    sec = ctypes.c_double()
    # The host arrays hold this rank's (or --shard-of's) units: (1, count, n, d), not the workload's (B, H).
    b, h, n, d = q32.shape
    assert (n, d) == (wl["tokens"], wl["head_dim"])
    st = lib.sab_dropin_bench(q32, k32, v32, b, h, n, d, int(wl["causal"]), iters, ctypes.byref(sec), None)
    if st != 0:
        return {"error": "sab_dropin_bench failed"}
    nbytes = q32.nbytes
    return {"seconds_per_call": sec.value, "h2d_bytes_per_step": 3 * nbytes, "d2h_bytes_per_step": nbytes,
            "how": "sageattn::sage_attention(in, SageVariant::B) from include/sageattn/attention.hpp on fp32 "
                   "Tensor4f in pageable std::vector memory (pinned-chunk staging inside the call), fp32 O "
                   "returned by value; wall clock, warm context pool"}


def device_inputs(count, n, d, first, dev):
    """This rank's shard of the synthetic Q/K/V (seeds 1/2/3), generated on the device."""
    import torch

    from paper_2410_02367_b200 import synth

    return [synth.tensor_torch(s, (count, n, d), first, device=dev).reshape(1, count, n, d) for s in (1, 2, 3)]


def time_steps(step, stream, flush, steps):
    import torch

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    for i in range(steps):
        flush.fill_(2)  # evict the previous step's data from L2 (outside the timed events)
        ev = evs[i]
        ev[0].record(stream)
        step(ev)
        ev[2].record(stream)
    torch.cuda.synchronize()
    return evs


# ----------------------------------------------------------------------------- main

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD)
    ap.add_argument("--pv-accum", default="fp32", choices=["fp32", "fp16"],
                    help="B/T P~V accumulator: fp32 (default, the parity-gated arm) or the binary16 arm")
    ap.add_argument("--variant", default="B", choices=["B", "T", "VB", "VT"],
                    help="B: SAGEAttn-B (per-block Q/K scales, the north-star path); T: SAGEAttn-T (per-token)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--groups", default="auto",
                    help="K1/K2 overlap: comma list of unit-group sizes (e.g. '8,24'), 'auto', or 'off'. "
                         "Group g's K2 runs on its own stream while group g+1's K1 runs")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-dropin", action="store_true")
    ap.add_argument("--cpu-threads", type=int, default=None)
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="strong (default): the workload as given, head x batch sharded over the ranks; "
                         "weak: N ranks run N x the workload's batch (fixed units per GPU)")
    ap.add_argument("--shard-of", type=int, default=None,
                    help="1-GPU strong-scaling probe: time rank 0's K3 shard of an N-GPU run of the workload "
                         "(e.g. --workload C2 --shard-of 8 = the 4 units one GPU holds at 8 GPUs)")
    args = ap.parse_args()
    wl = workload(args.workload)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    batch = wl["batch"] * (world if args.scaling == "weak" else 1)
    units_total = batch * wl["heads"]
    n, d, causal = wl["tokens"], wl["head_dim"], wl["causal"]
    total_ops = paper_ops(units_total, n, d, causal)
    per_token = args.variant in ("T", "VT")
    pv_int8 = args.variant in ("VB", "VT")
    config = {"workload": wl["name"], "variant": f"SAGEAttn-{args.variant}", "batch": batch, "heads": wl["heads"],
              "tokens": n, "head_dim": d, "causal": causal, "global_batch": batch,
              "parallelism": (f"head x batch shard over {world} GPUs, no collective" if world > 1 else "single GPU"),
              "scaling_mode": args.scaling + (" (batch grows with GPUs; units per GPU fixed)" if args.scaling == "weak"
                                              else " (fixed workload sharded)"),
              "l2": "inputs (3 x fp16 Q/K/V) larger than L2, and L2 flushed between timed steps"}
    if args.pv_accum != "fp32" and not pv_int8:
        config["pv_accum"] = args.pv_accum

    if args.impl == "reference":
        if rank != 0:
            return
        import numpy as np

        from paper_2410_02367_b200 import synth

        threads = args.cpu_threads or os.cpu_count() or 1
        q0, k0, v0 = (x[0] for x in synth.qkv(1, n, d, dtype=np.float32))
        for _ in range(args.warmup):
            cpu_reference_sample(wl, threads, target_s=1.0, q=q0, k=k0, v=v0)
        vals, secs = [], []
        s = None
        for _ in range(args.steps):
            s = cpu_reference_sample(wl, threads, target_s=1.0, q=q0, k=k0, v=v0)
            vals.append(s["value"])
            secs.append(s["seconds"])
        value = statistics.median(vals)
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(secs), "higher_is_better": True,
                "scaling": args.scaling, "vs_baseline": None, "dtype": "int8 QK / fp16 PV (binary16 emulated on CPU)",
                "data": "synthetic N(0,1) fp16 (seeded counter RNG), widened to fp32 for the reference",
                "config": config, "impl": "reference",
                "cpu_baseline": {"value": value, "unit": UNIT, "cores": s["cores"], "kind": s["kind"],
                                 "sample": s["sample"]},
                "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import numpy as np
    import torch

    from paper_2410_02367_b200 import _lib, sageattn

    dist = None
    n_dev = torch.cuda.device_count()
    dev = torch.device("cuda", local_rank % max(1, n_dev))
    torch.cuda.set_device(dev)
    red_dev = dev
    if world > 1:
        import torch.distributed as dist

        # One rank per GPU over NCCL; if ranks outnumber GPUs (functional runs on a
        # 1-GPU box) the two host-side collectives (barrier, max of timings) use gloo.
        if n_dev >= world:
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
            red_dev = torch.device("cpu")
    first, count = _lib.shard_plan(units_total, world, rank)
    if args.shard_of and world == 1:
        first, count = _lib.shard_plan(units_total, args.shard_of, 0)
        total_ops = paper_ops(count, n, d, causal)
        config["shard_of"] = {"gpus": args.shard_of, "rank": 0, "first_unit": first, "units": count,
                              "note": "value is this shard's paper-OPS / its step time on one GPU"}

    q, k, v = device_inputs(count, n, d, first, dev)
    data = ("synthetic N(0,1) fp16 from the seeded counter RNG (global index; synth.tensor_torch, generated on "
            "the device), Q/K/V seeds 1/2/3")
    o = torch.empty_like(q)
    desc = sageattn.make_desc(q, causal, out_dtype=torch.float16, per_token=per_token, pv_int8=pv_int8,
                               pv_accum="fp32" if pv_int8 else args.pv_accum)
    ws = sageattn.Workspace(desc, dev)
    lay = _lib.SabWsLayout()
    _lib.check(_lib.load().sab_workspace_layout(ctypes.byref(desc), ctypes.byref(lay)))
    config["kv_split"] = {"kv_chunk_tiles": lay.kv_chunk, "chunks": lay.kv_nchunk} if lay.kv_chunk else "off"
    # K2's launch mode, mirroring launch_k2's heuristic (persistent for causal or <= 8 items/SM).
    sms_dev = torch.cuda.get_device_properties(dev).multi_processor_count
    k2_items = count * ((-(-n // 128) + 1) // 2) if not lay.kv_chunk else None
    persist_env = os.environ.get("SAB_K2_PERSIST")
    many = k2_items is None or k2_items > sms_dev
    config["k2_launch"] = ("persistent" if many and (persist_env == "1" or (persist_env is None and (
        causal or (k2_items is not None and k2_items <= 8 * sms_dev)))) else "one CTA per item")
    flush = torch.empty(2 * L2_BYTES, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream
    lib = _lib.load()
    C = ctypes

    def step(ev=None):
        _lib.check(lib.sab_prepass(C.byref(desc), q.data_ptr(), k.data_ptr(), v.data_ptr() if pv_int8 else None,
                                   ws.ptr, ws.nbytes, sp))
        if ev is not None:  # an event between K1 and K2 also stops K2 launching behind K1 (PDL)
            ev[1].record(stream)
        _lib.check(lib.sab_attention(C.byref(desc), ws.ptr, ws.nbytes, v.data_ptr(), o.data_ptr(), sp))

    for _ in range(args.warmup):
        flush.fill_(1)
        step()
    torch.cuda.synchronize()
    _lib.check(sageattn.read_status(ws))

    # Overlapped step (optional): the shard's units in groups, each group with its own
    # workspace and stream; K1(g+1) overlaps K2(g).  Units are independent,
    # so the groups compute exactly what the one-launch step computes.
    groups = overlap_groups(args.groups, count, n, d)
    if len(groups) > 1:
        gsteps, g0 = [], 0
        for gi, gc in enumerate(groups):
            sl = slice(g0, g0 + gc)
            gq, gk, gv, go = (t[:, sl] for t in (q, k, v, o))
            gdesc = sageattn.make_desc(gq, causal, out_dtype=torch.float16, per_token=per_token, pv_int8=pv_int8,
                                       pv_accum="fp32" if pv_int8 else args.pv_accum)
            gsteps.append((gdesc, sageattn.Workspace(gdesc, dev), gq, gk, gv, go,
                           stream if gi == 0 else torch.cuda.Stream(dev), torch.cuda.Event()))
            g0 += gc
        join = [torch.cuda.Event() for _ in groups]
        fork = torch.cuda.Event()

        def step_overlap(ev=None):
            fork.record(stream)
            prev = fork
            for gi, (gdesc, gws, gq, gk, gv, go, gs, k1_done) in enumerate(gsteps):
                gs.wait_event(prev)
                gp = gs.cuda_stream
                _lib.check(lib.sab_prepass(C.byref(gdesc), gq.data_ptr(), gk.data_ptr(),
                                           gv.data_ptr() if pv_int8 else None, gws.ptr, gws.nbytes, gp))
                k1_done.record(gs)
                prev = k1_done
                _lib.check(lib.sab_attention(C.byref(gdesc), gws.ptr, gws.nbytes, gv.data_ptr(), go.data_ptr(), gp))
                join[gi].record(gs)
            for e in join[1:]:
                stream.wait_event(e)

        step()
        o_serial = o.clone()
        o.zero_()
        for _ in range(args.warmup):
            flush.fill_(1)
            step_overlap()
        torch.cuda.synchronize()
        if not torch.equal(o, o_serial):
            raise SystemExit("overlapped step differs from the one-launch step")
        for g in gsteps:
            _lib.check(sageattn.read_status(g[1]))

    probe = tensor_peak_probe() if rank == 0 else None
    sampler = ClockSampler(dev.index)
    with sampler:
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        # Split pass: an event between K1 and K2 gives the per-kernel times for the rooflines.
        evs = time_steps(lambda ev: step(ev), stream, flush, args.steps)
        t_serial = [ev[0].elapsed_time(ev[2]) for ev in evs]
        t_k1 = [ev[0].elapsed_time(ev[1]) for ev in evs]
        t_k2 = [ev[1].elapsed_time(ev[2]) for ev in evs]
        # Headline pass: the step exactly as a caller issues it (no event between K1 and
        # K2, so K2 launches behind K1's last wave), or the overlapped step.
        headline = (lambda ev: step_overlap()) if len(groups) > 1 else (lambda ev: step())
        evs = time_steps(headline, stream, flush, args.steps)
        t_step = [ev[0].elapsed_time(ev[2]) for ev in evs]
        if dist:
            dist.barrier()

    # ---- end to end through the C-ABI host-buffer call (pinned host fp16 in, fp16 out)
    e2e_steps = args.e2e_steps or max(3, min(args.steps, 10))
    host = [t.reshape(1, count, n, d).cpu() for t in (q, k, v)]
    hq, hk, hv = (h.contiguous().pin_memory().numpy() for h in host)
    ho = torch.empty(hq.shape, dtype=torch.float16).pin_memory().numpy()
    acc = "fp32" if pv_int8 else args.pv_accum
    sageattn.attention_fwd_host(hq, hk, hv, causal, ho, devices=[dev.index], per_token=per_token,
                                pv_int8=pv_int8, pv_accum=acc)  # warm pool
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        sageattn.attention_fwd_host(hq, hk, hv, causal, ho, devices=[dev.index], per_token=per_token,
                                    pv_int8=pv_int8, pv_accum=acc)
    e2e_s = time.perf_counter() - t0

    local = torch.tensor([sum(t_step), sum(t_k1), sum(t_k2), e2e_s, sum(t_serial)], dtype=torch.float64,
                         device=red_dev)
    if dist:
        dist.all_reduce(local, op=dist.ReduceOp.MAX)
    tot_ms, k1_ms, k2_ms, e2e_max, serial_ms = local.tolist()
    ms_per_step = tot_ms / args.steps
    value = total_ops / (ms_per_step * 1e-3) / 1e12
    e2e_value = total_ops * e2e_steps / e2e_max / 1e12

    # Roofline of K2 (dominant): paper-OPS per launch / mean K2 time on this rank.
    peaks, peak_src = measured_peaks()
    p_f16 = peaks["bf16_tflops"]
    pm = p_mix(2.0 * p_f16, p_f16)  # QK on the INT8 pipe (2x fp16 rate), PV on fp16
    shard_ops = paper_ops(count, n, d, causal)
    k2_mean_ms = statistics.mean(t_k2)
    k2_ach = shard_ops / (k2_mean_ms * 1e-3) / 1e12
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "k2_traffic.json")) as f:
            traffic = json.load(f).get(f"{args.workload}")  # bytes per launch, whole job
    except (OSError, ValueError):
        pass
    k1_bytes = count * (6 * n * d + 4 * (-(-n // 128) + -(-n // 64) + d)) + count * 2 * n * d  # + K re-read
    k1_alg = count * (6 * n * d + 4 * (-(-n // 128) + -(-n // 64) + d))
    k1_mean_ms = statistics.mean(t_k1)

    if dist:
        dist.destroy_process_group()
    if rank != 0:
        return
    clocks = sampler.summary()
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    line = {
        "metric": METRIC.replace("SageAttn-B", "SageAttn-" + {"B": "B", "T": "T", "VB": "vB", "VT": "vT"}[args.variant]),
        "value": value,
        "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "int8 QK^T (s32 acc) / fp16 PV (fp32 acc); fp16 Q/K/V/O",
        "data": data, "config": config,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 3 * (count if args.shard_of else units_total) * n * d * 2,
                "d2h_bytes_per_step": (count if args.shard_of else units_total) * n * d * 2,
                "how": "sab_attention_fwd_host on pinned host fp16 buffers, fp16 O; wall clock, max over ranks"},
        # k1_mean_and_q (+ fused tree top) + k1_k_fast + k2_attention; vB adds k1_v_amax + k1_v_quant
        "gpu_launches": args.steps * (5 if pv_int8 else 3) * len(groups),
        "roofline": {"bound": "tensor", "achieved": k2_ach, "peak": pm, "unit": "TFLOP/s",
                     "frac": k2_ach / pm, "traffic": traffic, "kernel": "k2_attention",
                     "ms_per_launch": k2_mean_ms,
                     "alg_work_per_launch": f"{shard_ops:.4e} paper-OPS (2*N^2*d int8 + 2*N^2*d fp16 per unit"
                                            f"{', halved' if causal else ''}; SURVEY 8(d))",
                     "peak_source": f"{peak_src} bf16_tflops={p_f16} for the fp16 PV half, 2x for the int8 QK half "
                                    "(datasheet ratio); paper-OPS are int8+fp16 ops",
                     "frac_of_int8_dense_peak": k2_ach / (2.0 * p_f16),
                     # The same roofline from the power-capped (sustained) bf16 rate: a 12 ms K2
                     # launch timed back to back runs under sw_power_cap like a long GEMM loop.
                     "peak_sustained": p_mix(2.0 * peaks["bf16_tflops_sustained"], peaks["bf16_tflops_sustained"]),
                     "frac_of_sustained": k2_ach / p_mix(2.0 * peaks["bf16_tflops_sustained"],
                                                         peaks["bf16_tflops_sustained"])},
        "roofline_k1": {"bound": "hbm", "achieved": k1_alg / (k1_mean_ms * 1e-3) / 1e9, "peak": peaks["hbm_gbs"],
                        "unit": "GB/s", "frac": k1_alg / (k1_mean_ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
                        "ms_per_step": k1_mean_ms, "alg_bytes": k1_alg, "min_dram_bytes_with_k_reread": k1_bytes},
        "clocks": clocks,
        "step_schedule": {"groups": groups, "ms_per_step_split_pass": serial_ms / args.steps,
                          "note": "K1(g+1) overlaps K2(g) on per-group streams" if len(groups) > 1
                          else "K1 then K2, one launch each (PDL: K2's prologue overlaps K1's tail)"},
        "contract_notes": ["O is written as fp16 (the reference returns fp32: relL1 cost ~1.8e-4, SURVEY P9); "
                           "e2e_dropin returns fp32",
                           "the device step runs with check_v=0 (sab_desc_init default): V's finiteness scan "
                           "(attention.hpp:101) is part of the drop-in path (e2e_dropin), not of this step"],
    }
    clk = clocks.get("sm_mhz") or clocks.get("sm_max_mhz") or 1965
    if probe:
        i8c, f16c = probe["i8"]["ops_per_clk_per_sm"], probe["f16"]["ops_per_clk_per_sm"]
        pk = p_mix(i8c * sms * clk * 1e6 / 1e12, f16c * sms * clk * 1e6 / 1e12)
        line["roofline"].update({
            "peak_at_clock": pk, "frac_at_clock": k2_ach / pk, "clock_mhz": clk,
            "int8_peak_at_clock": i8c * sms * clk * 1e6 / 1e12,
            "frac_of_int8_peak_at_clock": k2_ach / (i8c * sms * clk * 1e6 / 1e12),
            "tcgen05_probe": {"i8_ops_per_clk_per_sm": i8c, "f16_flops_per_clk_per_sm": f16c,
                              "i8_tops_probe": probe["i8"]["tops"], "f16_tflops_probe": probe["f16"]["tops"],
                              "probe_mhz": probe["i8"]["probe_mhz"],
                              "how": "bench_support/sab_peak.cu: M=128 N=256 SS tcgen05.mma back to back, "
                                     "148 CTAs, random operands"}})
    # Second bound of K2: one exp2 per attended (query, key) pair on MUFU (16 lanes/clk/SM,
    # profiles/r01_micro_mufu.txt); 2 of every 16 run on the FMA pipe instead.
    exps = shard_ops / (4.0 * d)
    line["roofline_xu"] = {"bound": "xu (MUFU ex2)", "achieved": exps / (k2_mean_ms * 1e-3) / 1e12,
                           "peak": 16.0 * sms * clk * 1e6 / 1e12, "unit": "Texp/s",
                           "frac": exps / (k2_mean_ms * 1e-3) / (16.0 * sms * clk * 1e6),
                           "note": "algorithmic exponentials (one per attended pair); 2/16 run on the FMA pipe"}
    if world == 1 and not args.no_dropin and args.variant == "B":
        dr = dropin_e2e(hq, hk, hv, wl, batch, iters=3)
        if dr and "seconds_per_call" in dr:
            line["e2e_dropin"] = {"value": total_ops / dr["seconds_per_call"] / 1e12, "unit": UNIT, **dr}
        elif dr:
            line["e2e_dropin"] = dr
    if world == 1 and not args.no_cpu_baseline and args.variant == "B":
        threads = args.cpu_threads or os.cpu_count() or 1
        q0, k0, v0 = (t[0, 0].float().cpu().numpy() for t in (q, k, v))
        s = cpu_reference_sample(wl, threads, q=q0, k=k0, v=v0)
        line["cpu_baseline"] = {"value": s["value"], "unit": UNIT, "cores": s["cores"], "kind": s["kind"],
                                "sample": s["sample"], "seconds": s["seconds"]}
        line["parity"] = parity_report(wl, q0, k0, v0, o[0, 0].float().cpu().numpy(), s, threads)
    if world == 1 and not args.no_secondary and args.workload != "C2" and args.variant == "B":
        line["secondary"] = secondary_c2(dev, flush, lib, stream)
    print(json.dumps(line))


def secondary_c2(dev, flush, lib, stream, steps: int = 10):
    """C2 (Llama-2-7B prefill, BASELINE configs[1]) device-time step, same timing rules."""
    import torch

    from paper_2410_02367_b200 import _lib, sageattn

    wl = workload("C2")
    n, d = wl["tokens"], wl["head_dim"]
    units = wl["batch"] * wl["heads"]
    q, k, v = device_inputs(units, n, d, 0, dev)
    o = torch.empty_like(q)
    desc = sageattn.make_desc(q, True, out_dtype=torch.float16)
    ws = sageattn.Workspace(desc, dev)
    sp = stream.cuda_stream

    def step(ev=None):
        _lib.check(lib.sab_prepass(ctypes.byref(desc), q.data_ptr(), k.data_ptr(), None, ws.ptr, ws.nbytes, sp))
        _lib.check(lib.sab_attention(ctypes.byref(desc), ws.ptr, ws.nbytes, v.data_ptr(), o.data_ptr(), sp))

    for _ in range(3):
        flush.fill_(1)
        step()
    evs = time_steps(step, stream, flush, steps)
    _lib.check(sageattn.read_status(ws))
    ms = statistics.mean(ev[0].elapsed_time(ev[2]) for ev in evs)
    return {"workload": wl["name"], "value": paper_ops(units, n, d, True) / (ms * 1e-3) / 1e12, "unit": UNIT,
            "ms_per_step": ms, "steps": steps, "warmup": 3, "how": "K1 + K2 device time, L2 flushed between steps"}


if __name__ == "__main__":
    main()
