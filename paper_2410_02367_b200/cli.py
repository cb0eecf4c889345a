"""NPY tensor I/O and the command-line surface of SPEC.md's io-cli module.

    python -m paper_2410_02367_b200.cli gen --shape 1,2,1024,64 --dist outlier --seed 7 --out /tmp/t
    python -m paper_2410_02367_b200.cli accuracy --shape 2,8,1024,64 --variant all --out report.json
    python -m paper_2410_02367_b200.cli calibrate --layers 4 --threshold 0.998 --out plan.json
    python -m paper_2410_02367_b200.cli bench --shape 1,32,8192,128 --causal --variant b --repeats 5

Commands and flags follow SPEC.md:401-405.  Every kernel call goes to the B200
library; the accuracy yardstick is binary64 exact attention on the device
(calibrate.exact_attention).  Reports are one JSON document per run.
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from typing import List, Sequence

import numpy as np

from . import synth
from .calibrate import accuracy, calibrate, exact_attention
from .sageattn import AttentionInput, SageOptions, SageVariant, kernel_config_for

_VARIANTS = {"t": SageVariant.T, "b": SageVariant.B, "vt": SageVariant.VT, "vb": SageVariant.VB}
_NAMES = {SageVariant.T: "SAGEAttn-T", SageVariant.B: "SAGEAttn-B", SageVariant.VT: "SAGEAttn-vT",
          SageVariant.VB: "SAGEAttn-vB"}


# ---------------------------------------------------------------------------- NPY v1.0

class TensorFileError(ValueError):
    """Base of the distinct tensor-file errors."""


class MalformedHeader(TensorFileError):
    pass


class UnsupportedLayout(TensorFileError):
    pass


class UnsupportedDtype(TensorFileError):
    pass


class ShapeError(TensorFileError):
    pass


class TruncatedPayload(TensorFileError):
    pass


def load_tensor(path: str) -> np.ndarray:
    """NPY v1.0, C order, '<f4' or '<f2', 4-D (B,H,N,d); binary16 is upcast to binary32."""
    import ast

    with open(path, "rb") as f:
        raw = f.read()
    if raw[:6] != b"\x93NUMPY" or len(raw) < 10:
        raise MalformedHeader(f"{path}: not an NPY file")
    if raw[6] != 1:
        raise MalformedHeader(f"{path}: NPY version {raw[6]}.{raw[7]} (1.0 expected)")
    hlen = int.from_bytes(raw[8:10], "little")
    try:
        hdr = ast.literal_eval(raw[10:10 + hlen].decode("latin1"))
        descr, fortran, shape = hdr["descr"], hdr["fortran_order"], tuple(hdr["shape"])
    except Exception as e:  # noqa: BLE001
        raise MalformedHeader(f"{path}: bad header ({e})") from None
    if fortran:
        raise UnsupportedLayout(f"{path}: Fortran-order arrays are not supported")
    if descr not in ("<f4", "<f2"):
        raise UnsupportedDtype(f"{path}: dtype {descr} (expected <f4 or <f2)")
    if len(shape) != 4 or min(shape) < 1:
        raise ShapeError(f"{path}: shape {shape} is not a 4-D (B,H,N,d) tensor")
    item = 4 if descr == "<f4" else 2
    payload = raw[10 + hlen:]
    need = int(np.prod(shape)) * item
    if len(payload) < need:
        raise TruncatedPayload(f"{path}: payload {len(payload)} bytes, header needs {need}")
    a = np.frombuffer(payload[:need], dtype=descr).reshape(shape)
    return a.astype(np.float32)


def save_tensor(t: np.ndarray, path: str) -> None:
    a = np.ascontiguousarray(t)
    if a.ndim != 4:
        raise ShapeError(f"save_tensor: shape {a.shape} is not 4-D")
    if a.dtype not in (np.float32, np.float16):
        raise UnsupportedDtype(f"save_tensor: dtype {a.dtype}")
    np.lib.format.write_array(open(path, "wb"), a, version=(1, 0))


# ---------------------------------------------------------------------------- synthetic inputs

def generate(shape: Sequence[int], dist: str = "normal", seed: int = 0, bias_scale: float = 10.0,
             noise_scale: float = 1.0, causal: bool = False) -> AttentionInput:
    """Deterministic (B,H,N,d) Q/K/V from the counter RNG; `outlier` = ChannelOutlier K."""
    b, h, n, d = (int(x) for x in shape)
    if min(b, h, n, d) < 1:
        raise ShapeError(f"generate: invalid shape {tuple(shape)}")
    units = b * h
    q = synth.tensor(3 * seed + 1, (units, n, d), dtype=np.float32)
    k = synth.tensor(3 * seed + 2, (units, n, d), dtype=np.float32, dist=dist, bias_scale=bias_scale,
                     noise_scale=noise_scale)
    v = synth.tensor(3 * seed + 3, (units, n, d), dtype=np.float32)
    return AttentionInput(*(x.reshape(b, h, n, d) for x in (q, k, v)), causal=causal)


# ---------------------------------------------------------------------------- commands

def _device_exact(inp: AttentionInput) -> np.ndarray:
    import torch

    dev = torch.device("cuda", 0)
    q, k, v = (torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (inp.q, inp.k, inp.v))
    return exact_attention(q, k, v, inp.causal).cpu().numpy()


def _input(args) -> AttentionInput:
    if args.q:
        q, k, v = (load_tensor(p) for p in (args.q, args.k, args.v))
        return AttentionInput(q, k, v, causal=args.causal)
    return generate(args.shape, args.dist, args.seed, args.bias_scale, args.noise_scale, args.causal)


def _variants(name: str) -> List[SageVariant]:
    return list(_VARIANTS.values()) if name == "all" else [_VARIANTS[name]]


def cmd_accuracy(args) -> dict:
    inp = _input(args)
    from .sageattn import sage_attention

    exact = _device_exact(inp)
    rows = {}
    for var in _variants(args.variant):
        for smooth in ([True, False] if args.no_smooth else [True]):
            o = sage_attention(inp, var, SageOptions(smooth_k=smooth))
            r = accuracy(o, exact)
            rows[_NAMES[var] + ("" if smooth else " (no smooth-K)")] = dict(cos_sim=r.cos_sim,
                                                                             relative_l1=r.relative_l1,
                                                                             rmse=r.rmse)
    return dict(command="accuracy", shape=list(inp.q.shape), causal=inp.causal, dist=args.dist, seed=args.seed,
                reference="exact attention, binary64", report=rows)


def cmd_calibrate(args) -> dict:
    import torch

    if args.layers < 1:
        raise ValueError("calibrate: empty calibration set")
    dev = torch.device("cuda", 0)
    layers = []
    for i in range(args.layers):
        batches = []
        for bt in range(args.batches):
            inp = generate(args.shape, args.dist, args.seed + 1000 * i + bt, args.bias_scale, args.noise_scale,
                           args.causal)
            batches.append(tuple(torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (inp.q, inp.k, inp.v))
                           + (inp.causal,))
        layers.append(batches)
    plan = calibrate(layers, threshold=args.threshold, aggregate=args.aggregate)
    vb = kernel_config_for(SageVariant.VB)
    return dict(command="calibrate", threshold=plan.threshold,
                layers=[dict(layer=i, kernel="SAGEAttn-vB" if c == vb else "SAGEAttn-B", cos_sim=s)
                        for i, (c, s) in enumerate(zip(plan.assignments, plan.cos_sim))])


def cmd_bench(args) -> dict:
    if args.repeats < 3:
        raise ValueError("bench: --repeats must be >= 3")
    import torch

    from .sageattn import sage_attention_cuda

    b, h, n, d = args.shape
    inp = generate(args.shape, args.dist, args.seed, causal=args.causal)
    dev = torch.device("cuda", 0)
    q, k, v = (torch.from_numpy(np.ascontiguousarray(x)).to(dev).half() for x in (inp.q, inp.k, inp.v))
    ops = 4.0 * b * h * n * n * d * (0.5 if args.causal else 1.0)
    rows = {}
    for var in _variants(args.variant):
        cfg = kernel_config_for(var)
        kw = dict(causal=args.causal, per_token=cfg.qk_granularity.name == "PerToken",
                  pv_int8=cfg.pv_path.name == "Int8", check=False)
        out = sage_attention_cuda(q, k, v, **kw)
        ts = []
        for _ in range(args.repeats):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            sage_attention_cuda(q, k, v, out=out, **kw)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e-3)
        t = float(np.median(ts))
        rows[_NAMES[var]] = dict(median_s=t, tops=ops / t / 1e12, s_stage_ops=2.0 * b * h * n * n * d)
    return dict(command="bench", shape=[b, h, n, d], causal=args.causal, repeats=args.repeats,
                timing="B200 device time (CUDA events), K1 + K2", report=rows)


def cmd_gen(args) -> dict:
    inp = generate(args.shape, args.dist, args.seed, args.bias_scale, args.noise_scale)
    paths = {}
    for name, t in (("q", inp.q), ("k", inp.k), ("v", inp.v)):
        paths[name] = f"{args.out}.{name}.npy"
        save_tensor(t, paths[name])
    return dict(command="gen", shape=list(inp.q.shape), dist=args.dist, seed=args.seed, files=paths)


def _shape(s: str):
    parts = [int(x) for x in s.split(",")]
    if len(parts) != 4:
        raise argparse.ArgumentTypeError("--shape takes B,H,N,d")
    return parts


def parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_2410_02367_b200.cli")
    sub = ap.add_subparsers(dest="command", required=True)
    for name in ("accuracy", "calibrate", "bench", "gen"):
        p = sub.add_parser(name)
        p.add_argument("--shape", type=_shape, default=[2, 8, 1024, 64])
        p.add_argument("--dist", choices=["normal", "outlier"], default="normal")
        p.add_argument("--bias-scale", type=float, default=10.0)
        p.add_argument("--noise-scale", type=float, default=1.0)
        p.add_argument("--seed", type=int, default=0)
        p.add_argument("--causal", action="store_true")
        p.add_argument("--out", default=None)
        if name in ("accuracy", "bench"):
            p.add_argument("--variant", choices=["t", "b", "vt", "vb", "all"], default="all")
        if name == "accuracy":
            p.add_argument("--no-smooth", action="store_true", help="add the no-smoothing ablation rows")
            p.add_argument("--q")
            p.add_argument("--k")
            p.add_argument("--v")
        if name == "calibrate":
            p.add_argument("--threshold", type=float, default=0.998)
            p.add_argument("--layers", type=int, default=4)
            p.add_argument("--batches", type=int, default=8)
            p.add_argument("--aggregate", choices=["mean", "min"], default="mean")
        if name == "bench":
            p.add_argument("--repeats", type=int, default=5)
    return ap


def main(argv=None) -> int:
    args = parser().parse_args(argv)
    if args.command == "gen" and not args.out:
        raise SystemExit("gen: --out is required")
    t0 = time.perf_counter()
    rep = {"accuracy": cmd_accuracy, "calibrate": cmd_calibrate, "bench": cmd_bench, "gen": cmd_gen}[args.command](args)
    rep["wall_s"] = time.perf_counter() - t0
    text = json.dumps(rep, indent=1)
    if args.out and args.command != "gen":
        with open(args.out, "w") as f:
            f.write(text + "\n")
    print(text)
    return 0


if __name__ == "__main__":
    sys.exit(main())
