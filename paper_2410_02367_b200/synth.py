"""Seeded counter-based synthetic inputs.

Every value is a pure function of (seed, global element index), so a
shard of units generated on its own equals the matching slice of the
whole tensor -- the property head x batch sharding relies on.

* ``normal``: N(0,1) from splitmix64 + Box-Muller, rounded to fp16 (the
  paper's "normal distribution").
* ``outlier``: ChannelOutlier K = bias[c] + noise, bias ~ bias_scale*N(0,1)
  shared by all tokens of a unit, used to stress smooth-K.

Seeds Q=1, K=2, V=3 by convention.
"""
from __future__ import annotations

import numpy as np

_GOLD = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x + _GOLD
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def normal(seed: int, start: int, count: int) -> np.ndarray:
    """float64 N(0,1) values for global indices [start, start+count)."""
    with np.errstate(over="ignore"):
        idx = np.arange(start, start + count, dtype=np.uint64)
        key = np.uint64(seed) * np.uint64(0xD1B54A32D192ED03)
        h = _splitmix64(idx ^ key)
    u1 = ((h >> np.uint64(40)).astype(np.float64) + 0.5) * (1.0 / (1 << 24))
    u2 = ((h & np.uint64(0xFFFFFF)).astype(np.float64) + 0.5) * (1.0 / (1 << 24))
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


def tensor(seed: int, shape, unit0: int = 0, dtype=np.float16, dist: str = "normal", bias_scale: float = 10.0,
           noise_scale: float = 1.0) -> np.ndarray:
    """(units, N, d) tensor for units [unit0, unit0 + units) of a global tensor of the same N, d."""
    units, n, d = shape
    per = n * d
    z = normal(seed, unit0 * per, units * per).reshape(units, n, d)
    if dist == "outlier":
        bias = normal(seed ^ 0x5EED, 1 << 40 | unit0 * d, units * d).reshape(units, 1, d) * bias_scale
        z = bias + noise_scale * z
    elif dist != "normal":
        raise ValueError(f"unknown distribution {dist!r}")
    return z.astype(np.float16).astype(dtype)


def qkv(units: int, n: int, d: int, unit0: int = 0, dtype=np.float16, dist: str = "normal"):
    """Q (seed 1), K (seed 2, `dist`), V (seed 3)."""
    shape = (units, n, d)
    return (tensor(1, shape, unit0, dtype), tensor(2, shape, unit0, dtype, dist=dist), tensor(3, shape, unit0, dtype))


def tensor_torch(seed: int, shape, unit0: int = 0, device="cuda", dtype=None, chunk_units: int = 8):
    """Same counter-based N(0,1) values as ``tensor(..., dist="normal")``, generated with torch on
    `device` (the bench's full-size inputs; numpy would take minutes at C4/C5 sizes).

    splitmix64 runs in int64 with wrap-around multiplies and masked (logical) right shifts;
    Box-Muller runs in float64, so values equal the numpy ones up to the last ulp of the
    binary64 log/cos before the fp16 rounding (a handful of fp16 ties can differ)."""
    import torch

    dtype = dtype or torch.float16
    units, n, d = shape
    per = n * d
    out = torch.empty((units, n, d), dtype=dtype, device=device)

    def u64(x: int) -> int:  # the int64 with the same 64 bits
        return x - (1 << 64) if x >= (1 << 63) else x

    def lsr(x, s):
        return (x >> s) & ((1 << (64 - s)) - 1)

    gold, m1, m2 = u64(0x9E3779B97F4A7C15), u64(0xBF58476D1CE4E5B9), u64(0x94D049BB133111EB)
    key = u64((seed * 0xD1B54A32D192ED03) % (1 << 64))
    for u0 in range(0, units, chunk_units):
        uc = min(chunk_units, units - u0)
        idx = torch.arange((unit0 + u0) * per, (unit0 + u0 + uc) * per, dtype=torch.int64, device=device)
        z = (idx ^ key) + gold
        z = (z ^ lsr(z, 30)) * m1
        z = (z ^ lsr(z, 27)) * m2
        h = z ^ lsr(z, 31)
        u1 = (lsr(h, 40).to(torch.float64) + 0.5) * (1.0 / (1 << 24))
        u2 = ((h & 0xFFFFFF).to(torch.float64) + 0.5) * (1.0 / (1 << 24))
        val = torch.sqrt(-2.0 * torch.log(u1)) * torch.cos(2.0 * torch.pi * u2)
        out[u0:u0 + uc] = val.reshape(uc, n, d).to(torch.float16).to(dtype)
    return out
