"""ctypes bindings for the CPU checkers -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg import
this module, and only as the checker: the product path
(paper_2410_02367_b200) never imports it and fails loudly without its CUDA
library.

Two libraries are bound:

* ``Oracle`` -> oracle/liboracle.so, the plain-C restatement in
  sage_oracle.c (each function cites the reference file:line it follows);
* ``Reference`` -> oracle/_ref/libsageref.so, the reference's own headers
  compiled where they lie under /root/reference (ref_driver.cpp).  The
  restatement is pinned bit-for-bit against it in tests/test_oracle.py.

Arrays are numpy, (units, N, d) row-major float32 unless stated.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsageref.so")

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i8p = np.ctypeslib.ndpointer(np.int8, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_intp = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")

BLOCK_Q = 128
BLOCK_KV = 64


def build():
    """Compile liboracle.so (and _ref/libsageref.so when /root/reference exists)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


class Oracle:
    """The C restatement (sage_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        lib = C.CDLL(path)
        lib.orc_snap_half.restype = C.c_double
        lib.orc_snap_half.argtypes = [C.c_double]
        lib.orc_half_bits.restype = C.c_uint16
        lib.orc_half_bits.argtypes = [C.c_double]
        lib.orc_mean_k.argtypes = [_f32p, C.c_int, C.c_int, _f32p]
        lib.orc_smooth_k.argtypes = [_f32p, C.c_int, C.c_int, _f32p, _f32p]
        lib.orc_fold_factor.restype = C.c_float
        lib.orc_fold_factor.argtypes = [C.c_int]
        lib.orc_quantize_int8_rows.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, _i8p, _f32p]
        lib.orc_prepass_unit.argtypes = [_f32p, _f32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                         _i8p, _f32p, _i8p, _f32p, _f32p]
        lib.orc_int8_tile_nt.argtypes = [_i8p, _i8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _i32p, C.c_int]
        lib.orc_causal_tile.argtypes = [C.c_int] * 5
        lib.orc_sage_b_tiles.argtypes = [_i8p, _f32p, _i8p, _f32p, _f32p, C.c_int, C.c_int, C.c_int, C.c_int,
                                         C.c_int, C.c_int, C.c_int, C.c_int, _f32p, _u64p]
        lib.orc_sage_b.argtypes = [_f32p, _f32p, _f32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                   C.c_int, _f32p, _u64p]
        lib.orc_sage.argtypes = [_f32p, _f32p, _f32p] + [C.c_int] * 8 + [_f32p, _u64p]
        lib.orc_sage_tiles.argtypes = [_i8p, _f32p, _i8p, _f32p, _f32p] + [C.c_int] * 10 + [_f32p, _u64p]
        lib.orc_sage_v.argtypes = [_f32p, _f32p, _f32p] + [C.c_int] * 9 + [_f32p, _u64p]
        lib.orc_quantize_int8_cols.argtypes = [_f32p, C.c_int, C.c_int, _i8p, _f32p]
        lib.orc_naive.argtypes = [_f32p, _f32p, _f32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _f64p]
        lib.orc_naive_rows.argtypes = [_f32p, _f32p, _f32p] + [C.c_int] * 5 + [_f64p]
        lib.orc_rope.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, _f32p, _f32p, C.c_int]
        self.lib = lib

    # -- RoPE (sab_prepass_rope's rotation, binary32 with every op rounded) ---------
    def rope(self, x, cos, sin, layout):
        """x (units, n, d) rotated by cos/sin (n, d/2); layout "interleaved" (pairs 2i, 2i+1)
        or "half" (pairs i, i + d/2).  Returns a new float32 array."""
        x = np.array(_f32(x), dtype=np.float32, copy=True)
        units, n, d = x.shape
        self.lib.orc_rope(x, units, n, d, _f32(cos), _f32(sin), {"interleaved": 1, "half": 2}[layout])
        return x

    # -- scalar numerics ------------------------------------------------
    def snap_half(self, x: float) -> float:
        return self.lib.orc_snap_half(float(x))

    def half_bits(self, x: float) -> int:
        return self.lib.orc_half_bits(float(x))

    # -- prepass ----------------------------------------------------------
    def prepass(self, q, k, smooth=True, block_q=BLOCK_Q, block_kv=BLOCK_KV, per_token=False):
        """Per-unit fold+quantize(Q) and smooth+quantize(K); per_token: one scale per
        token (variant T, Granularity::per_token = groups of one row).

        Returns dict(qcodes, qscales, kcodes, kscales, mean) or raises
        ValueError on non-finite input."""
        if per_token:
            block_q = block_kv = 1
        q, k = _f32(q), _f32(k)
        units, n, d = q.shape
        gq, gk = -(-n // block_q), -(-n // block_kv)
        out = dict(qcodes=np.empty((units, n, d), np.int8), qscales=np.empty((units, gq), np.float32),
                   kcodes=np.empty((units, n, d), np.int8), kscales=np.empty((units, gk), np.float32),
                   mean=np.empty((units, d), np.float32))
        for u in range(units):
            qc, qs, kc, ks, mn = (np.empty((n, d), np.int8), np.empty(gq, np.float32), np.empty((n, d), np.int8),
                                  np.empty(gk, np.float32), np.empty(d, np.float32))
            st = self.lib.orc_prepass_unit(np.ascontiguousarray(q[u]), np.ascontiguousarray(k[u]), n, d, block_q,
                                           block_kv, int(smooth), qc, qs, kc, ks, mn)
            if st == 2:
                raise ValueError("sage_attention: non-finite input")
            if st != 0:
                raise RuntimeError(f"oracle prepass failed: {st}")
            out["qcodes"][u], out["qscales"][u], out["kcodes"][u], out["kscales"][u], out["mean"][u] = qc, qs, kc, ks, mn
        return out

    def mean_k(self, k):
        k = _f32(k)
        units, n, d = k.shape
        out = np.empty((units, d), np.float32)
        for u in range(units):
            m = np.empty(d, np.float32)
            self.lib.orc_mean_k(np.ascontiguousarray(k[u]), n, d, m)
            out[u] = m
        return out

    def int8_tile(self, qc, kc, r0, bq, c0, bkv):
        n, d = qc.shape
        acc = np.empty((bq, bkv), np.int32)
        self.lib.orc_int8_tile_nt(np.ascontiguousarray(qc), np.ascontiguousarray(kc), d, r0, bq, c0, bkv, acc, bkv)
        return acc

    def causal_tile(self, i, j, bq, bkv, n):
        return self.lib.orc_causal_tile(i, j, bq, bkv, n)

    # -- attention --------------------------------------------------------
    def sage_b(self, q, k, v, causal=False, smooth=True, pv_fp32=True, threads=None):
        """SAGEAttn-B forward; returns (out float32 (units,N,d), macs uint64[2])."""
        q, k, v = _f32(q), _f32(k), _f32(v)
        units, n, d = q.shape
        out = np.empty_like(q)
        macs = np.zeros(2, np.uint64)
        st = self.lib.orc_sage_b(q, k, v, units, n, d, int(causal), int(smooth), int(pv_fp32),
                                 threads or os.cpu_count() or 1, out, macs)
        if st == 2:
            raise ValueError("sage_attention: non-finite input")
        if st == 3:
            raise OverflowError("sage_attention: binary16 P~V accumulator overflowed")
        if st != 0:
            raise RuntimeError(f"oracle failed: {st}")
        return out, macs

    def quantize_per_channel(self, a):
        """V^ of the vB/vT paths: (codes int8 (rows, cols), scales float32 (cols,)) (quant.hpp:128-173)."""
        a = _f32(a)
        rows, cols = a.shape
        codes = np.empty((rows, cols), np.int8)
        scales = np.empty(cols, np.float32)
        st = self.lib.orc_quantize_int8_cols(a, rows, cols, codes, scales)
        if st == 2:
            raise ValueError("sage_attention: non-finite input")
        return codes, scales

    def sage(self, q, k, v, causal=False, smooth=True, pv_fp32=True, per_token=False, threads=None,
             pv_int8=False):
        """SAGEAttn-B / -T (pv_int8=False) or -vB / -vT (pv_int8=True) forward; returns (out, macs)."""
        q, k, v = _f32(q), _f32(k), _f32(v)
        units, n, d = q.shape
        out = np.empty_like(q)
        macs = np.zeros(2, np.uint64)
        st = self.lib.orc_sage_v(q, k, v, units, n, d, int(causal), int(smooth), int(pv_fp32), int(per_token),
                                 int(pv_int8), threads or os.cpu_count() or 1, out, macs)
        if st == 2:
            raise ValueError("sage_attention: non-finite input")
        if st == 3:
            raise OverflowError("sage_attention: binary16 P~V accumulator overflowed")
        if st != 0:
            raise RuntimeError(f"oracle failed: {st}")
        return out, macs

    def sage_tiles(self, pre, v, unit, tiles, causal, pv_fp32=True, per_token=False):
        """sage_b_tiles for either variant (per_token: scale groups of one token)."""
        v = _f32(v)
        n, d = v.shape[1:]
        g_q, g_k = (1, 1) if per_token else (BLOCK_Q, BLOCK_KV)
        out = np.zeros((n, d), np.float32)
        macs = np.zeros(2, np.uint64)
        for t in tiles:
            st = self.lib.orc_sage_tiles(np.ascontiguousarray(pre["qcodes"][unit]), np.ascontiguousarray(pre["qscales"][unit]),
                                         np.ascontiguousarray(pre["kcodes"][unit]), np.ascontiguousarray(pre["kscales"][unit]),
                                         np.ascontiguousarray(v[unit]), n, d, int(causal), int(pv_fp32), BLOCK_Q, BLOCK_KV,
                                         g_q, g_k, int(t), int(t) + 1, out, macs)
            if st != 0:
                raise RuntimeError(f"oracle tiles failed: {st}")
        return out

    def sage_b_tiles(self, pre, v, unit, tiles, causal, pv_fp32=True):
        """Query tiles `tiles` of one unit from prepass outputs `pre`; returns (N,d) with only those rows set."""
        v = _f32(v)
        n, d = v.shape[1:]
        out = np.zeros((n, d), np.float32)
        macs = np.zeros(2, np.uint64)
        for t in tiles:
            st = self.lib.orc_sage_b_tiles(np.ascontiguousarray(pre["qcodes"][unit]), np.ascontiguousarray(pre["qscales"][unit]),
                                           np.ascontiguousarray(pre["kcodes"][unit]), np.ascontiguousarray(pre["kscales"][unit]),
                                           np.ascontiguousarray(v[unit]), n, d, int(causal), int(pv_fp32), BLOCK_Q,
                                           BLOCK_KV, int(t), int(t) + 1, out, macs)
            if st != 0:
                raise RuntimeError(f"oracle tiles failed: {st}")
        return out

    def naive_rows(self, q, k, v, causal, r0, r1):
        """Exact binary64 attention rows [r0, r1) of ONE unit (q/k/v (N, d)); (r1 - r0, d) float64."""
        q, k, v = _f32(q), _f32(k), _f32(v)
        n, d = q.shape
        out = np.empty((r1 - r0, d), np.float64)
        self.lib.orc_naive_rows(q, k, v, n, d, int(causal), int(r0), int(r1), out)
        return out

    def naive(self, q, k, v, causal=False, threads=None):
        q, k, v = _f32(q), _f32(k), _f32(v)
        units, n, d = q.shape
        out = np.empty(q.shape, np.float64)
        self.lib.orc_naive(q, k, v, units, n, d, int(causal), threads or os.cpu_count() or 1, out)
        return out


class Reference:
    """The reference headers compiled where they lie (oracle/_ref/libsageref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            build()
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: the reference tree was never compiled here")
        lib = C.CDLL(path)
        lib.ref_last_message.restype = C.c_char_p
        lib.ref_round_to_half.restype = C.c_uint16
        lib.ref_round_to_half.argtypes = [C.c_double]
        lib.ref_snap_to_half.restype = C.c_double
        lib.ref_snap_to_half.argtypes = [C.c_double]
        lib.ref_smooth_k.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_int, _f32p, _f32p]
        lib.ref_quantize_q.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _i8p, _f32p]
        lib.ref_quantize_k.argtypes = [_f32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _i8p, _f32p]
        lib.ref_int8_tile.argtypes = [_i8p, _i8p] + [C.c_int] * 6 + [_i32p]
        lib.ref_int8_matmul.argtypes = [_i8p, _i8p, C.c_int, C.c_int, C.c_int, _i32p]
        lib.ref_fp16_matmul.argtypes = [_f64p, _f64p, C.c_int, C.c_int, C.c_int, _f64p]
        lib.ref_causal_tile.argtypes = [C.c_int] * 5
        lib.ref_sage_attention.argtypes = [_f32p, _f32p, _f32p] + [C.c_int] * 9 + [_f32p, _u64p]
        lib.ref_sage_attention_mt.argtypes = [_f32p, _f32p, _f32p] + [C.c_int] * 7 + [_f32p]
        lib.ref_naive_attention.argtypes = [_f32p, _f32p, _f32p] + [C.c_int] * 5 + [_f64p]
        lib.ref_sage_b_tiles.argtypes = [_f32p, _f32p, _f32p, C.c_int, C.c_int, C.c_int, C.c_int, _intp, C.c_int,
                                         _f32p]
        lib.ref_quantize_qk_per_token.argtypes = [_f32p, _f32p] + [C.c_int] * 5 + [_i8p, _f32p, _i8p, _f32p]
        lib.ref_sage_attention_variant.argtypes = [_f32p, _f32p, _f32p] + [C.c_int] * 8 + [_f32p]
        lib.ref_static_scale_counts.argtypes = [_f32p, _f32p, _f32p] + [C.c_int] * 6 + [_u64p]
        lib.ref_quantize_per_channel.argtypes = [_f32p, C.c_int, C.c_int, _i8p, _f32p]
        self.lib = lib

    def _raise(self, st):
        msg = self.lib.ref_last_message().decode()
        if st == 1:
            raise ValueError(msg)
        if st == 3:
            raise OverflowError(msg)
        raise RuntimeError(f"reference status {st}: {msg}")

    def round_to_half_bits(self, x):
        return self.lib.ref_round_to_half(float(x))

    def snap_to_half(self, x):
        return self.lib.ref_snap_to_half(float(x))

    def smooth_k(self, k4):
        k4 = _f32(k4)
        b, h, n, d = k4.shape
        ks = np.empty_like(k4)
        mean = np.empty((b, h, d), np.float32)
        st = self.lib.ref_smooth_k(k4, b, h, n, d, ks, mean)
        if st:
            self._raise(st)
        return ks, mean

    def quantize_q(self, q4, block_q=BLOCK_Q):
        q4 = _f32(q4)
        b, h, n, d = q4.shape
        codes = np.empty(q4.shape, np.int8)
        scales = np.empty((b * h, -(-n // block_q)), np.float32)
        st = self.lib.ref_quantize_q(q4, b, h, n, d, block_q, codes, scales)
        if st:
            self._raise(st)
        return codes, scales

    def quantize_k(self, k4, smooth=True, block_kv=BLOCK_KV):
        k4 = _f32(k4)
        b, h, n, d = k4.shape
        codes = np.empty(k4.shape, np.int8)
        scales = np.empty((b * h, -(-n // block_kv)), np.float32)
        st = self.lib.ref_quantize_k(k4, b, h, n, d, block_kv, int(smooth), codes, scales)
        if st:
            self._raise(st)
        return codes, scales

    def quantize_per_token(self, q4, k4, smooth=True):
        """Variant T prepass: (qcodes, qscales[units][N], kcodes, kscales[units][N])."""
        q4, k4 = _f32(q4), _f32(k4)
        b, h, n, d = q4.shape
        qc, kc = np.empty(q4.shape, np.int8), np.empty(k4.shape, np.int8)
        qs, ks = np.empty((b * h, n), np.float32), np.empty((b * h, n), np.float32)
        st = self.lib.ref_quantize_qk_per_token(q4, k4, b, h, n, d, int(smooth), qc, qs, kc, ks)
        if st:
            self._raise(st)
        return qc, qs, kc, ks

    def sage_attention_variant(self, q4, k4, v4, variant="T", causal=False, smooth=True, pv_fp32=False):
        """sageattn::sage_attention(in, SageVariant::T|B|VT|VB, opts)."""
        q4, k4, v4 = _f32(q4), _f32(k4), _f32(v4)
        b, h, n, d = q4.shape
        out = np.empty_like(q4)
        code = {"T": 0, "B": 1, "VT": 2, "VB": 3}[variant]
        st = self.lib.ref_sage_attention_variant(q4, k4, v4, b, h, n, d, int(causal), code,
                                                 int(smooth), int(pv_fp32), out)
        if st:
            self._raise(st)
        return out

    def static_scale_counts(self, q4, k4, v4, causal=False, per_token=False):
        """SageDiagnostics static-scale counters of sage_attention(in, VB|VT) (attention.hpp:479-488):
        (elements, first-block mismatches, later-block mismatches)."""
        q4, k4, v4 = _f32(q4), _f32(k4), _f32(v4)
        b, h, n, d = q4.shape
        out = np.zeros(3, np.uint64)
        st = self.lib.ref_static_scale_counts(q4, k4, v4, b, h, n, d, int(causal), int(per_token), out)
        if st:
            self._raise(st)
        return tuple(int(x) for x in out)

    def quantize_per_channel(self, a):
        """quantize(a, Granularity::per_channel(), Int8): (codes (rows, cols), scales (cols,))."""
        a = _f32(a)
        rows, cols = a.shape
        codes = np.empty((rows, cols), np.int8)
        scales = np.empty(cols, np.float32)
        st = self.lib.ref_quantize_per_channel(a, rows, cols, codes, scales)
        if st:
            self._raise(st)
        return codes, scales

    def int8_tile(self, qc, kc, r0, bq, c0, bkv):
        n, d = qc.shape
        out = np.empty((bq, bkv), np.int32)
        self.lib.ref_int8_tile(np.ascontiguousarray(qc), np.ascontiguousarray(kc), n, d, r0, bq, c0, bkv, out)
        return out

    def int8_matmul(self, a, b):
        a, b = np.ascontiguousarray(a, np.int8), np.ascontiguousarray(b, np.int8)
        out = np.empty((a.shape[0], b.shape[1]), np.int32)
        st = self.lib.ref_int8_matmul(a, b, a.shape[0], a.shape[1], b.shape[1], out)
        if st:
            self._raise(st)
        return out

    def fp16_matmul(self, a, b):
        a, b = np.ascontiguousarray(a, np.float64), np.ascontiguousarray(b, np.float64)
        out = np.empty((a.shape[0], b.shape[1]), np.float64)
        st = self.lib.ref_fp16_matmul(a, b, a.shape[0], a.shape[1], b.shape[1], out)
        if st:
            self._raise(st)
        return out

    def causal_tile(self, i, j, bq, bkv, n):
        r = self.lib.ref_causal_tile(i, j, bq, bkv, n)
        if r < 0:
            self._raise(1)
        return r

    def sage_attention(self, q4, k4, v4, causal=False, smooth=True, pv_fp32=False, block_q=BLOCK_Q,
                       block_kv=BLOCK_KV):
        """sageattn::sage_attention(in, B config, opts); returns (out, macs)."""
        q4, k4, v4 = _f32(q4), _f32(k4), _f32(v4)
        b, h, n, d = q4.shape
        out = np.empty_like(q4)
        macs = np.zeros(2, np.uint64)
        st = self.lib.ref_sage_attention(q4, k4, v4, b, h, n, d, int(causal), block_q, block_kv, int(smooth),
                                         int(pv_fp32), out, macs)
        if st:
            self._raise(st)
        return out, macs

    def sage_attention_mt(self, q, k, v, causal=False, smooth=True, pv_fp32=False, threads=None):
        q, k, v = _f32(q), _f32(k), _f32(v)
        units, n, d = q.shape
        out = np.empty_like(q)
        st = self.lib.ref_sage_attention_mt(q, k, v, units, n, d, int(causal), int(smooth), int(pv_fp32),
                                            threads or os.cpu_count() or 1, out)
        if st:
            self._raise(st)
        return out

    def naive_attention(self, q4, k4, v4, causal=False):
        q4, k4, v4 = _f32(q4), _f32(k4), _f32(v4)
        b, h, n, d = q4.shape
        out = np.empty(q4.shape, np.float64)
        st = self.lib.ref_naive_attention(q4, k4, v4, b, h, n, d, int(causal), out)
        if st:
            self._raise(st)
        return out

    def sage_b_tiles(self, q, k, v, tiles, causal=False, pv_fp32=False):
        """Rows of query tiles `tiles` of ONE unit (q/k/v are (N,d)), from the reference's building blocks."""
        q, k, v = _f32(q), _f32(k), _f32(v)
        n, d = q.shape
        out = np.zeros((n, d), np.float32)
        t = np.ascontiguousarray(tiles, np.int32)
        st = self.lib.ref_sage_b_tiles(q, k, v, n, d, int(causal), int(pv_fp32), t, len(t), out)
        if st:
            self._raise(st)
        return out

    def sage_b_tiles_parallel(self, q, k, v, tile_lists, causal=False, pv_fp32=False):
        """Runs one ref_sage_b_tiles call per host thread (ctypes drops the GIL)."""
        outs = [None] * len(tile_lists)

        def work(i):
            outs[i] = self.sage_b_tiles(q, k, v, tile_lists[i], causal, pv_fp32)

        th = [threading.Thread(target=work, args=(i,)) for i in range(len(tile_lists))]
        for t in th:
            t.start()
        for t in th:
            t.join()
        return outs


# -- binary64 accuracy metrics -------------------------------

def cosine_sim(o, r):
    o, r = np.asarray(o, np.float64).ravel(), np.asarray(r, np.float64).ravel()
    den = np.sqrt((o * o).sum()) * np.sqrt((r * r).sum())
    return 0.0 if den == 0 else float((o * r).sum() / den)


def relative_l1(o, r):
    """sum|o - r| / sum|r| with r the reference."""
    o, r = np.asarray(o, np.float64).ravel(), np.asarray(r, np.float64).ravel()
    return float(np.abs(o - r).sum() / np.abs(r).sum())


def rmse(o, r):
    o, r = np.asarray(o, np.float64).ravel(), np.asarray(r, np.float64).ravel()
    return float(np.sqrt(((o - r) ** 2).mean()))
