"""Shared helpers of the as-benched GPU parity tests (tests/test_gpu_configs.py) and their
subprocess helpers (tests/raster_check.py, tests/dist_shard_check.py): bench.py's synthetic
inputs and bench.py's K1 + K2 step through the C ABI."""


def _inputs(units, n, d, dev, unit0=0):
    from paper_2410_02367_b200 import synth

    return [synth.tensor_torch(s, (units, n, d), unit0, device=dev).reshape(1, units, n, d) for s in (1, 2, 3)]


def _run_as_benched(q, k, v, causal):
    """bench.py's step: sab_prepass + sab_attention on the same stream, fp16 O."""
    import ctypes

    import torch

    from paper_2410_02367_b200 import _lib, sageattn

    desc = sageattn.make_desc(q, causal, out_dtype=torch.float16)
    ws = sageattn.Workspace(desc, q.device)
    o = torch.empty_like(q)
    lib = _lib.load()
    sp = torch.cuda.current_stream(q.device).cuda_stream
    _lib.check(lib.sab_prepass(ctypes.byref(desc), q.data_ptr(), k.data_ptr(), None, ws.ptr, ws.nbytes, sp))
    _lib.check(lib.sab_attention(ctypes.byref(desc), ws.ptr, ws.nbytes, v.data_ptr(), o.data_ptr(), sp))
    torch.cuda.synchronize()
    _lib.check(sageattn.read_status(ws))
    return o, ws
