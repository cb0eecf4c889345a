"""CPU, world_size 2 over gloo: the K3 head x batch partition used by bench.py
under torchrun.  Each rank takes its contiguous shard of the B*H units
(sab_shard_plan), generates it with the global-index RNG and runs the CPU
oracle on it; the gathered shards equal the unsharded tensors and outputs
bit-for-bit -- no data-path collective is needed."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

B, H, N, D = 1, 5, 200, 64


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import Oracle
        from paper_2410_02367_b200 import _lib, synth

        first, count = _lib.shard_plan(B * H, world, rank)
        qs, ks, vs = synth.qkv(count, N, D, unit0=first, dtype=np.float32)
        out, _ = Oracle().sage_b(qs, ks, vs, causal=True, threads=1) if count else (np.zeros((0, N, D), np.float32), 0)
        gathered = [None] * world
        dist.all_gather_object(gathered, (first, count, qs, out))
        if rank == 0:
            q.put(gathered)
    finally:
        dist.destroy_process_group()


def test_head_shards_over_two_gloo_ranks():
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from oracle.oracle import Oracle
    from paper_2410_02367_b200 import synth

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    os.environ["PYTHONPATH"] = root + os.pathsep + os.environ.get("PYTHONPATH", "")
    for p in procs:
        p.start()
    gathered = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    qa, ka, va = synth.qkv(B * H, N, D, dtype=np.float32)
    whole, _ = Oracle().sage_b(qa, ka, va, causal=True)
    covered = []
    for first, count, qs, out in sorted(gathered, key=lambda g: g[0]):
        covered.extend(range(first, first + count))
        assert np.array_equal(qs, qa[first:first + count])
        assert np.array_equal(out.view(np.uint32), whole[first:first + count].view(np.uint32))
    assert covered == list(range(B * H))
