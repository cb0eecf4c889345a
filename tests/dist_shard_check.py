"""Helper of tests/test_gpu_configs.py::test_two_rank_shards_equal_single_call, launched by
torchrun with 2 ranks on one GPU: each rank runs bench.py's step on its K3 shard
(sab_shard_plan, head x batch), the outputs are gathered over gloo, and rank 0
compares them with the one-call output.  Prints SHARDS EQUAL on success."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import torch
    import torch.distributed as dist

    from paper_2410_02367_b200 import _lib
    from gpu_helpers import _inputs, _run_as_benched

    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda:0")
    for units, n, d, causal in ((7, 1024, 128, True), (5, 777, 64, False)):
        first, count = _lib.shard_plan(units, world, rank)
        q, k, v = _inputs(count, n, d, dev, unit0=first)  # the shard, generated from global indices
        o, _ = _run_as_benched(q, k, v, causal)
        parts = [None] * world
        dist.all_gather_object(parts, (first, o.cpu()))
        if rank == 0:
            qa, ka, va = _inputs(units, n, d, dev)
            full, _ = _run_as_benched(qa, ka, va, causal)
            full = full.cpu()
            for f, part in parts:
                assert torch.equal(part, full[:, f:f + part.shape[1]]), (units, n, d, f)
    dist.barrier()
    if rank == 0:
        print("SHARDS EQUAL")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
