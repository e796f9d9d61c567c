"""Multi-process sharding on CPU (gloo, world_size 2).

Each rank takes its contiguous series range (sharding.shard_range), runs the
chain with series_offset = its first global row, and the gathered shards must
equal the single-process result bit for bit -- the property the multi-GPU
bench relies on.  The per-rank compute here is the CPU oracle (no GPU in this
container); on GPUs the same offsets go to Pipeline.run_device.
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench_inputs
        from oracle import oracle as O
        from paper_2601_03159_b200.sharding import shard_range

        pipe = bench_inputs.pipeline(5)
        x = bench_inputs.host_input(2, n=37)[:, :256].copy()
        lo, hi = shard_range(x.shape[0], rank, world)
        part = O.run_pipeline(pipe, x[lo:hi], series_offset=lo)
        parts = [None] * world
        dist.all_gather_object(parts, part)
        if rank == 0:
            np.save(out_path, np.concatenate(parts))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_sharding_is_bitwise(tmp_path):
    import bench_inputs
    from oracle import oracle as O

    out = str(tmp_path / "gathered.npy")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    x = bench_inputs.host_input(2, n=37)[:, :256].copy()
    full = O.run_pipeline(bench_inputs.pipeline(5), x)
    assert np.array_equal(np.load(out), full)


def test_shard_range_partitions():
    from paper_2601_03159_b200.sharding import shard_range

    for n in (0, 1, 7, 1000, 1_000_000):
        for world in (1, 2, 3, 8):
            ranges = [shard_range(n, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            assert max(b - a for a, b in ranges) - min(b - a for a, b in ranges) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)
