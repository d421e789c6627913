"""Multi-rank host logic on CPU (gloo, world size 2): window sharding, per-rank generation and
the stats allreduce. The per-rank plans come from the CPU oracle here (no GPU); on B200 the same
flow runs the CUDA path and NCCL (bench.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2207_00172_b200.shard import shard_ranges, work_per_window


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, per_rank, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # weak scaling as in bench.py: rank r owns windows [r * per_rank, (r + 1) * per_rank)
    wl = synth.make_config(2, window_offset=rank * per_rank, num_windows=per_rank)
    out = oracle.run(wl, threads=1)
    stats = torch.from_numpy(out["stats"].copy())
    dist.all_reduce(stats)
    # max over ranks of a per-rank "time" (the bench reports the slowest rank)
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        q.put((stats.numpy().copy(), float(t.item())))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_stats_allreduce_equals_single_run():
    world, per_rank = 2, 24
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, per_rank, q)) for r in range(world)]
    for p in procs:
        p.start()
    stats, tmax = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    whole = oracle.run(synth.make_config(2, num_windows=world * per_rank), threads=2)
    np.testing.assert_array_equal(stats, whole["stats"])
    assert tmax == 2.0


def test_shard_ranges_cover_and_balance():
    wl = synth.make_config(5, num_windows=4000)
    work = work_per_window(wl.num_frames, wl.budget, wl.num_exits)
    for world in (1, 2, 3, 4, 8):
        rs = shard_ranges(work, world)
        assert len(rs) == world and rs[0][0] == 0 and rs[-1][1] == len(work)
        for (a, b), (c, d) in zip(rs, rs[1:]):
            assert b == c and a <= b
        per = [work[a:b].sum() for a, b in rs]
        assert max(per) <= work.sum() / world + work.max()      # within one window of ideal


def test_shard_ranges_edge_cases():
    assert shard_ranges([], 4) == [(0, 0)] * 4
    assert shard_ranges([5, 5, 5, 5], 2) == [(0, 2), (2, 4)]
    assert shard_ranges([0, 0, 0], 3) == [(0, 1), (1, 2), (2, 3)]
    assert shard_ranges([1], 4)[0] == (0, 1) or sum(b - a for a, b in shard_ranges([1], 4)) == 1


def test_rank_shards_regenerate_identically():
    """A rank's shard generated alone equals the same windows of the whole batch (no scatter)."""
    whole = synth.make_config(3, num_windows=40)
    part = synth.make_config(3, window_offset=16, num_windows=8)
    np.testing.assert_array_equal(part.class_id, whole.subset(16, 24).class_id)


def _strong_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    # strong scaling as in bench.py --scaling strong: the config's whole window set, work-balanced
    wl = bench.make_workload("c2", rank, world, "strong")
    out = oracle.run(wl, threads=1)
    stats = torch.from_numpy(out["stats"].copy())
    dist.all_reduce(stats)
    n = torch.tensor([wl.num_windows, wl.total_cells], dtype=torch.int64)
    dist.all_reduce(n)
    if rank == 0:
        q.put((stats.numpy().copy(), n.tolist()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_strong_scaling_split_covers_config():
    """bench.py --scaling strong on 2 ranks: the shards partition config c2's 1024 windows, and the
    allreduced statistics equal a single run over the whole config."""
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_strong_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    stats, n = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    whole = synth.make_config(2)
    assert n == [whole.num_windows, whole.total_cells]
    np.testing.assert_array_equal(stats, oracle.run(whole, threads=4)["stats"])
