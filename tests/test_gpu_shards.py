"""Multi-GPU readiness on one GPU: windows are independent
("safe to run concurrently on distinct instances"), so the 2/4/8-rank
split of a config -- contiguous work-balanced ranges from shard.py, exactly what bench.py's
--scaling strong gives each rank -- run shard after shard through the CUDA path must reproduce
the unsharded run bit for bit, and the per-shard statistics vectors must sum (the NCCL allreduce
of a6) to the oracle's. Runs the shards one after another on one GPU (no kernel waits on another
rank, B200_PROFILING.md)."""
import numpy as np
import pytest

import synth
from paper_2207_00172_b200.shard import shard_ranges, work_per_window
from tests.parity import compare, gpu_run, oracle_run

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2207_00172_b200 import build, turbo
    build.build()
    turbo.load()


@pytest.fixture(scope="module")
def c5_whole():
    wl = synth.make_config(5, num_windows=4096)
    want = oracle_run(wl)
    got = gpu_run(wl, "all", 0)
    del got["batch"]
    compare(wl, got, want, check_options=False)
    return wl, want, got


@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_plans_equal_unsharded(c5_whole, world):
    wl, want, whole = c5_whole
    ranges = shard_ranges(work_per_window(wl.num_frames, wl.budget, wl.num_exits), world)
    assert ranges[0][0] == 0 and ranges[-1][1] == wl.num_windows
    stats = np.zeros(181, dtype=np.int64)
    ff = wl.first_frame
    for lo, hi in ranges:
        # the rank's shard regenerated from (seed, window id) alone, as each rank does
        part = synth.make_config(5, window_offset=lo, num_windows=hi - lo)
        got = gpu_run(part, "all", 0)
        f0 = int(ff[lo]) if lo < wl.num_windows else wl.total_frames
        f1 = int(ff[hi]) if hi < wl.num_windows else wl.total_frames
        np.testing.assert_array_equal(got["exits"], whole["exits"][f0:f1])
        for k in ("best_gain", "best_cost", "feasible", "budget"):
            np.testing.assert_array_equal(got[k], whole[k][lo:hi])
        assert int(got["status"][0]) == -1 and int(got["status"][1]) == -1
        stats += got["stats"].astype(np.int64)
    np.testing.assert_array_equal(stats, want["stats"])          # = the allreduced a6 vector
    np.testing.assert_array_equal(stats, whole["stats"])


@pytest.mark.parametrize("world", [2, 8])
def test_sharded_config3_stats(world):
    """c3-shaped (uniform windows): equal shards, summed statistics = the oracle's."""
    wl = synth.make_config(3, num_windows=512)
    ranges = shard_ranges(work_per_window(wl.num_frames, wl.budget, wl.num_exits), world)
    assert all(hi - lo == 512 // world for lo, hi in ranges)
    stats = np.zeros(181, dtype=np.int64)
    for lo, hi in ranges:
        part = synth.make_config(3, window_offset=lo, num_windows=hi - lo)
        got = gpu_run(part, "all", 0)
        compare(part, got, oracle_run(part), check_options=False)
        stats += got["stats"].astype(np.int64)
    np.testing.assert_array_equal(stats, oracle_run(wl)["stats"])
