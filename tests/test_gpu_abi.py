"""C-ABI error behaviour on the device (status words, rejected windows, workspace checks)."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tb():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2207_00172_b200 import build, turbo
    build.build()
    turbo.load()
    return turbo


def _run(tb, wl, fused=True):
    import torch
    b = tb.batch_from_workload(wl)
    tb.run_path(b, fused=fused)
    torch.cuda.synchronize()
    return b, tb.results(b)


@pytest.mark.parametrize("fused", [True, False])
def test_bad_class_sets_status0(tb, fused):
    wl = synth.make_config(2, num_windows=8)
    wl.class_id[45] = 200            # C = 10
    wl.class_id[100] = 11
    b, r = _run(tb, wl, fused)
    assert int(r["status"][0]) == 45
    assert int(r["status"][1]) == -1
    # the bad frame's option row is zero (same rule as the oracle's lookup)
    fo = r["first_option"]
    assert (r["opt_gain"][fo[1] + 15 * 5: fo[1] + 16 * 5] == 0).all()


@pytest.mark.parametrize("fused", [True, False])
def test_negative_cost_rejects_window(tb, fused):
    gain = np.tile(np.array([0, 5, 9], np.int32), 2)
    cost = np.array([0, 2, 4, 0, -1, 3], np.int32)
    wl = synth.Workload("neg", [gain], [cost], [(2, 3)], np.array([4, 3, 2], np.int32), np.array([5, 5, 5], np.int32),
                        np.array([5, 5, 5], np.int32), 0, np.array([0, 0, 0], np.int32),
                        np.array([0, 0, 0, 0, 0, 1, 0, 0, 1], np.uint8))
    b, r = _run(tb, wl, fused)
    assert int(r["status"][1]) == 1          # window 1 holds class 1 (cost -1)
    assert r["feasible"].tolist()[1] == 0 and r["best_gain"][1] == 0 and r["best_cost"][1] == 0
    assert r["exits"][4:7].tolist() == [0, 0, 0]
    assert r["feasible"][0] == 1


def test_gain_range_rule(tb):
    big = 1 << 24
    gain = np.array([0, big], np.int32)
    cost = np.array([0, 1], np.int32)
    wl = synth.Workload("range", [gain], [cost], [(1, 2)], np.array([2, 1], np.int32), np.array([2, 2], np.int32),
                        np.array([2, 2], np.int32), 0, np.array([0, 0], np.int32), np.zeros(3, np.uint8))
    b, r = _run(tb, wl)
    # window 0: sum max|g| = 2^25 -> rejected; window 1: 2^24 < 2^25 -> planned
    assert int(r["status"][1]) == 0
    assert r["feasible"].tolist() == [0, 1]
    assert int(r["best_gain"][1]) == big


def test_budget_above_bound_rejected(tb):
    import torch
    wl = synth.make_config(1)
    b = tb.batch_from_workload(wl)
    b.capacity.add_(5)               # a1 now derives budget 125 > layout bound 120
    tb.run_path(b)
    torch.cuda.synchronize()
    r = tb.results(b)
    assert int(r["status"][1]) == 0 and r["feasible"][0] == 0


def test_workspace_too_small(tb):
    import torch
    wl = synth.make_config(2, num_windows=4)
    b = tb.batch_from_workload(wl)
    small = torch.empty(16, dtype=torch.uint8, device="cuda")
    with pytest.raises(tb.TurboError) as ei:
        tb.mckp_plan(b.shape, b.windows_dev, b.opt_gain, b.opt_cost, small, b.best_gain, b.best_cost,
                     b.feasible, b.status)
    assert ei.value.code == 3
    with pytest.raises(tb.TurboError) as ei:
        tb.backtrack(b.shape, b.windows_dev, b.opt_cost, small, b.best_cost, b.feasible, b.exit_out)
    assert ei.value.code == 3


def test_misaligned_option_buffer(tb):
    wl = synth.make_config(1)
    b = tb.batch_from_workload(wl)
    with pytest.raises(tb.TurboError) as ei:
        tb.profile_lookup(b.shape, b.profiles_dev, b.windows_dev, b.class_id, b.capacity, b.base_cost,
                          b.opt_gain[1:], b.opt_cost, b.status)
    assert ei.value.code == 1


def test_stream_ordering_nondefault_stream(tb):
    import torch
    wl = synth.make_config(2, num_windows=64)
    b = tb.batch_from_workload(wl)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        tb.run_path(b, stream=s)
    s.synchronize()
    r = tb.results(b)
    import oracle
    want = oracle.run(wl)
    np.testing.assert_array_equal(r["exits"], want["exits"])


def test_launch_count_counts_the_kernels_of_a_call(tb):
    """turbo_launch_count: one fused launch for a batch whose planes stay on chip (c2 shape);
    DP + plane walk when the planes go to HBM (c3 shape); lookup + solve + stats on that path."""
    import torch
    for cfg, n, expect_sched in ((2, 16, 1), (3, 8, 2)):
        b = tb.batch_from_workload(synth.make_config(cfg, num_windows=n))
        c0 = tb.launch_count()
        tb.run_path(b, fused="all")
        torch.cuda.synchronize()
        assert tb.launch_count() - c0 == expect_sched
        c0 = tb.launch_count()
        tb.run_path(b, fused=True)
        torch.cuda.synchronize()
        assert tb.launch_count() - c0 == 2 + expect_sched
