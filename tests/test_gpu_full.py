"""GPU parity on EVERY window of the large configs, and on every branch of a1.

North star: "bit-exact plans vs the CPU oracle on all configs" (§5.2; tie-break
SPEC.md:275, reading R7). Compared element by element: exits, G*, C*, feasible, the a1 budget
written back, and the a6 statistics vector.

* c3: all 65,536 windows (300 frames, K = 8, B = 4096), as the eight 8,192-window shards the
  8-GPU run gives each rank, run one after another through turbo_schedule (the path bench.py
  times) on one GPU; the oracle runs on all host cores.
* c5: all 16,384 windows of the mixed sweep (K 2-16, B 64-16384, N 30-300) through
  turbo_schedule, the lookup + solve path and the plan + backtrack path.
* a1 (§3, reading R3): capacities that clamp the budget to 0 (including negative
  capacities), device budgets below the layout bound, the exact fit; and capacity = NULL, where
  the path plans the budgets the caller wrote into the device windows.
"""
import numpy as np
import pytest

import synth
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


def _free_cuda():
    import gc
    import torch
    gc.collect()
    torch.cuda.empty_cache()


@pytest.mark.parametrize("shard", range(8))
def test_config3_every_window(shard):
    """c3 shard `shard` of 8 (windows [8192 s, 8192 (s+1))): all 8,192 windows bit-exact."""
    wl = synth.make_config(3, window_offset=8192 * shard, num_windows=8192)
    got = gpu_run(wl, "all", 0)
    del got["batch"]
    _free_cuda()
    want = oracle_run(wl)
    compare(wl, got, want, check_options=False)


@pytest.fixture(scope="module")
def c5_full():
    wl = synth.make_config(5)
    assert wl.num_windows == 16384
    return wl, oracle_run(wl)


@pytest.mark.parametrize("fused", ["all", True, False], ids=["schedule", "solve", "plan+backtrack"])
def test_config5_every_window(c5_full, fused):
    wl, want = c5_full
    got = gpu_run(wl, fused, 0)
    del got["batch"]
    _free_cuda()
    compare(wl, got, want, check_options=fused != "all")


EDGE_CASES = {
    "c2": lambda: synth.make_config(2),
    "c5": lambda: synth.make_config(5, num_windows=512),
    "tie": lambda: synth.make_tie_heavy(seed=303, W=2000, max_frames=40, max_exits=16, max_budget=900),
    "c3": lambda: synth.make_config(3, num_windows=256),
    # long windows (grid kernel: halo path and L2-row path) next to short ones
    "long": lambda: synth.concat_workloads([synth.make_config(2, num_windows=8),
                                            synth.make_long_window(51, N=33, K=6, B=40000),
                                            synth.make_long_window(52, N=21, K=4, B=30000, c_max=6000,
                                                                   random_rows=True)]),
}
# variant 256: the 64-register kernels also for <= 4-warp launches (the default takes the 72-register
# instantiations of dp_small.cu there)
EDGE_PATHS = [("all", 0), (True, 0), (False, 0), (True, 1), (True, 2), ("all", 2), ("all", 256), (True, 256)]
EDGE_IDS = ["schedule", "solve", "plan+backtrack", "solve-smem", "solve-hbm", "schedule-hbm", "schedule-r64",
            "solve-r64"]


@pytest.mark.parametrize("case", sorted(EDGE_CASES))
@pytest.mark.parametrize("fused,variant", EDGE_PATHS, ids=EDGE_IDS)
def test_a1_clamp_and_under_bound(case, fused, variant):
    """Capacities below N u0 (a1 clamps to 0), negative capacities, budgets below the layout bound."""
    wl = synth.with_budget_edges(EDGE_CASES[case](), seed=17)
    want = oracle_run(wl)
    b = want["budget"].astype(np.int64)
    assert (b == 0).any() and ((b > 0) & (b < wl.budget)).any(), "edge generator must hit both branches"
    compare(wl, gpu_run(wl, fused, variant), want, check_options=fused != "all")


@pytest.mark.parametrize("case", sorted(EDGE_CASES))
@pytest.mark.parametrize("fused,variant", EDGE_PATHS, ids=EDGE_IDS)
def test_null_capacity_device_budgets(case, fused, variant):
    """capacity = NULL: turbo_profile_lookup / turbo_schedule leave a1 out and the DP plans the
    budgets stored in the device windows -- here random values in [0, bound], so most are
    below the layout bound the workspace was sized for."""
    wl = EDGE_CASES[case]()
    rng = np.random.default_rng(5)
    bud = np.floor(rng.random(wl.num_windows) * (wl.budget.astype(np.int64) + 1)).astype(np.int32)
    bud[::7] = 0
    bud[1::7] = wl.budget[1::7]
    want = oracle_run(wl, budgets=bud)
    compare(wl, gpu_run(wl, fused, variant, device_budgets=bud), want, check_options=fused != "all")


def test_device_budget_above_bound_rejected():
    """A device budget above the sizing bound rejects the window (reading R15): all-zero plan,
    G* = C* = 0, feasible = 0, status[1] = the smallest such window."""
    wl = synth.make_config(2, num_windows=64)
    bud = wl.budget.copy()
    bud[9] = wl.budget[9] + 1
    bud[40] = wl.budget[40] + 500
    for fused in ("all", True, False):
        got = gpu_run(wl, fused, 0, device_budgets=bud)
        assert int(got["status"][1]) == 9
        for w in (9, 40):
            assert got["feasible"][w] == 0 and got["best_gain"][w] == 0 and got["best_cost"][w] == 0
            assert (got["exits"][30 * w: 30 * w + 30] == 0).all()
        keep = np.setdiff1d(np.arange(64), [9, 40])
        want = oracle_run(wl, budgets=bud)
        for k in ("best_gain", "best_cost", "feasible"):
            np.testing.assert_array_equal(got[k][keep].astype(np.int64), want[k][keep].astype(np.int64))


# ---------------------------------------------------------------------------------------------
# The lockstep multi-window kernel (dp_pack.cu) serves single-class fixed-K batches with >= 2
# windows per SM when variant bit 8 is set (opt-in). These sets give it windows of DIFFERENT N and B
# inside one CTA, tie-heavy rows, infeasible windows, clamped budgets and bad class ids; variant 0
# runs the one-window-per-CTA kernel on the same inputs.
PACK_K = [4, 5, 6, 8]


def _pack_set(K, seed):
    """Budget bounds in [256, 1000] keep every window in one row-size class (the kernel's domain);
    the a1 edges then lower (or clamp) the device budgets below those bounds."""
    wl = synth.make_tie_heavy(seed=seed, W=1500, max_frames=40, max_exits=K, fixed_exits=K, max_budget=1000,
                              max_cost=150)
    wl.budget = (256 + wl.budget.astype(np.int64) % 745).astype(np.int32)
    wl.capacity = (wl.budget.astype(np.int64) + wl.num_frames.astype(np.int64) * wl.base_cost).astype(np.int32)
    return synth.with_budget_edges(wl, seed=seed + 1)


@pytest.mark.parametrize("K", PACK_K)
@pytest.mark.parametrize("fused", ["all", True], ids=["schedule", "solve"])
def test_lockstep_kernel_mixed_windows(K, fused):
    wl = _pack_set(K, 500 + K)
    want = oracle_run(wl)
    compare(wl, gpu_run(wl, fused, 0), want, check_options=fused != "all")
    compare(wl, gpu_run(wl, fused, 8), want, check_options=fused != "all")


def test_lockstep_kernel_bad_class_and_range():
    wl = _pack_set(5, 77)
    wl.class_id[1234] = 200
    wl.class_id[99] = 10
    a = gpu_run(wl, "all", 0)
    c = gpu_run(wl, "all", 8)
    assert int(a["status"][0]) == 99 and int(c["status"][0]) == 99
    for k in ("exits", "best_gain", "best_cost", "feasible", "stats", "budget"):
        np.testing.assert_array_equal(a[k], c[k])


# The runtime-K kernel (dp_gen.cu) serves the mixed-K plan-mode launches of row classes 0-2 by
# default (72-register instantiation for <= 4 warps per window; variant 256: the 64-register one);
# variant 16 extends it to the longest-row class, variant 32 turns it off (fifteen K-specific
# bodies). Every combination must give the same bits as the oracle.
@pytest.mark.parametrize("variant", [0, 16, 32, 256])
@pytest.mark.parametrize("fused", ["all", True, False], ids=["schedule", "solve", "plan+backtrack"])
def test_runtime_k_body(variant, fused):
    tie = synth.make_tie_heavy(seed=909, W=600, max_frames=60, max_exits=16, max_budget=6000, max_cost=40,
                               base_cost=84)
    wl = synth.with_budget_edges(synth.concat_workloads([synth.make_config(5, num_windows=700), tie]), seed=4)
    want = oracle_run(wl)
    compare(wl, gpu_run(wl, fused, variant), want, check_options=fused != "all")
