"""Long windows (rows > TURBO_BIG_CELLS cells): the cluster kernel (rows up to TURBO_CLUSTER_CELLS,
one thread-block cluster per window, dp_cluster.cu) and the cooperative grid kernel (longer rows,
and every long row with variant 512), bit-exact against the oracle; mixed batches (routing
between the CTA, cluster and grid kernels) and config c4 at full size (3000 frames, B = 2^20)."""
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


# 0: long rows up to TURBO_CLUSTER_CELLS on the cluster kernel; 512: every long row on the grid kernel
LONG = [0, 512]
LONG_IDS = ["cluster", "grid"]


@pytest.mark.parametrize("variant", LONG, ids=LONG_IDS)
@pytest.mark.parametrize("fused", [True, False, "all"], ids=["solve", "plan+backtrack", "schedule"])
def test_long_window_paper_profile(fused, variant):
    wl = synth.make_long_window(3, N=120, K=6, B=40000)
    compare(wl, gpu_run(wl, fused, variant), oracle_run(wl), check_options=fused != "all")


@pytest.mark.parametrize("variant", LONG, ids=LONG_IDS)
@pytest.mark.parametrize("K", [2, 3, 4, 5, 6, 7, 8, 11, 16])
def test_long_window_random_rows(K, variant):
    """Random (non-monotone, negative) gains, costs up to 700, ragged top tile; N not a multiple
    of the backtrack's frames per round (tail rounds)."""
    wl = synth.make_long_window(10 + K, N=90 + K % 5, K=K, B=30001 + 37 * K, c_max=700, random_rows=True)
    compare(wl, gpu_run(wl, True, variant), oracle_run(wl))


@pytest.mark.parametrize("variant", LONG, ids=LONG_IDS)
def test_mixed_batch_routes_small_and_long_windows(variant):
    parts = [synth.make_config(2, num_windows=40), synth.make_long_window(5, N=64, K=5, B=50000),
             synth.make_config(1), synth.make_long_window(6, N=40, K=5, B=26000, c_max=3000)]
    for p in parts:
        p.base_cost = 84
        p.capacity = (p.budget.astype(np.int64) + p.num_frames.astype(np.int64) * 84).astype(np.int32)
    wl = synth.concat_workloads(parts)
    for fused in (True, False):
        compare(wl, gpu_run(wl, fused, variant), oracle_run(wl))
    # turbo_schedule: the long windows go to the cluster / grid kernel with a1/a2/a6 fused into it
    compare(wl, gpu_run(wl, "all", variant), oracle_run(wl), check_options=False)


@pytest.mark.parametrize("variant", LONG, ids=LONG_IDS)
@pytest.mark.parametrize("fused", [True, False, "all"], ids=["solve", "plan+backtrack", "schedule"])
def test_long_windows_a1_edges(fused, variant):
    """a1 on long windows: clamped (budget 0), under-bound and exact-fit capacities."""
    parts = [synth.make_long_window(40 + s, N=20 + 7 * s, K=4 + s, B=30000 + 999 * s, c_max=600, random_rows=True)
             for s in range(6)]
    wl = synth.with_budget_edges(synth.concat_workloads(parts), seed=3)
    want = oracle_run(wl)
    assert (want["budget"] < wl.budget).any()
    compare(wl, gpu_run(wl, fused, variant), want, check_options=fused != "all")


@pytest.mark.parametrize("fused", [True, "all"], ids=["lookup+solve+stats", "schedule"])
def test_graph_replay_with_changed_inputs(fused):
    """A captured graph replayed with NEW class ids must plan the new inputs (the halo
    ring tags continue on the device across replays, so a slot of an earlier replay is never taken
    for the current one). Short long windows (N <= 2 x ring depth) are the exposed case."""
    import dataclasses
    import torch
    from paper_2207_00172_b200 import turbo
    parts = [synth.make_long_window(70 + s, N=6 + 3 * s, K=5, B=28000 + 500 * s, c_max=900, random_rows=True)
             for s in range(4)]
    wl = synth.concat_workloads(parts)
    variants = [wl]
    for v in range(1, 3):
        rng = np.random.default_rng(v)
        variants.append(dataclasses.replace(wl, class_id=rng.integers(0, 10, wl.total_frames).astype(np.uint8)))
    b = turbo.batch_from_workload(wl)
    turbo.run_path(b, fused=fused)               # warm-up (kernel attributes) before capture
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        turbo.run_path(b, fused=fused)
    for rep in range(6):
        cur = variants[rep % 3]
        b.class_id[: cur.total_frames].copy_(torch.as_tensor(cur.class_id))
        g.replay()
        torch.cuda.synchronize()
        got = turbo.results(b)
        compare(cur, got, oracle_run(cur), check_options=fused != "all")


@pytest.mark.parametrize("variant", LONG, ids=LONG_IDS)
@pytest.mark.parametrize("fused", [True, False, "all"], ids=["solve", "plan+backtrack", "schedule"])
def test_long_window_costs_beyond_the_halo(fused, variant):
    """Option costs above the halo capacity (TURBO_BIG_MAX_COST cells) take the L2-row path
    (rows in global memory, a grid barrier per frame) -- planned exactly, no longer rejected
    (reading R17). The batch mixes such windows with halo-path windows, K fixed and mixed."""
    parts = [synth.make_long_window(7, N=30, K=4, B=30000, c_max=5000),
             synth.make_long_window(8, N=41, K=6, B=60000, c_max=4097, random_rows=True),
             synth.make_long_window(9, N=25, K=5, B=40000, c_max=900, random_rows=True),
             synth.make_long_window(10, N=17, K=3, B=27000, c_max=26000, random_rows=True)]
    wl = synth.concat_workloads(parts)
    want = oracle_run(wl)
    got = gpu_run(wl, fused, variant)
    assert int(got["status"][1]) == -1
    compare(wl, got, want, check_options=fused != "all")


@pytest.mark.parametrize("fused", [True, False, "all"], ids=["solve", "plan+backtrack", "schedule"])
def test_cluster_kernel_edges(fused):
    """The cluster kernel at its edges, in ONE batch with grid-kernel rows: rows of exactly
    TURBO_CLUSTER_CELLS cells (8 CTAs of 16,384 cells) and one cell more (grid kernel), the smallest
    long row (24,577 cells), costs reaching several segments down and below cell 0, every segment
    size (4,096 / 8,192 / 16,384 cells), tie-heavy rows, and more long windows than clusters."""
    parts = [synth.make_long_window(81, N=9, K=5, B=131071, c_max=40000, random_rows=True),
             synth.make_long_window(82, N=7, K=4, B=131072, c_max=3000, random_rows=True),
             synth.make_long_window(83, N=33, K=6, B=24576, c_max=24000, random_rows=True),
             synth.make_long_window(84, N=21, K=3, B=65535, c_max=65000, random_rows=True),
             synth.make_long_window(85, N=12, K=8, B=32767, c_max=9000, random_rows=True),
             synth.make_long_window(86, N=0, K=5, B=40000, c_max=100),            # no frames
             synth.make_long_window(87, N=1, K=5, B=70000, c_max=69000, random_rows=True)]
    parts += [synth.make_long_window(90 + s, N=5 + s % 7, K=2 + s % 15, B=24577 + 2311 * s, c_max=50 + 97 * s,
                                     random_rows=s % 2 == 1) for s in range(40)]
    wl = synth.concat_workloads(parts)
    want = oracle_run(wl)
    got = gpu_run(wl, fused, 0)
    assert int(got["status"][1]) == -1
    compare(wl, got, want, check_options=fused != "all")


def test_config4_full_size():
    """c4 at full size: G*, C* and the whole exit vector against the oracle's full suffix table
    (25 GB of int64 on the host; skipped if the host lacks the memory)."""
    import psutil
    wl = synth.make_config(4)
    got = gpu_run(wl, True)
    assert int(got["status"][0]) == -1 and int(got["status"][1]) == -1
    og = got["opt_gain"][:3000 * 6].reshape(3000, 6)
    oc = got["opt_cost"][:3000 * 6].reshape(3000, 6)
    ex = got["exits"].astype(np.int64)
    assert og[np.arange(3000), ex].sum() == got["best_gain"][0]
    assert oc[np.arange(3000), ex].sum() == got["best_cost"][0] <= (1 << 20)
    if psutil.virtual_memory().available < 40 * 2**30:
        want = oracle_run(wl, mode="value")
        assert int(got["best_gain"][0]) == int(want["best_gain"][0])
        assert int(got["best_cost"][0]) == int(want["best_cost"][0])
        pytest.skip("host memory too small for the full oracle table; G*/C* checked")
    want = oracle_run(wl)
    compare(wl, got, want)
