"""NEXT-4 on the GPU (turbo_batched_plan) against the batched oracle: bit-exact exits, G*, C*
and feasibility on random supermodular sets (K = 2..16, infeasible windows), the b1/b2
workloads, gains WITHOUT R19 (the general program, reading R20; with a workspace), the general
program forced on R19 windows (variant 64: must equal the canonical plans), and the error paths
(R19 violation without a workspace, bad class id, unsupported sizes)."""
import numpy as np
import pytest

import oracle
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


def _gpu(tb, wl, workspace=True, variant=0):
    import torch
    b = tb.make_batch(wl.profiles_gain, wl.profiles_cost, wl.profiles_shape, wl.num_frames, wl.budget, wl.profile,
                      class_id=wl.class_id, with_plan_workspace=False)
    bt = tb.batch_cost_table(wl.profiles_batch, wl.profiles_shape, wl.batch_cap)
    ws = None
    if workspace:
        n = tb.batched_workspace(b.shape)
        ws = torch.empty(max(n, 16), dtype=torch.uint8, device="cuda") if n else None
    b.status.fill_(-1)
    tb.debug_set_variant(variant)
    try:
        tb.batched_plan(b.shape, b.windows_dev, b.profiles_dev, bt, wl.batch_cap, b.class_id, b.best_gain,
                        b.best_cost, b.feasible, b.exit_out, b.status, workspace=ws)
    finally:
        tb.debug_set_variant(0)
    torch.cuda.synchronize()
    W, F = wl.num_windows, wl.total_frames
    return (b.exit_out[:F].cpu().numpy(), b.best_gain[:W].cpu().numpy(), b.best_cost[:W].cpu().numpy(),
            b.feasible[:W].cpu().numpy(), b.status.cpu().numpy())


def _check(tb, wl, variant=0):
    ex, g, c, f, st = _gpu(tb, wl, variant=variant)
    oe, og, oc, of = oracle.batched(wl)
    assert st[0] == -1 and st[1] == -1, st
    np.testing.assert_array_equal(f, of)
    np.testing.assert_array_equal(g, og)
    np.testing.assert_array_equal(c, oc)
    np.testing.assert_array_equal(ex, oe)


@pytest.mark.parametrize("seed,K,C,nmax", [(1, 2, 4, 12), (2, 3, 4, 10), (3, 4, 5, 9), (4, 5, 3, 8), (5, 3, 10, 40),
                                          (6, 16, 4, 6), (7, 8, 6, 7)])
def test_random_sets(tb, seed, K, C, nmax):
    _check(tb, synth.make_batched_random(seed, 300, max_frames=nmax, K=K, C=C, max_budget=12 * nmax))


def test_linear_tables(tb):
    _check(tb, synth.make_batched_random(11, 300, max_frames=10, K=4, C=4, max_budget=40, linear=True))


@pytest.mark.parametrize("k", [1, 2])
def test_config_windows(tb, k):
    _check(tb, synth.make_batched_config(k, num_windows=None if k == 1 else 256))


@pytest.mark.parametrize("seed,K,C,nmax", [(21, 3, 4, 9), (22, 4, 4, 8), (23, 2, 6, 14), (24, 5, 3, 7),
                                          (25, 8, 4, 5), (26, 3, 10, 30)])
def test_general_gains(tb, seed, K, C, nmax):
    """Gains without R19: the general program (reading R20) against the oracle's."""
    wl = synth.make_batched_random(seed, 300, max_frames=nmax, K=K, C=C, max_budget=12 * nmax, general=True)
    _check(tb, wl)


@pytest.mark.parametrize("k", [1, 2])
def test_general_program_forced_on_r19(tb, k):
    """Variant 64 plans every valid window with the general program: on R19 profiles it must give
    exactly the canonical plans of the count-vector enumeration (b1, and 128 windows of b2)."""
    _check(tb, synth.make_batched_config(k, num_windows=None if k == 1 else 128), variant=64)
    _check(tb, synth.make_batched_random(33, 200, max_frames=12, K=4, C=5, max_budget=60), variant=64)


def test_r19_violation_without_workspace_is_rejected(tb):
    wl = synth.make_batched_random(12, 6, max_frames=6, K=3, C=3)
    p0 = int(wl.profile[2])
    g = wl.profiles_gain[p0].copy().reshape(3, 3)
    g[0, 2] += 50
    wl.profiles_gain[p0] = g.reshape(-1)
    wl.profile[:] = (p0 + 1) % len(wl.profiles_gain)
    wl.profile[2] = p0
    ex, gg, cc, f, st = _gpu(tb, wl, workspace=False)
    assert st[1] == 2 and f[2] == 0 and gg[2] == 0 and cc[2] == 0
    ex, gg, cc, f, st = _gpu(tb, wl, workspace=True)           # planned by the general program
    oe, og, oc, of = oracle.batched(wl)
    assert st[1] == -1
    np.testing.assert_array_equal(ex, oe)
    np.testing.assert_array_equal(gg, og)


def test_r19_violation_and_bad_class(tb):
    wl = synth.make_batched_random(12, 6, max_frames=6, K=3, C=3)
    p0 = int(wl.profile[2])
    g = wl.profiles_gain[p0].copy().reshape(3, 3)
    g[0, 2] += 50
    wl.profiles_gain[p0] = g.reshape(-1)
    wl.profile[:] = (p0 + 1) % len(wl.profiles_gain)
    wl.profile[2] = p0
    ff = wl.first_frame
    x = int(ff[4]) if wl.num_frames[4] > 0 else None
    if x is not None:
        wl.class_id[x] = 200
    ex, gg, cc, f, st = _gpu(tb, wl, workspace=False)
    assert st[1] == 2 and f[2] == 0 and gg[2] == 0 and cc[2] == 0
    if x is not None:
        assert st[0] == x and f[4] == 0
    assert (ex[ff[2]: ff[2] + wl.num_frames[2]] == 0).all()


def test_unsupported_sizes(tb):
    wl = synth.make_batched_random(13, 2, max_frames=6, K=3, C=3)
    import torch
    b = tb.make_batch(wl.profiles_gain, wl.profiles_cost, wl.profiles_shape, wl.num_frames, wl.budget, wl.profile,
                      class_id=wl.class_id, with_plan_workspace=False)
    bt = tb.batch_cost_table(wl.profiles_batch, wl.profiles_shape, wl.batch_cap)
    with pytest.raises(RuntimeError):
        tb.batched_plan(b.shape, b.windows_dev, b.profiles_dev, bt, 2, b.class_id, b.best_gain, b.best_cost,
                        b.feasible, b.exit_out, b.status)      # batch_cap below the window length
