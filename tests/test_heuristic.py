"""NEXT-1: the paper's prune-and-search heuristic, oracle pins on CPU and
GPU parity (marked gpu). Pins: SPEC.md:269's worked instance (the heuristic also reaches
(2, 0, 2), gain 1200, in two downgrades), the unconstrained budget (zero steps), the K = 2 /
uniform-cost case where the loop reduces to a sort (an independent closed form), dominance by
the exact optimum ("upper" >= heuristic), termination and feasibility."""
import numpy as np
import pytest

import oracle
import synth


def _h(g, c, B):
    N, K = g.shape
    ex, G, C, fe, st = oracle.heuristic([N], [B], [K], g.reshape(-1), c.reshape(-1))
    return ex.tolist(), int(G[0]), int(C[0]), int(fe[0]), int(st[0])


def test_worked_instance():
    g = np.array([[0, 400, 600], [0, 100, 150], [0, 400, 600]], np.int32)
    c = np.tile(np.array([0, 5, 10], np.int32), (3, 1))
    assert _h(g, c, 20) == ([2, 0, 2], 1200, 20, 1, 2)


def test_unconstrained_budget_no_steps():
    rng = np.random.default_rng(1)
    for _ in range(50):
        N, K = int(rng.integers(1, 30)), int(rng.integers(2, 9))
        g = rng.integers(-5, 20, size=(N, K)).astype(np.int32)
        c = rng.integers(0, 9, size=(N, K)).astype(np.int32)
        B = int(c[:, K - 1].sum())
        ex, G, C, fe, st = _h(g, c, B)
        assert st == 0 and ex == [K - 1] * N and fe == 1


def test_k2_uniform_cost_is_a_sort():
    """K = 2, (g0, c0) = (0, 0), enhancement cost cc for all: the loop downgrades frames in the
    order (gain asc, id asc) until at most floor(B / cc) frames remain enhanced."""
    rng = np.random.default_rng(2)
    for _ in range(1000):
        N = int(rng.integers(1, 25))
        cc = int(rng.integers(1, 5))
        g1 = rng.integers(-3, 7, size=N)
        B = int(rng.integers(0, cc * N + 1))
        g = np.stack([np.zeros(N, np.int64), g1], 1).astype(np.int32)
        c = np.stack([np.zeros(N, np.int64), np.full(N, cc)], 1).astype(np.int32)
        order = sorted(range(N), key=lambda i: (int(g1[i]), i))
        n_drop = max(0, N - B // cc)
        dropped = set(order[:n_drop])
        want = [0 if i in dropped else 1 for i in range(N)]
        ex, G, C, fe, st = _h(g, c, B)
        assert ex == want and st == n_drop


def test_dominated_by_exact_and_terminates():
    wl = synth.make_tie_heavy(seed=41, W=3000, max_frames=8, max_exits=5)
    og, oc, _, _ = oracle.lookup(wl)
    K = wl.num_exits
    hx, hg, hc, hf, hs = oracle.heuristic(wl.num_frames, wl.budget, K, og, oc)
    ex, eg, ec, ef = oracle.plan(wl.num_frames, wl.budget, K, og, oc)
    both = (hf == 1) & (ef == 1)
    assert (hg[both] <= eg[both]).all()
    assert (hf <= ef).all()                          # heuristic feasible => exact feasible
    # an infeasible heuristic plan is the all-zero plan, and it does exceed the budget
    ff = wl.first_frame
    fo = np.r_[0, np.cumsum(wl.num_frames.astype(np.int64) * K)[:-1]]
    for w in np.flatnonzero(hf == 0):
        n, k = int(wl.num_frames[w]), int(K[w])
        assert (hx[ff[w]: ff[w] + n] == 0).all()
        assert oc[fo[w]: fo[w] + n * k].reshape(n, k)[:, 0].sum() > wl.budget[w]
    assert (hs <= wl.num_frames.astype(np.int64) * (K - 1)).all()
    assert (hc[hf == 1] <= wl.budget[hf == 1]).all()


def test_gap_on_paper_profiles_is_small_and_nonnegative():
    """On Appendix-B concave profiles with linear costs the heuristic is near-optimal."""
    wl = synth.make_config(2, num_windows=64)
    out = oracle.run(wl)
    hx, hg, hc, hf, hs = oracle.heuristic(wl.num_frames, out["budget"], wl.num_exits, out["opt_gain"],
                                          out["opt_cost"])
    gap = (out["best_gain"] - hg) / np.maximum(out["best_gain"], 1)
    assert (gap >= 0).all() and gap.mean() < 0.01


@pytest.mark.gpu
@pytest.mark.parametrize("which", ["tie", "c2", "c5"])
def test_gpu_heuristic_matches_oracle(which):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2207_00172_b200 import turbo
    wl = {"tie": lambda: synth.make_tie_heavy(seed=43, W=2000, max_frames=40, max_exits=16, max_budget=200),
          "c2": lambda: synth.make_config(2),
          "c5": lambda: synth.make_config(5, num_windows=256)}[which]()
    b = turbo.batch_from_workload(wl)
    turbo.run_path(b, fused=True)
    W = wl.num_windows
    dev = b.best_gain.device
    hg = torch.zeros(W, dtype=torch.int32, device=dev)
    hc = torch.zeros(W, dtype=torch.int32, device=dev)
    hf = torch.zeros(W, dtype=torch.uint8, device=dev)
    hs = torch.zeros(W, dtype=torch.int32, device=dev)
    hx = torch.zeros(max(wl.total_frames, 1), dtype=torch.uint8, device=dev)
    turbo.heuristic_plan(b.shape, b.windows_dev, b.opt_gain, b.opt_cost, hg, hc, hf, hx, hs)
    torch.cuda.synchronize()
    og, oc, _, _ = oracle.lookup(wl)
    bud = oracle.budget(wl.capacity, wl.num_frames, wl.base_cost)
    ex, g, c, f, s = oracle.heuristic(wl.num_frames, bud, wl.num_exits, og, oc)
    np.testing.assert_array_equal(hx[:wl.total_frames].cpu().numpy(), ex)
    np.testing.assert_array_equal(hg.cpu().numpy(), g)
    np.testing.assert_array_equal(hc.cpu().numpy(), c)
    np.testing.assert_array_equal(hf.cpu().numpy(), f)
    np.testing.assert_array_equal(hs.cpu().numpy(), s)
