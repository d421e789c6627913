"""Pins for the CPU oracle (oracle/), run without a GPU.

Each test checks the oracle against something other than itself:
  * an independent numpy enumeration of all plans (the total order of reading R7);
  * SPEC.md:269's worked instance (tests/golden/spec_worked_instance.json);
  * closed forms: unconstrained budget, B = 0, K = 2 with a uniform enhancement
    cost (reduces to a sort), K = 2 general (textbook 0/1 knapsack);
  * an independent ILP solver (scipy.optimize.milp / HiGHS) for G* at K > 2;
  * invariants: C* <= B, sum of chosen (g, c) = (G*, C*), G* non-decreasing in B
    (PAPER.md:640, :942 -- more idle budget never hurts), G* invariant under frame
    permutation, table == brute on 10^4 tie-heavy windows.
"""
import itertools
import json
import os

import numpy as np
import pytest

import synth
from synth.rng import rand_int, rand_uniform

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _rand_window(rng, N, K, g_lo=-2, g_hi=8, c_lo=0, c_hi=4, zero_base=True):
    g = rng.integers(g_lo, g_hi + 1, size=(N, K)).astype(np.int32)
    c = rng.integers(c_lo, c_hi + 1, size=(N, K)).astype(np.int32)
    if zero_base:
        c[:, 0] = 0
    return g, c


def _enumerate(g, c, B):
    """Independent numpy enumeration: argmax of (gain, -cost, -lex) over feasible plans."""
    N, K = g.shape
    if N == 0:
        return [], 0, 0, 1
    plans = np.array(list(itertools.product(range(K), repeat=N)), dtype=np.int64)  # lexicographic
    gains = g[np.arange(N)[None, :], plans].sum(axis=1)
    costs = c[np.arange(N)[None, :], plans].sum(axis=1)
    ok = costs <= B
    if not ok.any():
        return [0] * N, int(g[:, 0].sum()), int(c[:, 0].sum()), 0
    idx = np.flatnonzero(ok)
    # lexsort: last key primary. primary gain desc, then cost asc, then enumeration index asc.
    order = np.lexsort((idx, costs[idx], -gains[idx]))
    best = idx[order[0]]
    return plans[best].tolist(), int(gains[best]), int(costs[best]), 1


def _plan1(oracle_lib, g, c, B, mode="table"):
    N, K = g.shape
    ex, bg, bc, fe = oracle_lib.plan([N], [B], [K], g.reshape(-1), c.reshape(-1), mode, threads=1)
    return ex.tolist(), int(bg[0]), int(bc[0]), int(fe[0])


# ----------------------------------------------------------------------------- worked instance
def _golden():
    with open(os.path.join(GOLDEN, "spec_worked_instance.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("form", ["incremental_form", "absolute_form"])
def test_spec_worked_instance(oracle_lib, form):
    gd = _golden()
    inst, f = gd["instance"], gd[form]
    rows = f.get("gain_rows", gd["incremental_form"]["gain_rows"])
    cls = inst["classes"]
    g = np.array([rows[str(x)] for x in cls], dtype=np.int32)
    c = np.array([f["cost_row"]] * len(cls), dtype=np.int32)
    B = oracle_lib.budget([f["capacity"]], [len(cls)], f["base_cost"])[0]
    assert B == f["expected_budget"]
    for mode in ("table", "brute"):
        ex, G, C, fe = _plan1(oracle_lib, g, c, B, mode)
        assert ex == f["expected_exits"]
        assert G == f["expected_gain"]
        assert C == f["expected_cost"]
        assert fe == f["expected_feasible"]


def test_worked_instance_through_lookup(oracle_lib):
    """Same instance through a1+a2 (profile of 10 buckets, classes 9, 5, 9)."""
    gd = _golden()
    f = gd["incremental_form"]
    gain = np.zeros((10, 3), dtype=np.int32)
    gain[9] = f["gain_rows"]["9"]
    gain[5] = f["gain_rows"]["5"]
    cost = np.tile(np.array(f["cost_row"], dtype=np.int32), (10, 1))
    wl = synth.Workload("worked", [gain.reshape(-1)], [cost.reshape(-1)], [(10, 3)],
                        np.array([3], np.int32), np.array([20], np.int32), np.array([50], np.int32), 10,
                        np.array([0], np.int32), np.array(gd["instance"]["classes"], np.uint8))
    out = oracle_lib.run(wl)
    assert out["budget"].tolist() == [20]
    assert out["exits"].tolist() == [2, 0, 2]
    assert out["best_gain"].tolist() == [1200] and out["best_cost"].tolist() == [20]
    st = out["stats"]
    assert st[2] == 2 and st[0] == 1 and st[176] == 1200 and st[177] == 20 and st[178] == 1 and st[179] == 3


# ----------------------------------------------------------------------------- brute force
def test_brute_and_table_vs_independent_enumeration(oracle_lib):
    rng = np.random.default_rng(1234)
    n_checked = 0
    for trial in range(1500):
        N = int(rng.integers(0, 7))
        K = int(rng.integers(2, 5))
        g, c = _rand_window(rng, N, K, zero_base=bool(rng.random() < 0.7))
        B = int(rng.integers(0, 3 * max(N, 1) + 1))
        want = _enumerate(g, c, B)
        for mode in ("brute", "table"):
            got = _plan1(oracle_lib, g, c, B, mode)
            assert got == (want[0], want[1], want[2], want[3]), (trial, mode, g, c, B, got, want)
        n_checked += 1
    assert n_checked == 1500


def test_table_equals_brute_10k_tie_heavy(oracle_lib):
    """10^4 tie-heavy windows (N <= 8, K <= 4), SURVEY.md §8(c) pin 1."""
    wl = synth.make_tie_heavy(seed=77, W=10000, max_frames=8, max_exits=4)
    og, oc, _, bad = oracle_lib.lookup(wl)
    assert bad == -1
    K = wl.num_exits
    a = oracle_lib.plan(wl.num_frames, wl.budget, K, og, oc, "table")
    b = oracle_lib.plan(wl.num_frames, wl.budget, K, og, oc, "brute")
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)
    assert (a[3] == 0).sum() > 100      # infeasible windows exercised
    assert (a[3] == 1).sum() > 5000


# ----------------------------------------------------------------------------- closed forms
def test_closed_form_unconstrained_budget(oracle_lib):
    """B >= sum_i max_k c_ik: frames separate; each takes argmax (g desc, c asc, k asc)."""
    rng = np.random.default_rng(5)
    for _ in range(300):
        N, K = int(rng.integers(1, 40)), int(rng.integers(2, 17))
        g, c = _rand_window(rng, N, K, -5, 20, 0, 9)
        B = int(c.max(axis=1).sum()) + int(rng.integers(0, 5))
        want = []
        for i in range(N):
            best = min(range(K), key=lambda k: (-int(g[i, k]), int(c[i, k]), k))
            want.append(best)
        ex, G, C, fe = _plan1(oracle_lib, g, c, B)
        assert ex == want
        assert G == int(g[np.arange(N), want].sum()) and C == int(c[np.arange(N), want].sum()) and fe == 1


def test_closed_form_zero_budget(oracle_lib):
    """B = 0 with c_i0 = 0: each frame takes its best zero-cost option, smallest k."""
    rng = np.random.default_rng(6)
    for _ in range(300):
        N, K = int(rng.integers(1, 40)), int(rng.integers(2, 17))
        g, c = _rand_window(rng, N, K, -5, 20, 0, 3)
        want = []
        for i in range(N):
            zs = [k for k in range(K) if c[i, k] == 0]
            want.append(min(zs, key=lambda k: (-int(g[i, k]), k)))
        ex, G, C, fe = _plan1(oracle_lib, g, c, 0)
        assert ex == want and C == 0 and fe == 1


def test_closed_form_k2_uniform_cost_sort(oracle_lib):
    """K = 2, (g_0, c_0) = (0, 0), enhancement cost c for every frame: enhance the
    floor(B/c) frames with positive gain ranked by (gain desc, index desc)."""
    rng = np.random.default_rng(7)
    for _ in range(2000):
        N = int(rng.integers(1, 30))
        cc = int(rng.integers(1, 6))
        g1 = rng.integers(-3, 6, size=N)
        B = int(rng.integers(0, cc * N + 1))
        g = np.stack([np.zeros(N, np.int64), g1], axis=1).astype(np.int32)
        c = np.stack([np.zeros(N, np.int64), np.full(N, cc)], axis=1).astype(np.int32)
        pos = [i for i in range(N) if g1[i] > 0]
        pos.sort(key=lambda i: (-int(g1[i]), -i))
        chosen = set(pos[: B // cc])
        want = [1 if i in chosen else 0 for i in range(N)]
        ex, G, C, fe = _plan1(oracle_lib, g, c, B)
        assert ex == want, (g1.tolist(), cc, B, ex, want)


def _knapsack01(profit, weight, cap):
    """Textbook 0/1 knapsack (1-D array, reverse capacity loop)."""
    best = [0] * (cap + 1)
    for p, w in zip(profit, weight):
        for b in range(cap, w - 1, -1):
            best[b] = max(best[b], best[b - w] + p)
    return best[cap]


def test_k2_general_equals_01_knapsack(oracle_lib):
    rng = np.random.default_rng(8)
    for _ in range(500):
        N = int(rng.integers(1, 25))
        g0 = rng.integers(-5, 6, size=N)
        g1 = rng.integers(-5, 12, size=N)
        c1 = rng.integers(0, 8, size=N)
        B = int(rng.integers(0, 30))
        g = np.stack([g0, g1], 1).astype(np.int32)
        c = np.stack([np.zeros(N, np.int64), c1], 1).astype(np.int32)
        want = int(g0.sum()) + _knapsack01((g1 - g0).tolist(), c1.tolist(), B)
        ex, G, C, fe = _plan1(oracle_lib, g, c, B)
        assert G == want


def test_general_k_optimum_vs_milp(oracle_lib):
    """G* against an independent MILP solver (HiGHS via scipy): x_ik binary,
    sum_k x_ik = 1, sum c x <= B, maximise sum g x."""
    from scipy.optimize import LinearConstraint, milp, Bounds
    rng = np.random.default_rng(9)
    for _ in range(60):
        N, K = int(rng.integers(1, 25)), int(rng.integers(2, 9))
        g, c = _rand_window(rng, N, K, -3, 40, 0, 15)
        B = int(rng.integers(0, 8 * N))
        n = N * K
        A_eq = np.zeros((N, n))
        for i in range(N):
            A_eq[i, i * K:(i + 1) * K] = 1
        cons = [LinearConstraint(A_eq, 1, 1), LinearConstraint(c.reshape(1, -1).astype(float), -np.inf, B)]
        res = milp(-g.reshape(-1).astype(float), constraints=cons, integrality=np.ones(n), bounds=Bounds(0, 1))
        assert res.success
        ex, G, C, fe = _plan1(oracle_lib, g, c, B)
        assert G == int(round(-res.fun))


# ----------------------------------------------------------------------------- invariants
def test_invariants_paper_profiles(oracle_lib):
    wl = synth.make_config(2, num_windows=64)
    out = oracle_lib.run(wl)
    og, oc = out["opt_gain"].reshape(-1, 5), out["opt_cost"].reshape(-1, 5)
    ex = out["exits"].astype(np.int64)
    F = len(ex)
    chosen_g = og[np.arange(F), ex]
    chosen_c = oc[np.arange(F), ex]
    ff = wl.first_frame
    for w in range(wl.num_windows):
        s = slice(ff[w], ff[w] + wl.num_frames[w])
        assert chosen_g[s].sum() == out["best_gain"][w]
        assert chosen_c[s].sum() == out["best_cost"][w] <= out["budget"][w]
        assert out["feasible"][w] == 1
        assert out["best_gain"][w] >= 0           # >= all-zero plan (P_0 = 0)


def test_budget_monotonicity_and_permutation(oracle_lib):
    rng = np.random.default_rng(10)
    for _ in range(100):
        N, K = int(rng.integers(1, 20)), int(rng.integers(2, 8))
        g, c = _rand_window(rng, N, K, -2, 30, 0, 10, zero_base=bool(rng.random() < 0.8))
        prev = None
        for B in range(0, 40, 3):
            _, G, C, fe = _plan1(oracle_lib, g, c, B)
            val = G if fe else None
            if prev is not None:
                assert val is not None and val >= prev
            prev = val if val is not None else prev
            if fe:
                assert C <= B
        perm = rng.permutation(N)
        B = int(rng.integers(0, 40))
        a = _plan1(oracle_lib, g, c, B)
        b = _plan1(oracle_lib, g[perm], c[perm], B)
        assert a[1] == b[1] and a[2] == b[2] and a[3] == b[3]


def test_value_mode_matches_table(oracle_lib):
    wl = synth.make_tie_heavy(seed=3, W=500, max_frames=40, max_exits=9)
    og, oc, _, _ = oracle_lib.lookup(wl)
    a = oracle_lib.plan(wl.num_frames, wl.budget, wl.num_exits, og, oc, "table")
    b = oracle_lib.plan(wl.num_frames, wl.budget, wl.num_exits, og, oc, "value")
    for x, y in zip(a[1:], b[1:]):
        np.testing.assert_array_equal(x, y)


# ----------------------------------------------------------------------------- a1, a2, a6
def test_budget_rule(oracle_lib):
    cap = np.array([50, 10, 0, 1000, 7], np.int32)
    nf = np.array([3, 5, 0, 30, 1], np.int32)
    got = oracle_lib.budget(cap, nf, 10)
    assert got.tolist() == [20, 0, 0, 700, 0]


def test_lookup_is_gather(oracle_lib):
    wl = synth.make_config(5, num_windows=200)
    og, oc, fo, bad = oracle_lib.lookup(wl)
    assert bad == -1
    ff = wl.first_frame
    for w in range(0, 200, 7):
        p = wl.profile[w]
        C, K = wl.profiles_shape[p]
        G = wl.profiles_gain[p].reshape(C, K)
        Cc = wl.profiles_cost[p].reshape(C, K)
        cls = wl.class_id[ff[w]: ff[w] + wl.num_frames[w]]
        n = wl.num_frames[w] * K
        np.testing.assert_array_equal(og[fo[w]: fo[w] + n], G[cls].reshape(-1))
        np.testing.assert_array_equal(oc[fo[w]: fo[w] + n], Cc[cls].reshape(-1))


def test_lookup_bad_class(oracle_lib):
    wl = synth.make_config(1)
    wl.class_id[7] = 12
    _, _, _, bad = oracle_lib.lookup(wl)
    assert bad == 7


def test_stats_vs_bincount(oracle_lib):
    wl = synth.make_tie_heavy(seed=11, W=300, max_frames=8, max_exits=4)
    out = oracle_lib.run(wl)
    st = out["stats"]
    ex = out["exits"].astype(np.int64)
    np.testing.assert_array_equal(st[:16], np.bincount(ex, minlength=16))
    ce = np.zeros((10, 16), np.int64)
    np.add.at(ce, (wl.class_id.astype(np.int64), ex), 1)
    np.testing.assert_array_equal(st[16:176].reshape(10, 16), ce)
    assert st[176] == out["best_gain"].sum() and st[177] == out["best_cost"].sum()
    assert st[178] == wl.num_windows and st[179] == wl.total_frames
    assert st[180] == (out["feasible"] == 0).sum()


# ----------------------------------------------------------------------------- adversarial set
def test_adversarial_cases(oracle_lib):
    wl = synth.make_adversarial()
    out = oracle_lib.run(wl)
    ff = wl.first_frame
    ex = out["exits"]

    def plan(w):
        return ex[ff[w]: ff[w] + wl.num_frames[w]].tolist()

    # window index = case number - 1 (case 6 has two windows 6a, 6b -> cases >= 7 shift by 0
    # because case 1 is window 0): case 8 -> window 8, etc.
    assert plan(8) == [1, 0] and out["best_gain"][8] == 3 and out["best_cost"][8] == 2  # cost-before-lex
    assert plan(9) == [0, 1]                                # case 9: lex
    assert plan(10) == [1] and out["best_cost"][10] == 5    # case 10: min cost within frame
    assert out["feasible"][12] == 0 and plan(12) == [0, 0]  # case 12: c_0 > 0 infeasible
    assert out["best_gain"][12] == 3 and out["best_cost"][12] == 5
    assert out["best_gain"][0] == 0 and out["feasible"][0] == 1   # case 1: N = 0
    assert out["best_gain"][15] == 999 * 32767               # case 15: range limit
    # every window equals an independent enumeration where enumerable
    og, oc = out["opt_gain"], out["opt_cost"]
    fo = out["first_option"]
    K = wl.num_exits
    for w in range(wl.num_windows):
        N = int(wl.num_frames[w])
        if int(K[w]) ** N > 200000:
            continue
        g = og[fo[w]: fo[w] + N * K[w]].reshape(N, K[w])
        c = oc[fo[w]: fo[w] + N * K[w]].reshape(N, K[w])
        want = _enumerate(g, c, int(out["budget"][w]))
        assert (plan(w), int(out["best_gain"][w]), int(out["best_cost"][w]), int(out["feasible"][w])) == \
            (want[0], want[1], want[2], want[3]), w


def test_generator_deterministic_and_shardable():
    a = synth.make_config(3, window_offset=100, num_windows=5)
    b = synth.make_config(3, window_offset=0, num_windows=110)
    np.testing.assert_array_equal(a.class_id, b.subset(100, 105).class_id)
    c = synth.make_config(5, num_windows=50)
    d = synth.make_config(5, num_windows=50)
    np.testing.assert_array_equal(c.class_id, d.class_id)
    np.testing.assert_array_equal(c.budget, d.budget)
    assert rand_int(1, 2, np.arange(5), 0, 9).tolist() == rand_int(1, 2, np.arange(5), 0, 9).tolist()
    u = rand_uniform(1, 2, np.arange(100000))
    assert 0.49 < u.mean() < 0.51


def test_paper_profile_calibration():
    """Appendix B: kappa5 - kappa1 = 6.15 pts; bucket 9 - bucket 8 = 5.54 pts."""
    g = synth.paper_gain_table(6).reshape(10, 6)
    assert g[9, 5] - g[9, 1] == 615
    assert g[9, 5] - g[8, 5] == 554
    assert (np.diff(g, axis=1) >= 0).all() and (np.diff(g, axis=0) >= 0).all()
    assert synth.regular_costs(8, 41).tolist() == [0, 6, 12, 18, 24, 30, 36, 41]
    assert synth.regular_costs(6, 1049).tolist() == [0, 210, 420, 630, 840, 1049]
