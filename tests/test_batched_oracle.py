"""NEXT-4 oracle pins (batched-cost GAP; readings R18/R19 in DESIGN.md).

The count-vector oracle (oracle_batched_enum) is pinned to: the plain definition by brute force
over all K^N plans; the per-frame MCKP oracle when batches cost exactly n singles (linear
tables reduce the problem to the MCKP); the unconstrained closed form; the canonical form of
its plans; the R19 precondition."""
import itertools

import numpy as np
import pytest

import oracle
import synth


def _window(wl, w):
    ff = int(wl.first_frame[w])
    n = int(wl.num_frames[w])
    p = int(wl.profile[w])
    C, K = wl.profiles_shape[p]
    return (wl.class_id[ff:ff + n], wl.profiles_gain[p], C, K, wl.profiles_batch[p], wl.batch_cap,
            int(wl.budget[w]), ff, n)


def _gain_cost(cls, exits, g, K, I, cap):
    gain = sum(int(g[int(c) * K + int(k)]) for c, k in zip(cls, exits))
    cnt = np.bincount(np.asarray(exits, dtype=np.int64), minlength=K)
    cost = sum(int(I[k * (cap + 1) + cnt[k]]) for k in range(K))
    return gain, cost, cnt


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_enum_equals_brute_force(seed):
    wl = synth.make_batched_random(seed, 400, max_frames=7, K=3, C=4, max_budget=40)
    exits, G, Cs, fe = oracle.batched(wl)
    for w in range(wl.num_windows):
        cls, g, C, K, I, cap, B, ff, n = _window(wl, w)
        bg, bc, bcnt, bfe = oracle.batched_brute(cls, g, C, K, I, cap, B)
        assert (G[w], Cs[w], fe[w]) == (bg, bc, bfe), w
        gain, cost, cnt = _gain_cost(cls, exits[ff:ff + n], g, K, I, cap)
        assert gain == bg and cost == bc, w
        assert (cnt == bcnt).all(), w                     # R18: lexicographically smallest counts


def test_brute_force_is_the_definition():
    """The C brute force against an independent pure-Python enumeration (tiny windows)."""
    wl = synth.make_batched_random(9, 60, max_frames=5, K=3, C=3, max_budget=30)
    for w in range(wl.num_windows):
        cls, g, C, K, I, cap, B, ff, n = _window(wl, w)
        best = None
        for plan in itertools.product(range(K), repeat=n):
            gain, cost, cnt = _gain_cost(cls, plan, g, K, I, cap)
            if cost > B:
                continue
            key = (gain, -cost, tuple(-int(x) for x in cnt[::-1]))
            if best is None or key > best[0]:
                best = (key, gain, cost, cnt)
        bg, bc, bcnt, bfe = oracle.batched_brute(cls, g, C, K, I, cap, B)
        if best is None:
            assert bfe == 0 and (bcnt == [n] + [0] * (K - 1)).all()
        else:
            assert bfe == 1 and (bg, bc) == (best[1], best[2]) and (bcnt == best[3]).all()


def test_linear_batches_reduce_to_the_mckp():
    """I_k(n) = n c_k: the batched problem IS the per-frame MCKP (reading R1), so G* and C*
    must equal the MCKP oracle's on the same windows."""
    wl = synth.make_batched_random(4, 300, max_frames=8, K=4, C=4, max_budget=40, linear=True)
    _, G, Cs, fe = oracle.batched(wl)
    og, oc, fo, bad = oracle.lookup(wl)
    _, mg, mc, mf = oracle.plan(wl.num_frames, wl.budget, wl.num_exits, og, oc, "table")
    assert (fe == mf).all()
    feas = fe == 1
    assert (G[feas] == mg[feas]).all() and (Cs[feas] == mc[feas]).all()


def test_unconstrained_budget_closed_form():
    """B >= every plan's cost: G* = sum_x max_k g[c_x][k] (frames independent)."""
    wl = synth.make_batched_random(5, 200, max_frames=8, K=4, C=4, max_budget=40)
    wl.budget[:] = 10 ** 6
    _, G, Cs, fe = oracle.batched(wl)
    for w in range(wl.num_windows):
        cls, g, C, K, I, cap, B, ff, n = _window(wl, w)
        gt = np.asarray(g).reshape(C, K)
        assert G[w] == sum(int(gt[int(c)].max()) for c in cls) and fe[w] == 1


def test_canonical_form_and_b2_invariants():
    wl = synth.make_batched_config(2, num_windows=16)
    exits, G, Cs, fe = oracle.batched(wl)
    for w in range(wl.num_windows):
        cls, g, C, K, I, cap, B, ff, n = _window(wl, w)
        e = exits[ff:ff + n]
        order = sorted(range(n), key=lambda x: (int(cls[x]), x))
        assert all(e[order[j]] <= e[order[j + 1]] for j in range(n - 1))      # contiguous level blocks
        gain, cost, _ = _gain_cost(cls, e, g, K, I, cap)
        assert (gain, cost) == (G[w], Cs[w]) and cost <= B and fe[w] == 1


def test_budget_monotone():
    wl = synth.make_batched_config(2, num_windows=8)
    prev = None
    for B in (0, 200, 400, 700, 1000, 2000):
        wl.budget[:] = B
        _, G, _, _ = oracle.batched(wl)
        if prev is not None:
            assert (G >= prev).all()
        prev = G


def test_r19_violation_goes_to_the_general_program():
    """The count-vector enumeration refuses gains without R19; the batch entry then plans the window
    with the general program (reading R20) instead of rejecting it."""
    wl = synth.make_batched_random(6, 4, max_frames=4, K=3, C=3)
    p = int(wl.profile[0])
    g = wl.profiles_gain[p].copy().reshape(3, 3)
    g[0, 2] += 50                                          # easiest class gains most: breaks R19
    wl.profiles_gain[p] = g.reshape(-1)
    cls, gg, C, K, I, cap, B, ff, n = _window(wl, 0)
    with pytest.raises(RuntimeError):
        oracle.batched_enum(cls, gg, C, K, I, cap, B)
    ex, G, Cs, fe = oracle.batched(wl)
    want = oracle.batched_brute_plan(cls, gg, C, K, I, cap, B)
    assert (G[0], Cs[0], fe[0]) == want[1:]
    np.testing.assert_array_equal(ex[ff:ff + n], want[0])


# ---- NEXT-4 for any gain table (reading R20): the program over the canonical prefix and its counts
def _r19(g, C, K):
    g = np.asarray(g, dtype=np.int64).reshape(C, K)
    return bool((np.diff(np.diff(g, axis=1), axis=0) >= 0).all())


@pytest.mark.parametrize("seed", [21, 22, 23, 24])
def test_general_program_equals_brute_force_plan(seed):
    """G*, C*, the count vector AND the assignment against the plain R20 definition (all K^N plans)."""
    wl = synth.make_batched_random(seed, 300, max_frames=7, K=3 + seed % 2, C=4, max_budget=40, general=True)
    n_non_r19 = 0
    for w in range(wl.num_windows):
        cls, g, C, K, I, cap, B, ff, n = _window(wl, w)
        n_non_r19 += not _r19(g, C, K)
        got = oracle.batched_dp(cls, g, C, K, I, cap, B)
        want = oracle.batched_brute_plan(cls, g, C, K, I, cap, B)
        assert got[1:] == want[1:], w
        np.testing.assert_array_equal(got[0], want[0], err_msg=f"window {w}")
    assert n_non_r19 > wl.num_windows // 2                 # the set really exercises non-R19 gains


@pytest.mark.parametrize("seed", [31, 32])
def test_general_program_equals_canonical_under_r19(seed):
    """Under R19 the R20 plan is R18's canonical plan: identical to the count-vector enumeration."""
    wl = synth.make_batched_random(seed, 300, max_frames=16, K=4, C=5, max_budget=60)
    for w in range(wl.num_windows):
        cls, g, C, K, I, cap, B, ff, n = _window(wl, w)
        assert _r19(g, C, K)
        got = oracle.batched_dp(cls, g, C, K, I, cap, B)
        want = oracle.batched_enum(cls, g, C, K, I, cap, B)
        assert got[1:] == want[1:], w
        np.testing.assert_array_equal(got[0], want[0], err_msg=f"window {w}")


def test_general_program_gain_is_the_transportation_optimum():
    """For the chosen count vector, G* equals the C x K transportation LP optimum (scipy HiGHS,
    an independent solver; the LP is integral), and the plan realises it."""
    from scipy.optimize import linprog
    wl = synth.make_batched_random(41, 80, max_frames=14, K=4, C=4, max_budget=70, general=True)
    checked = 0
    for w in range(wl.num_windows):
        cls, g, C, K, I, cap, B, ff, n = _window(wl, w)
        ex, G, Cst, fe = oracle.batched_dp(cls, g, C, K, I, cap, B)
        if not fe or n == 0:
            continue
        gain, cost, cnt = _gain_cost(cls, ex, g, K, I, cap)
        assert (gain, cost) == (G, Cst)
        h = np.bincount(np.asarray(cls, dtype=np.int64), minlength=C)
        # variables y[c][k] >= 0: sum_k y = h_c, sum_c y = n_k; maximise sum g y
        A_eq, b_eq = [], []
        for c in range(C):
            row = np.zeros(C * K)
            row[c * K:(c + 1) * K] = 1
            A_eq.append(row)
            b_eq.append(h[c])
        for k in range(K):
            row = np.zeros(C * K)
            row[k::K] = 1
            A_eq.append(row)
            b_eq.append(cnt[k])
        res = linprog(-np.asarray(g[:C * K], dtype=np.float64), A_eq=np.array(A_eq), b_eq=np.array(b_eq),
                      bounds=(0, None), method="highs")
        assert res.status == 0
        assert round(-res.fun) == G, w
        checked += 1
    assert checked > 40
