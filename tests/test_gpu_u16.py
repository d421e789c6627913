"""NEXT-5: u16 DP rows, bit-exact against the oracle.

With variant bit 128 (opt-in: measured slower than the int32 rows on c2) the fixed-K
CTA kernels (staged options, walk in the kernel: turbo_schedule and turbo_mckp_solve) plan a
window on u16 rows when its values fit 16 bits -- every gain >= 0, a cost-0 exit in every
frame, sum_i max_k g_ik + max g + 1 <= 65535 (dp_kernel.cuh dp_tile_u16) -- and on the int32
packed-key rows otherwise. The recurrence and the tie-break (§5.2, reading R7)
are the same, so the plans must equal the oracle's bit for bit either way. Each set runs with the
u16 rows allowed (variant 128, + 1 = planes in smem, + 2 = planes in HBM, where the DP runs in plan
mode on int32 rows) and off (variant 0), and a device counter (turbo_debug_u16_counter) proves
which rows served the batch.
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


def _counted(wl, fused, variant, **kw):
    """gpu_run with the u16 window counter on; returns (results, windows planned on u16 rows)."""
    import torch
    from paper_2207_00172_b200 import turbo
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    turbo.debug_u16_counter(cnt)
    try:
        got = gpu_run(wl, fused, variant, **kw)
        torch.cuda.synchronize()
    finally:
        turbo.debug_u16_counter(None)
    return got, int(cnt.item())


def _eligible(wl):
    """Host restatement of the u16 rule per window (test logic: which windows MAY take u16)."""
    out = np.zeros(wl.num_windows, dtype=bool)
    ff = wl.first_frame
    for w in range(wl.num_windows):
        N = int(wl.num_frames[w])
        if N == 0:
            continue
        p = int(wl.profile[w])
        C, K = wl.profiles_shape[p]
        g = wl.profiles_gain[p].reshape(C, K).astype(np.int64)
        c = wl.profiles_cost[p].reshape(C, K)
        cls = wl.class_id[ff[w]: ff[w] + N].astype(np.int64)
        if (cls >= C).any():
            continue
        gw, cw = g[cls], c[cls]
        out[w] = (gw >= 0).all() and (cw == 0).any(axis=1).all() and gw.max(axis=1).sum() + gw.max() + 1 <= 65535
    return out


SETS = {
    # tie-heavy short rows (one warp, rows updated in place)
    "tie_short": dict(max_frames=40, min_budget=0, max_budget=200, max_gain=8, max_cost=4),
    # several warps per window, odd and even shifts
    "tie_mid": dict(max_frames=40, min_budget=200, max_budget=4000, max_gain=8, max_cost=41),
    # paper-scale gains (sum of max gains up to 56,000) over rows of every size class
    "paper_scale": dict(max_frames=40, min_budget=500, max_budget=20000, max_gain=1400, max_cost=301),
    # shifts beyond the 256-cell pad (the checked tile path) next to ineligible windows (profiles
    # without a cost-0 exit); rows short enough for smem planes
    "wide_cost_mixed": dict(max_frames=30, min_budget=600, max_budget=4000, max_gain=1400, max_cost=901,
                            no_zero_frac=0.3),
}
U16 = 128
PATHS = [("all", U16), (True, U16), (True, U16 | 1), (True, U16 | 2), ("all", U16 | 2), ("all", 0), (True, 0)]
PATH_IDS = ["schedule", "solve", "solve-smem", "solve-hbm", "schedule-hbm", "schedule-int32", "solve-int32"]


@pytest.mark.parametrize("K", [4, 5, 6, 8])
@pytest.mark.parametrize("name", sorted(SETS))
def test_u16_rows_parity(name, K):
    wl = synth.make_nonneg_set(seed=800 + K, W=600, K=K, **SETS[name])
    elig = _eligible(wl)
    want = oracle_run(wl)
    for (fused, variant), pid in zip(PATHS, PATH_IDS):
        got, n16 = _counted(wl, fused, variant)
        compare(wl, got, want, check_options=fused != "all")
        if not variant & U16 or variant & 2:      # HBM planes: the DP runs in plan mode (int32 rows)
            assert n16 == 0, pid
        else:
            assert 0 < n16 <= int(elig.sum()), (pid, n16, "the u16 rows never ran")


def test_u16_rows_every_eligible_window_on_c2():
    """c2 (the headline config): all 1,024 windows qualify and all are planned on u16 rows."""
    wl = synth.make_config(2)
    assert _eligible(wl).all()
    want = oracle_run(wl)
    got, n16 = _counted(wl, "all", U16)
    compare(wl, got, want, check_options=False)
    assert n16 == wl.num_windows
    got, n16 = _counted(wl, "all", 0)
    compare(wl, got, want, check_options=False)
    assert n16 == 0


@pytest.mark.parametrize("y,u16", [(2534, True), (2535, False)])
def test_u16_boundary(y, u16):
    """sum max g + max g + 1 = 65535 exactly: u16 rows, top value v = 65535; one more: int32."""
    wl = synth.make_u16_boundary(y)
    assert _eligible(wl).all() == u16
    want = oracle_run(wl)
    for fused, variant in [("all", U16), (True, U16), (True, U16 | 1), (True, U16 | 2)]:
        got, n16 = _counted(wl, fused, variant)
        compare(wl, got, want, check_options=fused != "all")
        assert n16 == (wl.num_windows if u16 and not variant & 2 else 0)


@pytest.mark.parametrize("fused", ["all", True], ids=["schedule", "solve"])
def test_u16_rows_with_a1_edges_and_device_budgets(fused):
    """a1 clamps and device budgets below the layout bound on u16 rows (B = 0 included)."""
    wl = synth.with_budget_edges(synth.make_nonneg_set(seed=901, W=800, K=5, max_frames=40, min_budget=0,
                                                       max_budget=3000, max_gain=1400, max_cost=77), seed=3)
    want = oracle_run(wl)
    got, n16 = _counted(wl, fused, U16)
    compare(wl, got, want, check_options=fused != "all")
    assert n16 > 0
    rng = np.random.default_rng(11)
    bud = np.floor(rng.random(wl.num_windows) * (wl.budget.astype(np.int64) + 1)).astype(np.int32)
    want = oracle_run(wl, budgets=bud)
    got, n16 = _counted(wl, fused, U16, device_budgets=bud)
    compare(wl, got, want, check_options=fused != "all")
    assert n16 > 0


def test_u16_and_int32_windows_share_ctas():
    """Eligible and ineligible windows interleaved in one launch: the CTA restores the int32 -inf
    pads after a u16 window (a grid-stride CTA serves many windows)."""
    a = synth.make_nonneg_set(seed=77, W=3000, K=5, max_frames=30, min_budget=0, max_budget=900, max_gain=30,
                              max_cost=60, no_zero_frac=0.5)
    tie = synth.make_tie_heavy(seed=78, W=3000, max_frames=30, max_exits=5, fixed_exits=5, max_budget=900,
                               max_cost=60, base_cost=5)
    wl = synth.concat_workloads([a, tie])
    perm_ok = _eligible(wl)
    assert perm_ok.any() and (~perm_ok).any()
    want = oracle_run(wl)
    for fused in ("all", True):
        got, n16 = _counted(wl, fused, U16)
        compare(wl, got, want, check_options=fused != "all")
        assert 0 < n16 <= int(perm_ok.sum())
