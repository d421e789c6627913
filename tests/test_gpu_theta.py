"""NEXT-3 fused into the path: turbo_schedule_theta reads the discriminator's difficulty scores
theta'_x and buckets them inside the DP launch (PAPER.md:511 buckets of width 0.1 on
d = 1 - theta, reading R6). It must be bit-identical to bucketize -> schedule: the oracle buckets the
scores (oracle_bucketize) and plans the resulting class ids; class_out must equal those ids.
Covers the one-CTA-per-window kernels, the runtime-K kernel + HBM walk, the lockstep kernel
(variant 8) and the long-window grid kernel + walk."""
import dataclasses

import numpy as np
import pytest

import oracle
import synth
from tests.parity import compare, oracle_run

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


def _scores(wl, seed):
    """Scores whose buckets follow the workload's class mix, plus bucket edges, NaN, +-inf and
    out-of-range values (clamped by the rule)."""
    rng = np.random.default_rng(seed)
    F = wl.total_frames
    th = (1.0 - (wl.class_id.astype(np.float64) + rng.random(F)) / 10.0).astype(np.float32)
    k = max(F // 50, 1)
    idx = rng.choice(F, size=min(6 * k, F), replace=False)
    special = np.array([np.nan, np.inf, -np.inf, 1.5, -0.7, 0.3], np.float32)
    th[idx] = special[np.arange(len(idx)) % len(special)]
    edges = rng.choice(F, size=min(k, F), replace=False)
    th[edges] = (1.0 - np.round(rng.random(len(edges)), 1)).astype(np.float32)       # exactly on edges
    return th


def _run(tb, wl, th, variant=0):
    import torch
    tb.debug_set_variant(variant)
    try:
        b = tb.batch_from_workload(wl, with_plan_workspace=False)
        F = wl.total_frames
        theta = torch.as_tensor(th, device="cuda")
        cls_out = torch.full((max(F, 1),), 255, dtype=torch.uint8, device="cuda")
        b.status.fill_(-1)
        b.stats.zero_()
        tb.schedule_theta(b.shape, b.profiles_dev, b.windows_dev, theta, 0.1, cls_out, b.capacity, b.base_cost,
                          b.solve_ws, b.best_gain, b.best_cost, b.feasible, b.exit_out, b.stats, b.status)
        torch.cuda.synchronize()
        out = tb.results(b)
        out["class_out"] = cls_out[:F].cpu().numpy()
    finally:
        tb.debug_set_variant(0)
    return out


CASES = {
    "c2": (lambda: synth.make_config(2), 0),
    "c2-lockstep": (lambda: synth.make_config(2), 8),
    "c5": (lambda: synth.make_config(5, num_windows=600), 0),
    "c3": (lambda: synth.make_config(3, num_windows=64), 0),
    "long": (lambda: synth.concat_workloads([synth.make_long_window(31, N=60, K=6, B=40000),
                                             synth.make_long_window(32, N=45, K=5, B=30000, c_max=5000,
                                                                    random_rows=True)]), 0),
}


@pytest.mark.parametrize("case", sorted(CASES))
def test_schedule_theta_equals_bucketize_then_schedule(tb, case):
    make, variant = CASES[case]
    wl = make()
    th = _scores(wl, 7)
    cls = oracle.bucketize(th, num_classes=10, width=0.1)
    wl_c = dataclasses.replace(wl, class_id=cls)
    got = _run(tb, wl, th, variant)
    np.testing.assert_array_equal(got["class_out"], cls)
    compare(wl_c, got, oracle_run(wl_c), check_options=False)
