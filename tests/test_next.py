"""NEXT-3 (score -> class) and NEXT-2 (plan -> per-exit batches): oracle pins on CPU and GPU
parity (marked gpu)."""
import numpy as np
import pytest

import oracle
import synth


def test_bucketize_known_values():
    """PAPER.md:511 buckets of width 0.1 on d = 1 - theta (reading R6), clamped; NaN -> 0."""
    th = np.array([1.0, 0.96, 0.85, 0.45, 0.05, 0.0, -2.0, 3.0, np.nan, np.inf, -np.inf], np.float32)
    assert oracle.bucketize(th).tolist() == [0, 0, 1, 5, 9, 9, 9, 0, 0, 0, 9]


def test_bucketize_monotone_and_bucket_edges():
    """Class is non-increasing in theta, and every class is hit by its bucket's midpoint."""
    th = np.linspace(-0.2, 1.2, 20001).astype(np.float32)
    c = oracle.bucketize(th).astype(int)
    assert (np.diff(c) <= 0).all()
    mids = (1.0 - (np.arange(10) + 0.5) / 10).astype(np.float32)
    assert oracle.bucketize(mids).tolist() == list(range(10))
    assert oracle.bucketize(np.array([0.5], np.float32), num_classes=4, width=0.25).tolist() == [2]


def test_batches_is_a_stable_sort():
    """The per-exit order equals a stable argsort of the window's exits (library routine)."""
    rng = np.random.default_rng(3)
    nf = rng.integers(0, 70, size=50).astype(np.int32)
    ex = rng.integers(0, 16, size=int(nf.sum())).astype(np.uint8)
    count, order = oracle.batches(nf, ex)
    f0 = 0
    for w, n in enumerate(nf):
        e = ex[f0: f0 + n]
        assert count[w].tolist() == np.bincount(e, minlength=16).tolist()
        assert order[f0: f0 + n].tolist() == np.argsort(e, kind="stable").tolist()
        f0 += n


@pytest.fixture(scope="module")
def tb():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2207_00172_b200 import build, turbo
    build.build()
    turbo.load()
    return turbo


@pytest.mark.gpu
@pytest.mark.parametrize("n", [0, 1, 3, 4, 5, 1023, 100003])
def test_gpu_bucketize_matches_oracle(tb, n):
    import torch
    rng = np.random.default_rng(n)
    th = rng.uniform(-0.3, 1.3, size=n).astype(np.float32)
    if n > 10:
        th[:10] = np.array([1.0, 0.9, 0.8, 0.7, 0.1, 0.0, np.nan, np.inf, -np.inf, 0.5], np.float32)
        th[10: n // 2] = (1.0 - np.round(rng.uniform(0, 1, n // 2 - 10), 1)).astype(np.float32)   # on edges
    t = torch.zeros(max(n, 4), dtype=torch.float32, device="cuda")
    t[:n] = torch.from_numpy(th)
    out = torch.zeros(max(n, 4), dtype=torch.uint8, device="cuda")
    tb.bucketize(t[:n], out)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out[:n].cpu().numpy(), oracle.bucketize(th))


@pytest.mark.gpu
def test_gpu_batches_matches_oracle(tb):
    import torch
    wl = synth.make_config(5, num_windows=300)
    b = tb.batch_from_workload(wl)
    tb.run_path(b, fused="all")
    W, F = wl.num_windows, wl.total_frames
    count = torch.zeros(W * 16, dtype=torch.int32, device="cuda")
    order = torch.zeros(F, dtype=torch.int32, device="cuda")
    tb.batches(b.shape, b.windows_dev, b.exit_out, count, order)
    torch.cuda.synchronize()
    ex = b.exit_out[:F].cpu().numpy()
    want_c, want_o = oracle.batches(wl.num_frames, ex)
    np.testing.assert_array_equal(count.cpu().numpy().reshape(W, 16), want_c)
    np.testing.assert_array_equal(order.cpu().numpy(), want_o)


# ---- NEXT-2 executed latency f = sum_k I_k(n_k)
def _linear_tables(wl, cap):
    """I_k(n) = n c_k for every profile: a batch costs exactly n singles (reading R1)."""
    tabs = []
    for c, (C, K) in zip(wl.profiles_cost, wl.profiles_shape):
        ck = np.asarray(c, dtype=np.int64).reshape(C, K)[0]
        tabs.append((np.arange(cap + 1)[None, :] * ck[:, None]).reshape(-1).astype(np.int32))
    return tabs


def test_batch_latency_hand_example():
    # K = 3: I_0 = 0, I_1(n) = 5 + 2n (n > 0), I_2(n) = 9 + 4n (n > 0); counts (2, 3, 1) -> 0 + 11 + 13
    I = np.array([0, 0, 0, 0, 0, 7, 9, 11, 0, 13, 17, 21], np.int32)
    cnt = np.zeros((2, 16), np.int32)
    cnt[0, :3] = [2, 3, 1]
    cnt[1, :3] = [0, 4, 0]                    # n_1 = 4 > ncap = 3 -> -1
    lat = oracle.batch_latency(cnt, [3, 3], [0, 0], [I], 3)
    assert lat.tolist() == [24, -1]


def test_batch_latency_linear_tables_equal_plan_cost():
    """With linear batch tables the executed latency is the plan's summed per-frame cost, i.e. the
    MCKP optimum's C* (class-independent costs) -- computed by a different routine."""
    wl = synth.make_config(5, num_windows=200)
    out = oracle.run(wl)
    count, _ = oracle.batches(wl.num_frames, out["exits"])
    cap = int(wl.num_frames.max())
    lat = oracle.batch_latency(count, wl.num_exits, wl.profile, _linear_tables(wl, cap), cap)
    feas = out["feasible"].astype(bool)
    np.testing.assert_array_equal(lat[feas], out["best_cost"][feas])


def test_batch_latency_of_batched_plans_equals_their_cost():
    """NEXT-4 plans: the executed latency of the optimal plan's batches is the optimum's cost C*."""
    wl = synth.make_batched_random(11, W=300, max_frames=8, K=3, C=4, max_budget=40)
    ex, g, c, fe = oracle.batched(wl)
    count, _ = oracle.batches(wl.num_frames, ex)
    lat = oracle.batch_latency(count, wl.num_exits, wl.profile, wl.profiles_batch, wl.batch_cap)
    np.testing.assert_array_equal(lat, c)


@pytest.mark.gpu
@pytest.mark.parametrize("which", ["linear", "batched"])
def test_gpu_batch_latency_matches_oracle(tb, which):
    import torch
    if which == "linear":
        wl = synth.make_config(5, num_windows=300)
        cap = int(wl.num_frames.max())
        tabs = _linear_tables(wl, cap)
    else:
        wl = synth.make_batched_config(2, num_windows=200)
        cap = wl.batch_cap
        tabs = wl.profiles_batch
    b = tb.batch_from_workload(wl)
    tb.run_path(b, fused="all")
    W, F = wl.num_windows, wl.total_frames
    count = torch.zeros(W * 16, dtype=torch.int32, device="cuda")
    order = torch.zeros(F, dtype=torch.int32, device="cuda")
    lat = torch.zeros(W, dtype=torch.int64, device="cuda")
    st = torch.full((2,), -1, dtype=torch.int64, device="cuda")
    bt = tb.batch_cost_table(tabs, wl.profiles_shape, cap)
    tb.batches(b.shape, b.windows_dev, b.exit_out, count, order, bt, cap, lat, st)
    torch.cuda.synchronize()
    ex = b.exit_out[:F].cpu().numpy()
    want_c, _ = oracle.batches(wl.num_frames, ex)
    want = oracle.batch_latency(want_c, wl.num_exits, wl.profile, tabs, cap)
    np.testing.assert_array_equal(lat.cpu().numpy(), want)
    assert st.cpu().tolist() == [-1, -1]
    if which == "linear":
        feas = b.feasible[:W].cpu().numpy().astype(bool)
        np.testing.assert_array_equal(want[feas], b.best_cost[:W].cpu().numpy()[feas])
