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
