"""CPU checks of the parity-set generators added for NEXT-5 and the cluster kernel (inputs only:
they must have the structure their GPU tests rely on)."""
import numpy as np

import synth


def _max_gain_sum(wl, w):
    p = int(wl.profile[w])
    C, K = wl.profiles_shape[p]
    g = wl.profiles_gain[p].reshape(C, K).astype(np.int64)
    ff = wl.first_frame
    cls = wl.class_id[ff[w]: ff[w] + wl.num_frames[w]].astype(np.int64)
    return int(g[cls].max(axis=1).sum()), int(g[cls].max())


def test_u16_boundary_sits_on_the_rule():
    """sum_i max_k g + max g + 1 = 65535 for y = 2534 and 65536 for y = 2535 (every window)."""
    for y, total in ((2534, 65535), (2535, 65536)):
        wl = synth.make_u16_boundary(y)
        for w in range(wl.num_windows):
            s, m = _max_gain_sum(wl, w)
            assert s + m + 1 == total


def test_nonneg_set_structure():
    """Gains >= 0; every class row has a cost-0 exit except in the profiles drawn without one."""
    wl = synth.make_nonneg_set(seed=3, W=200, K=6, max_frames=20, min_budget=0, max_budget=500, max_gain=50,
                               max_cost=30, no_zero_frac=0.4)
    with_zero = 0
    for g, c, (C, K) in zip(wl.profiles_gain, wl.profiles_cost, wl.profiles_shape):
        assert (g >= 0).all() and K == 6
        z = (c.reshape(C, K) == 0).any(axis=1)
        assert z.all() or not z.any()                 # a profile has a cost-0 exit in every row or none
        with_zero += int(z.all())
    assert 0 < with_zero < len(wl.profiles_gain)
    assert (wl.budget >= 0).all() and (wl.budget <= 500).all()


def test_long_windows_of_the_cluster_edges():
    """The cluster-kernel edge set spans the routing boundaries (24,577 and 131,072 / 131,073 cells)."""
    cells = {w.budget[0] + 1 for w in (synth.make_long_window(81, N=9, K=5, B=131071, c_max=40000, random_rows=True),
                                       synth.make_long_window(82, N=7, K=4, B=131072, c_max=3000, random_rows=True),
                                       synth.make_long_window(83, N=33, K=6, B=24576, c_max=24000, random_rows=True))}
    assert cells == {131072, 131073, 24577}
