"""C-ABI contract checks that need no GPU: the library builds/loads, exports every symbol
declared in include/turbo.h, and the host-only sizing call (turbo_mckp_workspace)
validates arguments and lays out windows as documented."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def tb():
    from paper_2207_00172_b200 import build, turbo
    build.build()
    turbo.load()
    return turbo


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "turbo.h")).read()
    return sorted(set(re.findall(r"\b(turbo_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(tb):
    lib = ctypes.CDLL(tb.LIB_PATH)
    syms = _declared_symbols()
    assert "turbo_profile_lookup" in syms and "turbo_mckp_plan" in syms and "turbo_backtrack" in syms
    for s in syms:
        getattr(lib, s)      # raises AttributeError if missing
    assert set(tb.EXPORTS) == set(syms)


def test_abi_version_and_strings(tb):
    lib = tb.load()
    assert lib.turbo_abi_version() == 1
    assert lib.turbo_status_string(0) == b"ok"
    assert lib.turbo_status_string(3) == b"workspace too small"


def test_struct_sizes(tb):
    assert ctypes.sizeof(tb.Window) == 48
    assert ctypes.sizeof(tb.Profile) == 24
    assert ctypes.sizeof(tb.Shape) == 192


def _profiles(tb, Ks, C=10):
    return [tb.Profile(C, K, 0x1000, 0x2000) for K in Ks]


def _wins(tb, nf, bud, prof):
    w = np.zeros(len(nf), dtype=tb.WINDOW_DTYPE)
    ff = np.zeros(len(nf), dtype=np.int64)
    ff[1:] = np.cumsum(np.asarray(nf[:-1], dtype=np.int64))
    w["first_frame"] = ff
    w["num_frames"] = nf
    w["budget"] = bud
    w["profile"] = prof
    return w


def test_serving_order_groups_classes_and_puts_long_work_first(tb):
    """turbo_window_t.order: a permutation, row-size classes ascending (long windows last),
    largest N (B+1) (K+1) first inside a class, index ascending on ties (turbo.h)."""
    profs = _profiles(tb, [5, 4, 16])
    nf = [30, 7, 0, 300, 30, 60, 5, 30]
    bud = [1000, 100, 5, 4096, 200, 100, 30000, 1000]
    prof = [0, 1, 2, 0, 2, 1, 0, 0]
    w = _wins(tb, nf, bud, prof)
    s = tb.mckp_workspace(profs, w)
    assert s.ordered == 1
    order = w["order"].tolist()
    assert sorted(order) == list(range(len(nf)))
    K = w["num_exits"]
    bounds = [256, 1024, 4608, 24576]

    def cls(i):
        cells = int(bud[i]) + 1
        return next((c for c, b in enumerate(bounds) if cells <= b), 4)

    def work(i):
        return int(nf[i]) * (int(bud[i]) + 1) * (int(K[i]) + 1)
    keys = [(cls(i), -work(i), i) for i in order]
    assert keys == sorted(keys)
    assert cls(order[-1]) == 4                      # the long window is served last
    # one class, even work: index order, not flagged
    w2 = _wins(tb, [30] * 5, [1000] * 5, [0] * 5)
    s2 = tb.mckp_workspace(profs, w2)
    assert s2.ordered == 0 and w2["order"].tolist() == list(range(5))


def test_workspace_layout(tb):
    profs = _profiles(tb, [5, 4, 16])
    w = _wins(tb, [30, 7, 0, 300], [1000, 100, 5, 4096], [0, 1, 2, 0])
    s = tb.mckp_workspace(profs, w)
    assert s.num_windows == 4 and s.max_frames == 300 and s.max_budget == 4096
    assert s.min_exits == 4 and s.max_exits == 16
    # option blocks aligned to 4 int32 (16 B)
    assert w["first_option"].tolist() == [0, 152, 180, 180]
    assert s.total_options == 180 + 300 * 5
    # choice plane bytes = N * tiles * 128, 4-bit tiles of 256 cells, 2-bit tiles of 512 cells
    t0 = -(-1001 // 256)   # K = 5
    t1 = -(-101 // 512)    # K = 4
    t3 = -(-4097 // 256)
    assert w["choice_offset"].tolist() == [0, 30 * t0 * 128, 30 * t0 * 128 + 7 * t1 * 128,
                                           30 * t0 * 128 + 7 * t1 * 128]
    assert s.workspace_bytes == 30 * t0 * 128 + 7 * t1 * 128 + 300 * t3 * 128
    assert w["num_exits"].tolist() == [5, 4, 16, 5]
    assert w["budget_bound"].tolist() == [1000, 100, 5, 4096]
    assert s.total_cells == 30 * 1001 + 7 * 101 + 0 + 300 * 4097
    assert s.total_frames == 337


@pytest.mark.parametrize("case,code", [
    ("bad_K", 1), ("bad_C", 1), ("bad_profile_index", 1), ("neg_frames", 1), ("neg_budget", 1),
    ("too_many_frames", 2), ("budget_too_big", 2),
])
def test_workspace_errors(tb, case, code):
    profs = _profiles(tb, [5])
    w = _wins(tb, [3], [10], [0])
    if case == "bad_K":
        profs = _profiles(tb, [17])
    elif case == "bad_C":
        profs = [tb.Profile(0, 5, 1, 1)]
    elif case == "bad_profile_index":
        w["profile"] = 1
    elif case == "neg_frames":
        w["num_frames"] = -1
    elif case == "neg_budget":
        w["budget"] = -3
    elif case == "too_many_frames":
        w["num_frames"] = 65536
    elif case == "budget_too_big":
        w["budget"] = 1 << 30
    with pytest.raises(tb.TurboError) as ei:
        tb.mckp_workspace(profs, w)
    assert ei.value.code == code


def test_device_calls_reject_null_shape(tb):
    lib = tb.load()
    assert lib.turbo_mckp_plan(None, None, None, None, None, 0, None, None, None, None, None) == 1
    assert lib.turbo_backtrack(None, None, None, None, 0, None, None, None, None) == 1
    assert lib.turbo_stats(None, None, None, None, None, None, None, None, None) == 1
    assert lib.turbo_debug_set_variant(7) == 1 and lib.turbo_debug_set_variant(3) == 1


def test_empty_batch_is_noop(tb):
    s = tb.mckp_workspace([], np.zeros(0, dtype=tb.WINDOW_DTYPE))
    lib = tb.load()
    # nothing to launch: returns OK without touching the device
    assert lib.turbo_mckp_plan(ctypes.addressof(s), None, None, None, None, 0, None, None, None, None, None) == 0
    assert lib.turbo_profile_lookup(ctypes.addressof(s), None, None, None, None, 0, None, None, None, None) == 0


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2207_00172_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "turbo_oracle" not in txt and "liboracle" not in txt, f
