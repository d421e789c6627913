"""Shared helpers of the GPU parity tests: run the CUDA path (through the C ABI) and the CPU
oracle on the same seeded workload and compare them element by element (bit-exact: the
path is integer-only)."""
from __future__ import annotations

import numpy as np

import oracle


def gpu_run(wl, fused=True, variant=0, with_stats=True, device_budgets=None):
    """device_budgets: run with capacity = NULL after writing these budgets into the device
    windows (the layout bound stays wl.budget)."""
    import torch
    from paper_2207_00172_b200 import turbo
    turbo.debug_set_variant(variant)
    try:
        b = turbo.batch_from_workload(wl, with_plan_workspace=not fused or (variant & 3) == 2,
                                      null_capacity=device_budgets is not None)
        if device_budgets is not None:
            turbo.set_device_budgets(b, device_budgets)
        turbo.run_path(b, fused=fused, with_stats=with_stats)
        torch.cuda.synchronize()
        out = turbo.results(b)
    finally:
        turbo.debug_set_variant(0)
    out["batch"] = b
    out["path"] = fused
    return out


def oracle_run(wl, mode="table", threads=None, budgets=None):
    """budgets: plan these budgets directly (the capacity = NULL path) instead of a1."""
    return oracle.run(wl, mode=mode, threads=threads, budgets=budgets)


def compare(wl, got, want, check_options=True, windows=None):
    """Element-by-element comparison of every output of the path."""
    W = wl.num_windows
    idx = np.arange(W) if windows is None else np.asarray(windows)
    np.testing.assert_array_equal(got["budget"][idx], want["budget"][idx], err_msg="a1 budget")
    np.testing.assert_array_equal(got["feasible"][idx], want["feasible"][idx], err_msg="feasible")
    np.testing.assert_array_equal(got["best_gain"][idx].astype(np.int64), want["best_gain"][idx], err_msg="G*")
    np.testing.assert_array_equal(got["best_cost"][idx].astype(np.int64), want["best_cost"][idx], err_msg="C*")
    ff = wl.first_frame
    nf = wl.num_frames
    K = wl.num_exits
    if windows is None:
        np.testing.assert_array_equal(got["exits"], want["exits"], err_msg="exits")
    else:
        for w in idx:
            np.testing.assert_array_equal(got["exits"][ff[w]: ff[w] + nf[w]], want["exits"][ff[w]: ff[w] + nf[w]],
                                          err_msg=f"exits window {w}")
    if check_options:
        gfo, ofo = got["first_option"], want["first_option"]
        for w in idx:
            n = int(nf[w]) * int(K[w])
            np.testing.assert_array_equal(got["opt_gain"][gfo[w]: gfo[w] + n], want["opt_gain"][ofo[w]: ofo[w] + n],
                                          err_msg=f"opt_gain window {w}")
            np.testing.assert_array_equal(got["opt_cost"][gfo[w]: gfo[w] + n], want["opt_cost"][ofo[w]: ofo[w] + n],
                                          err_msg=f"opt_cost window {w}")
    if windows is None and want.get("stats") is not None:
        np.testing.assert_array_equal(got["stats"], want["stats"], err_msg="stats")
    assert int(got["status"][0]) == -1 and int(got["status"][1]) == -1, got["status"]
