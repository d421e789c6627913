"""B200-native hot path of Turbo's enhancement scheduler (arXiv 2207.00172, §5).

The package holds the C-ABI library sources (csrc/, include/turbo.h at the repo root),
the in-tree build (build.py -> libturbo.so) and a thin ctypes binding (turbo.py).
It never imports oracle/ (the CPU oracle is test infrastructure only).
"""
from . import turbo  # noqa: F401
from .turbo import (  # noqa: F401
    TurboError, load, make_batch, batch_from_workload, run_path, results,
    mckp_workspace, profile_lookup, mckp_plan, backtrack, mckp_solve, mckp_solve_workspace, schedule, stats,
)
