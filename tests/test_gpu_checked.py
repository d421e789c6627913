"""Bounds-checked build on the GPU (compute-sanitizer is closed on this pool): the library compiled
with TURBO_CHECKS turns every TCHECK (row and pad ranges of the shared-memory tiles, the choice
plane extents, the halo stage and ring, the L2 rows, the staged option tables, the walks' cell and
frame ranges) into a device report. Every kernel path (scripts/sanitize_cases.py) and a parity
subset run against checked/libturbo.so in a subprocess; any report fails the test."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_2207_00172_b200", "checked", "libturbo.so")


@pytest.fixture(scope="module")
def checked_lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, TURBO_CHECKS="1")
    subprocess.run([sys.executable, "-m", "paper_2207_00172_b200.build"], cwd=ROOT, env=env, check=True,
                   capture_output=True, timeout=1800)
    assert os.path.exists(CHECKED)
    return CHECKED


def _run(lib, args):
    env = dict(os.environ, TURBO_LIB=lib)
    r = subprocess.run([sys.executable, *args], cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    out = r.stdout + r.stderr
    reports = [ln for ln in out.splitlines() if ln.startswith("TCHECK")]
    assert not reports, "\n".join(reports[:20])
    assert r.returncode == 0, out[-3000:]
    return out


SELFTEST = ("import torch; from paper_2207_00172_b200 import turbo; turbo.load(); "
            "turbo._check('selftest', turbo.load().turbo_debug_tcheck_selftest(None)); torch.cuda.synchronize(); "
            "print('selftest done')")


def test_reporting_path_is_live(checked_lib):
    """A deliberately violated check reports in the checked library (and not in production)."""
    env = dict(os.environ, TURBO_LIB=checked_lib)
    r = subprocess.run([sys.executable, "-c", SELFTEST], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "selftest done" in r.stdout, r.stdout + r.stderr
    assert any(ln.startswith("TCHECK") and "v != 7" in ln for ln in r.stdout.splitlines()), r.stdout
    r = subprocess.run([sys.executable, "-c", SELFTEST], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "TCHECK" not in r.stdout


def test_every_kernel_path_checked(checked_lib):
    out = _run(checked_lib, [os.path.join("scripts", "sanitize_cases.py")])
    assert "sanitize cases ok" in out


def test_parity_subset_checked(checked_lib):
    _run(checked_lib, ["-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                       "tests/test_gpu_parity.py::test_adversarial", "tests/test_gpu_parity.py::test_tie_heavy_wide",
                       "tests/test_gpu_long.py::test_long_window_costs_beyond_the_halo",
                       "tests/test_gpu_long.py::test_long_window_random_rows",
                       "tests/test_gpu_full.py::test_lockstep_kernel_mixed_windows",
                       "tests/test_gpu_full.py::test_runtime_k_body"])
