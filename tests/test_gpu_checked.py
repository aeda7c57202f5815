"""The checked build (make checked, kernels.cuh Checker) over tools/sanitize_cases.py:
every global PDF access of the sweeps, the direct ghost stores and the bounce-back
list inside the grid allocations; every element written at most once per step
(the single-writer claims of DESIGN.md sections 7-9, incl. the in-place AA
kernels and the direct / fused ghost stores); no element read by one thread and
written by another within a launch.  compute-sanitizer is closed on the GPU pool,
so this is the memcheck / racecheck substitute.  A negative control injects
double stores and must be caught."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_1007_1388_b200", "liblbm_b200_checked.so")


def run_cases(extra_env=None, args=()):
    assert os.path.exists(CHECKED), "checked build missing (make checked / __graft_entry__.build())"
    env = dict(os.environ, LBM_LIBRARY=CHECKED, **(extra_env or {}))
    return subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py"), *args], env=env,
                          capture_output=True, text=True, timeout=900)


def test_checked_build_finds_nothing():
    r = run_cases()
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "sanitize cases done" in r.stdout


def test_checked_build_catches_injected_double_writes():
    r = run_cases({"LBM_CHECKED_INJECT": "1"}, ("--first",))
    assert r.returncode != 0
    assert "written twice" in (r.stdout + r.stderr)
