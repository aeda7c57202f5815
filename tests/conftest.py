"""Shared test fixtures.  `gpu` tests call the CUDA path through the C ABI;
everything else runs on the CPU (oracle pins, host logic, ABI symbol checks)."""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200")
    # Build the oracle (and the CUDA library) if missing; nvcc cross-compiles here.
    need = [os.path.join(ROOT, "oracle", "liblbm_oracle.so"),
            os.path.join(ROOT, "paper_1007_1388_b200", "liblbm_b200.so")]
    if not all(os.path.exists(p) for p in need):
        subprocess.run(["make", "-C", ROOT, "-j8"], check=False,
                       stdout=subprocess.DEVNULL)


def read_golden(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as fh:
        for line in fh:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            rows.append(line.split())
    return rows


@pytest.fixture(scope="session")
def golden_table():
    """(e[19,3], w as Fractions, opp[19]) from tests/golden/d3q19_table.txt."""
    from fractions import Fraction
    rows = read_golden("d3q19_table.txt")
    e = np.array([[int(r[1]), int(r[2]), int(r[3])] for r in rows])
    w = [Fraction(int(r[4]), int(r[5])) for r in rows]
    opp = np.array([int(r[6]) for r in rows])
    assert [int(r[0]) for r in rows] == list(range(19))
    return e, w, opp
