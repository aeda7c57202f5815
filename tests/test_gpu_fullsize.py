"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

The whole lattice is too large for the oracle to follow for many steps, so the
oracle recomputes sampled planes one step at a time: read the GPU state at step
t on planes z-1..z+1 (lbm_get_pdfs_at), advance the GPU one step, and compare
plane z at t+1 with the oracle's update of that plane (oracle.step_slab on the
three-plane sub-lattice, whose only other input is the global flag array).
Sampled planes cover the bottom wall, the interior and the lid.
"""
import numpy as np
import pytest

import oracle
from paper_1007_1388_b200 import inputs

pytestmark = pytest.mark.gpu


def plane_cells(nx, ny, z0, z1):
    zz, yy, xx = np.meshgrid(np.arange(z0, z1), np.arange(ny), np.arange(nx), indexing="ij")
    return np.stack([xx.ravel(), yy.ravel(), zz.ravel()], 1)


@pytest.mark.parametrize("n,prec,patch,layout", [(256, 8, 256, "ab"), (256, 4, 256, "ab"), (384, 8, 384, "ab"),
                                                 (256, 4, 64, "ab"), (256, 8, 256, "aa"), (256, 4, 64, "aa")])
def test_full_size_sampled_planes(n, prec, patch, layout):
    """AA cases: the 5 warm-up steps leave the streamed state (odd count), the
    sampled step the swapped one -- both representations are read back."""
    from paper_1007_1388_b200 import lbm
    N = (n, n, n)
    fl, wu = inputs.ldc_flags(N)
    L = lbm.Lattice(N, (patch,) * 3, inputs.LDC_OMEGA, prec, device=0,
                    layout=lbm.LBM_LAYOUT_AA if layout == "aa" else lbm.LBM_LAYOUT_AB)
    try:
        L.set_flags(fl, wu)
        L.init_noise(inputs.NOISE_SEED)
        L.step(5)  # bench launch path: graph pair + single step
        planes = [0, 1, n // 2, n - 2, n - 1]
        before = {}
        for z in planes:
            lo, hi = max(z - 1, 0), min(z + 2, n)
            before[z] = (lo, hi, L.get_pdfs_at(plane_cells(n, n, lo, hi)).reshape(hi - lo, n, n, 19))
        L.step(1)
        tol = 1e-12 if prec == 8 else 1e-5
        for z in planes:
            lo, hi, src = before[z]
            got = L.get_pdfs_at(plane_cells(n, n, z, z + 1)).reshape(n, n, 19)
            sub_flags = np.ascontiguousarray(fl[lo:hi + 2])
            dst = np.zeros_like(src)
            # the GPU state is in the ctx precision; the oracle computes this one step in fp64
            oracle.step_slab(np.ascontiguousarray(src), dst, sub_flags, wu, inputs.LDC_OMEGA, z - lo, z - lo + 1,
                             nthreads=oracle.max_threads())
            err = float(np.abs(got - dst[z - lo]).max())
            # one step from an fp32 state: only rounding of this step (<< 1e-5)
            assert err <= tol, (z, err)
    finally:
        L.close()


@pytest.fixture(scope="module")
def ldc256_ref():
    """The oracle's LDC 256^3 state after 100 steps from the dyadic-noise start
    (~20 s on the host cores), shared by the precision / layout cases."""
    n = (256, 256, 256)
    fl, wu = inputs.ldc_flags(n)
    f0 = inputs.noise_pdfs(n)
    return fl, wu, oracle.run(f0, fl, wu, inputs.LDC_OMEGA, 100, nthreads=oracle.max_threads())


@pytest.mark.parametrize("prec,layout", [(8, "ab"), (4, "ab"), (8, "aa"), (4, "aa")])
def test_ldc256_100_steps_every_cell_vs_oracle(prec, layout, ldc256_ref):
    """BASELINE configs[1] (LDC 256^3 fp64 and fp32, dyadic
    noise start, the bench's launch path: graph pairs, the bounce-back list after
    every sweep) after 100 steps, every PDF of every fluid cell against the OpenMP
    oracle: <= 1e-12 (fp64), <= 1e-5 (fp32); two grids and the AA layout (blind
    PULL scatter + the list's fix-up)."""
    from paper_1007_1388_b200 import lbm
    n = (256, 256, 256)
    fl, wu, ref = ldc256_ref
    with lbm.Lattice(n, n, inputs.LDC_OMEGA, prec, device=0,
                     layout=lbm.LBM_LAYOUT_AA if layout == "aa" else lbm.LBM_LAYOUT_AB) as L:
        L.set_flags(fl, wu)
        L.init_noise(inputs.NOISE_SEED)  # the same state as the oracle's start, generated on the device
        L.step(100)
        got = L.get_pdfs()
    mask = fl[1:-1, 1:-1, 1:-1] == 0
    err = float(np.abs(got[mask] - ref[mask]).max())
    assert err <= (1e-12 if prec == 8 else 1e-5), err
