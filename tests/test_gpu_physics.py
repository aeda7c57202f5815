"""Closed-form physics through the CUDA path alone (no oracle): the GPU result must
reproduce the textbook solutions the oracle pins are checked against.

* plane Couette (half-way walls at z = -1/2 and N - 1/2, lid U): u_x = U (z + 1/2) / N
* shear wave u_x = A sin(2 pi z / N) decays as exp(-nu k^2 t), nu = (1/omega - 1/2)/3
  (P:433-435), in both layouts and precisions.
"""
import numpy as np
import pytest

from paper_1007_1388_b200 import inputs

pytestmark = pytest.mark.gpu


def lbm():
    from paper_1007_1388_b200 import lbm as m
    return m


@pytest.mark.parametrize("prec,layout", [(8, 0), (4, 0), (8, 1)])
def test_couette_closed_form_on_gpu(prec, layout):
    N = 16
    fl, wu, per = inputs.couette_flags(N)
    nx = 8  # several x cells and patches so the exchange is exercised too
    fl = np.repeat(fl, nx, axis=2)[:, :, : nx + 2]
    L = lbm().Lattice((nx, 1, N), (4, 1, 8), 1.0 / 0.8, prec, periodic=per, layout=layout)
    L.set_flags(fl, wu)
    L.step(12000)
    _, u = L.get_macroscopic()
    L.close()
    expect = inputs.LDC_U * (np.arange(N) + 0.5) / N
    tol = 1e-6 if prec == 8 else 2e-4
    np.testing.assert_allclose(u[:, 0, :, 0], np.repeat(expect[:, None], nx, axis=1), rtol=tol)


@pytest.mark.parametrize("prec,layout", [(8, 0), (4, 0), (8, 1)])
def test_shear_wave_viscosity_on_gpu(prec, layout):
    N, omega, T, A = 32, 1.2, 400, 1e-3
    n = (4, 4, N)
    # equilibrium of u_x = A sin(2 pi z / N), written out from eq:feq (centred, rho0 = 1)
    e = np.array([[0, 0, 0], [1, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1], [0, 0, -1],
                  [1, 1, 0], [-1, -1, 0], [1, -1, 0], [-1, 1, 0], [1, 0, 1], [-1, 0, -1], [1, 0, -1],
                  [-1, 0, 1], [0, 1, 1], [0, -1, -1], [0, 1, -1], [0, -1, 1]])
    w = np.array([1 / 3] + [1 / 18] * 6 + [1 / 36] * 12)
    z = np.arange(N)
    ux = A * np.sin(2 * np.pi * z / N)
    eu = e[:, 0][None, :] * ux[:, None]
    feq = w[None, :] * (3 * eu + 4.5 * eu ** 2 - 1.5 * ux[:, None] ** 2)
    f0 = np.broadcast_to(feq[:, None, None, :], (N, 4, 4, 19)).copy()
    L = lbm().Lattice(n, (4, 4, 8), omega, prec, periodic=(1, 1, 1), layout=layout)
    L.set_flags(np.zeros((N + 2, 6, 6), np.uint8))
    L.set_pdfs(f0)
    L.step(T)
    _, u = L.get_macroscopic()
    L.close()
    amp = 2.0 / N * np.sum(u[:, 0, 0, 0] * np.sin(2 * np.pi * z / N))
    nu = (1.0 / omega - 0.5) / 3.0
    assert amp == pytest.approx(A * np.exp(-nu * (2 * np.pi / N) ** 2 * T), rel=0.015)


@pytest.mark.parametrize("prec,layout", [(8, "ab"), (8, "aa"), (4, "ab")])
def test_total_mass_conserved_and_matches_inputs(prec, layout):
    """lbm_total_mass: equals N_fluid + sum of the input f~ right after set_pdfs,
    is conserved by collision + bounce-back in the closed lid-driven cavity
     over 400 steps (and an odd AA step count), and equals the
    oracle's sum of rho after 20 steps."""
    import oracle
    from paper_1007_1388_b200 import lbm
    n = (40, 36, 32)
    fl, wu = inputs.ldc_flags(n)
    fl = inputs.add_obstacles(fl, 0.03, seed=59)
    f0 = inputs.noise_pdfs(n, seed=61)
    fluid = fl[1:-1, 1:-1, 1:-1] == 0
    m0 = float(fluid.sum()) + float(f0[fluid].sum())
    L = lbm.Lattice(n, (20, 18, 16), inputs.LDC_OMEGA, prec,
                    layout=lbm.LBM_LAYOUT_AA if layout == "aa" else lbm.LBM_LAYOUT_AB)
    try:
        L.set_flags(fl, wu)
        L.set_pdfs(f0)
        assert abs(L.total_mass() - m0) <= 1e-9
        L.step(20)
        ref = oracle.run(f0, fl, wu, inputs.LDC_OMEGA, 20, nthreads=oracle.max_threads())
        m_or = float(fluid.sum()) + float(ref[fluid].sum())
        tol = 1e-9 if prec == 8 else 1e-3
        assert abs(L.total_mass() - m_or) <= tol
        L.step(381)  # odd total: AA streamed representation
        assert abs(L.total_mass() - m0) <= (1e-9 if prec == 8 else 1e-2)
    finally:
        L.close()
