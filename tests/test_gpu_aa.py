"""AA-pattern layout (one PDF array, alternating PULL / LOCAL steps) against the
two-grid layout and the oracle.  After every even step count the AA state
equals the two-grid state bitwise; after an odd count the export
un-streams the state, which at moving walls subtracts the wall term it added
(rounding-level difference, tolerance below)."""
import numpy as np
import pytest

import oracle
from paper_1007_1388_b200 import inputs

pytestmark = pytest.mark.gpu

TOL = {8: 1e-12, 4: 1e-5}
ODD_TOL_VS_AB = {8: 1e-16, 4: 1e-8}


def lbm():
    from paper_1007_1388_b200 import lbm as m
    return m


def fluid(fl):
    return fl[1:-1, 1:-1, 1:-1] == 0


def run(n, fl, wu, f0, steps, prec, layout, patch=None, calls=None, **kw):
    L = lbm().Lattice(n, patch or n, inputs.LDC_OMEGA, prec, layout=layout, **kw)
    try:
        L.set_flags(fl, wu)
        L.set_pdfs(f0)
        for s in (calls or [steps]):
            L.step(s)
        rho, u = L.get_macroscopic()
        return L.get_pdfs(), rho, u, L.info()
    finally:
        L.close()


def case(seed=31):
    n = (40, 26, 22)
    fl, wu = inputs.ldc_flags(n, periodic=(0, 1, 0))
    fl = inputs.add_obstacles(fl, 0.05, seed=seed, kinds=(inputs.NOSLIP, inputs.VELOCITY0 + 1))
    wu = np.vstack([wu, [[0.0, 0.02, -0.01]]])
    return n, fl, wu, inputs.noise_pdfs(n, seed=seed)


@pytest.mark.parametrize("prec", [8, 4])
@pytest.mark.parametrize("steps", [0, 1, 2, 7, 20])
def test_aa_equals_two_grid(prec, steps):
    m = lbm()
    n, fl, wu, f0 = case()
    ab, rho_ab, u_ab, _ = run(n, fl, wu, f0, steps, prec, m.LBM_LAYOUT_AB, periodic=(0, 1, 0))
    aa, rho_aa, u_aa, info = run(n, fl, wu, f0, steps, prec, m.LBM_LAYOUT_AA, periodic=(0, 1, 0))
    assert info["layout"] == m.LBM_LAYOUT_AA and info["aa_phase"] == steps % 2
    if steps % 2 == 0:
        np.testing.assert_array_equal(aa, ab)
        np.testing.assert_array_equal(rho_aa, rho_ab)
    else:
        assert np.abs(aa - ab).max() <= ODD_TOL_VS_AB[prec]
    if steps:
        ref = oracle.run(f0, fl, wu, inputs.LDC_OMEGA, steps, periodic=(0, 1, 0), nthreads=oracle.max_threads())
        mk = fluid(fl)
        assert np.abs(aa[mk] - ref[mk]).max() <= TOL[prec]


@pytest.mark.parametrize("prec", [8, 4])
def test_aa_multi_patch_forced_buffers_graphs(prec):
    """3x3x3 ragged patches (periodic y): AA exchange (two half-exchanges, the
    second masked to entries the sender computed) bitwise equal to one patch,
    through direct local copies and through pack / buffer / unpack; graph and
    non-graph paths and odd call splits agree."""
    m = lbm()
    n, fl, wu, f0 = case(seed=5)
    n2 = (36, 30, 24)
    fl, wu = inputs.ldc_flags(n2, periodic=(0, 1, 0))
    fl = inputs.add_obstacles(fl, 0.05, seed=6, kinds=(inputs.NOSLIP, inputs.VELOCITY0 + 1))
    wu = np.vstack([wu, [[0.01, 0.0, 0.02]]])
    f0 = inputs.noise_pdfs(n2, seed=8)
    kw = dict(periodic=(0, 1, 0))
    one, *_ = run(n2, fl, wu, f0, 12, prec, m.LBM_LAYOUT_AA, **kw)
    ab, *_ = run(n2, fl, wu, f0, 12, prec, m.LBM_LAYOUT_AB, **kw)
    many, *_ = run(n2, fl, wu, f0, 12, prec, m.LBM_LAYOUT_AA, patch=(12, 10, 8), **kw)
    forced, *_ = run(n2, fl, wu, f0, 12, prec, m.LBM_LAYOUT_AA, patch=(12, 10, 8),
                     exchange_mode=m.LBM_EXCHANGE_FORCE_BUFFERS, **kw)
    split, *_ = run(n2, fl, wu, f0, 12, prec, m.LBM_LAYOUT_AA, patch=(12, 10, 8), calls=[3, 4, 1, 4],
                    use_graphs=0, **kw)
    np.testing.assert_array_equal(one, ab)
    np.testing.assert_array_equal(many, one)
    np.testing.assert_array_equal(forced, one)
    np.testing.assert_array_equal(split, one)
    # odd count through patches
    odd_many, *_ = run(n2, fl, wu, f0, 9, prec, m.LBM_LAYOUT_AA, patch=(12, 10, 8), **kw)
    odd_one, *_ = run(n2, fl, wu, f0, 9, prec, m.LBM_LAYOUT_AA, **kw)
    np.testing.assert_array_equal(odd_many, odd_one)


def test_aa_fully_periodic_self_exchange_and_sampling():
    m = lbm()
    n = (16, 12, 10)
    fl = np.zeros((n[2] + 2, n[1] + 2, n[0] + 2), np.uint8)
    f0 = inputs.noise_pdfs(n, seed=4)
    ab, *_ = run(n, fl, None, f0, 10, 8, m.LBM_LAYOUT_AB, periodic=(1, 1, 1))
    aa, *_ = run(n, fl, None, f0, 10, 8, m.LBM_LAYOUT_AA, periodic=(1, 1, 1))
    np.testing.assert_array_equal(aa, ab)
    L = m.Lattice(n, (8, 6, 5), 1.7, 8, periodic=(1, 1, 1), layout=m.LBM_LAYOUT_AA)
    L.set_flags(fl)
    L.set_pdfs(f0)
    L.step(3)
    full = L.get_pdfs()
    cells = [(0, 0, 0), (15, 11, 9), (7, 5, 4)]
    np.testing.assert_array_equal(L.get_pdfs_at(cells), np.array([full[c[2], c[1], c[0]] for c in cells]))
    L.close()


def test_aa_state_rules():
    m = lbm()
    n = (8, 8, 8)
    fl, wu = inputs.ldc_flags(n)
    L = m.Lattice(n, layout=m.LBM_LAYOUT_AA)
    L.set_flags(fl, wu)
    L.init_noise(3)
    np.testing.assert_array_equal(L.get_pdfs(), np.where(fluid(fl)[..., None], inputs.noise_pdfs(n, seed=3), 0.0))
    L.step(1)
    with pytest.raises(m.LbmError) as ei:
        L.set_flags(fl, wu)  # only after an even step count in the AA layout
    assert ei.value.status == 2
    L.step(1)
    L.set_flags(fl, wu)
    L.close()
    # one PDF array instead of two (compared before any host transfer: those
    # add the persistent staging buffers to device_bytes)
    La, Lb = m.Lattice(n, layout=m.LBM_LAYOUT_AA), m.Lattice(n)
    assert La.info()["device_bytes"] < 0.7 * Lb.info()["device_bytes"]
    La.close()
    Lb.close()


@pytest.mark.parametrize("prec", [8, 4])
@pytest.mark.parametrize("n,patch", [((150, 14, 12), None), ((134, 18, 16), (67, 9, 8))])
def test_aa_variants_bitwise(prec, n, patch, monkeypatch):
    """Both AA kernel variants (LBM_SWEEP_VARIANT 0 / 1: occupancy targets) and
    their straight-line path for wall-free pairs equal the two-grid layout
    bitwise: x extents spanning several 64-cell tiles with a ragged last warp,
    odd patch widths, obstacles on the x faces, two moving walls, periodic y."""
    m = lbm()
    fl, wu = inputs.ldc_flags(n, periodic=(0, 1, 0))
    fl = inputs.add_obstacles(fl, 0.08, seed=41, kinds=(inputs.NOSLIP, inputs.VELOCITY0 + 1))
    wu = np.vstack([wu, [[0.01, 0.0, 0.02]]])
    f0 = inputs.noise_pdfs(n, seed=43)
    out = {}
    for v in ("0", "1"):
        monkeypatch.setenv("LBM_SWEEP_VARIANT", v)
        out[v] = run(n, fl, wu, f0, 10, prec, m.LBM_LAYOUT_AA, patch=patch, periodic=(0, 1, 0))[0]
    monkeypatch.delenv("LBM_SWEEP_VARIANT")
    ab = run(n, fl, wu, f0, 10, prec, m.LBM_LAYOUT_AB, patch=patch, periodic=(0, 1, 0))[0]
    for v in ("0", "1"):
        np.testing.assert_array_equal(out[v], ab)


@pytest.mark.parametrize("prec", [8, 4])
@pytest.mark.parametrize("n,patch,periodic", [((64, 30, 24), (16, 10, 12), (1, 0, 1)),
                                              ((60, 30, 24), (15, 30, 8), (1, 1, 0)),
                                              ((6, 4, 6), (1, 1, 2), (1, 1, 1))])
def test_aa_direct_stores_equal_half_exchanges(prec, n, patch, periodic, monkeypatch):
    """AA layout, many patches on one GPU: the sweep's direct stores (LOCAL: own
    cell into the neighbour's ghost, slot opp(q); PULL: scatter target in the
    neighbour, slot q) give bitwise the half-exchange copies and the two-grid
    layout, at even and odd step counts (odd: un-streamed export)."""
    m = lbm()
    fl, wu = inputs.ldc_flags(n, periodic=periodic)
    fl = inputs.add_obstacles(fl, 0.06, seed=47, kinds=(inputs.NOSLIP, inputs.VELOCITY0 + 1))
    wu = np.vstack([wu, [[0.0, 0.01, 0.02]]])
    f0 = inputs.noise_pdfs(n, seed=53)
    for steps in (4, 7):
        out = {}
        for ld in ("1", "0"):
            monkeypatch.setenv("LBM_LOCAL_DIRECT", ld)
            aa, rho, _, info = run(n, fl, wu, f0, steps, prec, m.LBM_LAYOUT_AA, patch=patch, periodic=periodic)
            assert info["local_direct"] == int(ld)
            out[ld] = aa
        np.testing.assert_array_equal(out["1"], out["0"])
        monkeypatch.delenv("LBM_LOCAL_DIRECT")
        ab = run(n, fl, wu, f0, steps, prec, m.LBM_LAYOUT_AB, patch=patch, periodic=periodic)[0]
        if steps % 2 == 0:
            np.testing.assert_array_equal(out["1"], ab)
        else:
            assert np.abs(out["1"] - ab).max() <= ODD_TOL_VS_AB[prec]
