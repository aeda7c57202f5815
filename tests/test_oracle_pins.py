"""Pins of the CPU oracle to what the paper and the mathematics fix (not to itself).

Each test names the passage (P:n = PAPER.md line) and the plausible oracle
mistake it would catch.  CPU only.
"""
from fractions import Fraction as Fr

import numpy as np
import pytest

import oracle
from oracle import exact
from paper_1007_1388_b200 import inputs
from conftest import read_golden

RNG = np.random.default_rng(20100707)


# --------------------------------------------------------------------------- table
def test_table_matches_golden(golden_table):
    """Oracle's frozen direction table == golden (R2); catches a transposed or
    mis-signed velocity, a wrong weight or a wrong opposite."""
    e, w, opp = golden_table
    oe, ow, oopp = oracle.table()
    np.testing.assert_array_equal(oe, e)
    np.testing.assert_array_equal(oopp, opp)
    np.testing.assert_array_equal(ow, np.array([float(x) for x in w]))
    # the exact-rational oracle uses the same frozen order
    np.testing.assert_array_equal(np.array(exact.E), e)
    assert exact.W == w and exact.OPP == list(opp)


def test_lattice_isotropy_exact(golden_table):
    """D3Q19 moment identities (c_s^2 = 1/3, R5):
    sum w = 1, sum w e = 0, sum w e_a e_b = delta/3,
    sum w e_a e_b e_c e_d = (d_ab d_cd + d_ac d_bd + d_ad d_bc)/9, and e_opp = -e."""
    e, w, opp = golden_table
    assert sum(w) == 1
    for a in range(3):
        assert sum(w[i] * e[i, a] for i in range(19)) == 0
        for b in range(3):
            assert sum(w[i] * e[i, a] * e[i, b] for i in range(19)) == (Fr(1, 3) if a == b else 0)
            for c in range(3):
                for d in range(3):
                    lhs = sum(w[i] * e[i, a] * e[i, b] * e[i, c] * e[i, d] for i in range(19))
                    dl = lambda p, q: 1 if p == q else 0
                    rhs = Fr(dl(a, b) * dl(c, d) + dl(a, c) * dl(b, d) + dl(a, d) * dl(b, c), 9)
                    assert lhs == rhs
    for i in range(19):
        assert tuple(e[opp[i]]) == tuple(-e[i])
    # D3Q19: 1 rest, 6 faces (|e|^2 = 1), 12 edges (|e|^2 = 2), no corners
    norms = sorted(int((e[i] ** 2).sum()) for i in range(19))
    assert norms == [0] + [1] * 6 + [2] * 12


# --------------------------------------------------------------------------- equilibrium
def test_equilibrium_golden_values():
    """Hand evaluation of eq:feq at u = (0.1,0,0): f~_1 = 11/600."""
    feq = oracle.equilibrium(0.0, [0.1, 0.0, 0.0])
    for i, num, den in read_golden("feq_example.txt"):
        assert feq[int(i)] == pytest.approx(int(num) / int(den), abs=1e-17)


def test_equilibrium_special_cases():
    """(rho0, 0) -> all zeros exactly (centring); (rho0+drho, 0) -> w_i drho."""
    assert np.all(oracle.equilibrium(0.0, [0, 0, 0]) == 0.0)
    _, w, _ = oracle.table()
    np.testing.assert_allclose(oracle.equilibrium(0.0123, [0, 0, 0]), w * 0.0123, rtol=0, atol=1e-18)


def test_equilibrium_moments_closed_form(golden_table):
    """Moments of eq:feq (textbook): sum f~eq = drho, sum e f~eq = rho0 u,
    sum e_a e_b f~eq = drho/3 delta_ab + rho0 u_a u_b.  The second moment catches
    a dropped 4.5 (e.u)^2 or -1.5 u^2 term even when both are dropped together."""
    e, _, _ = golden_table
    for _ in range(20):
        drho = RNG.uniform(-0.05, 0.05)
        u = RNG.uniform(-0.1, 0.1, 3)
        feq = oracle.equilibrium(drho, u)
        assert feq.sum() == pytest.approx(drho, abs=1e-16)
        np.testing.assert_allclose(e.T @ feq, u, atol=1e-16)
        pi = np.einsum("ia,ib,i->ab", e, e, feq)
        np.testing.assert_allclose(pi, drho / 3 * np.eye(3) + np.outer(u, u), atol=1e-16)


# --------------------------------------------------------------------------- collision
def test_collision_conserves_mass_and_momentum(golden_table):
    """BGK with f^eq built from the same (drho, j = rho0 u) conserves both
    (P:410-415).  Catches u = j/rho instead of j/rho0 (R7) and
    f^eq built with rho0 instead of rho (R8)."""
    e, _, _ = golden_table
    for omega in (0.3, 1.0, 1.0 / 0.65, 1.9):
        for _ in range(20):
            p = RNG.uniform(-0.02, 0.02, 19)
            p[0] += 0.05  # sizable drho, so rho != rho0 matters
            out = oracle.collide(p, omega)
            assert out.sum() == pytest.approx(p.sum(), abs=1e-16)
            np.testing.assert_allclose(e.T @ out, e.T @ p, atol=1e-16)


def test_collision_omega_one_depends_only_on_moments():
    """omega = 1 (tau = 1): dst = f~eq(moments of pulled), so two pulled
    states with equal drho and j collide to the same result."""
    p = RNG.uniform(-0.02, 0.02, 19)
    v = np.zeros(19)
    v[[1, 2]] = 0.003      # +x and -x
    v[[3, 4]] = -0.003     # +y and -y : v carries zero mass and zero momentum
    out1 = oracle.collide(p, 1.0)
    out2 = oracle.collide(p + v, 1.0)
    np.testing.assert_allclose(out1, out2, atol=1e-17)
    # and omega = 0 leaves the pulled values untouched
    np.testing.assert_array_equal(oracle.collide(p, 0.0), p)


# --------------------------------------------------------------------------- whole-lattice invariants
def test_rest_is_bitwise_fixed_point():
    """f~ = 0 with no-slip walls only (U = 0) stays exactly 0."""
    n = (6, 5, 7)
    fl = inputs.shell_flags(n)
    f = np.zeros((n[2], n[1], n[0], 19))
    out = oracle.run(f, fl, np.zeros((0, 3)), 1.0 / 0.65, 10)
    assert np.all(out == 0.0)


def test_uniform_equilibrium_periodic_fixed_point():
    """A uniform equilibrium state on a fully periodic box is invariant."""
    n = (5, 4, 6)
    feq = oracle.equilibrium(0.01, [0.03, -0.02, 0.01])
    f = np.broadcast_to(feq, (n[2], n[1], n[0], 19)).copy()
    fl = np.zeros((n[2] + 2, n[1] + 2, n[0] + 2), np.uint8)
    out = oracle.run(f, fl, np.zeros((0, 3)), 1.3, 10, periodic=(1, 1, 1))
    np.testing.assert_allclose(out, f, atol=1e-16)


def test_mass_conserved_in_closed_cavity_with_lid():
    """Each src PDF is pulled exactly once and the tangential lid corrections cancel
    pairwise, so sum over fluid cells of sum_i f~_i is constant.
    Absolute bound because the sum is ~0."""
    n = (12, 10, 9)
    fl, wu = inputs.ldc_flags(n)
    f0 = inputs.noise_pdfs(n)
    m0 = f0.sum()
    out = oracle.run(f0, fl, wu, inputs.LDC_OMEGA, 100)
    assert abs(out.sum() - m0) <= 1e-12


def test_momentum_conserved_fully_periodic(golden_table):
    e, _, _ = golden_table
    n = (6, 5, 4)
    f0 = inputs.noise_pdfs(n)
    fl = np.zeros((n[2] + 2, n[1] + 2, n[0] + 2), np.uint8)
    out = oracle.run(f0, fl, np.zeros((0, 3)), 1.7, 20, periodic=(1, 1, 1))
    np.testing.assert_allclose(np.einsum("zyxi,ia->a", out, e), np.einsum("zyxi,ia->a", f0, e), atol=1e-13)
    assert abs(out.sum() - f0.sum()) <= 1e-13


def test_couette_closed_form():
    """Plane Couette (textbook): walls half-way at z = -1/2 and z = N - 1/2,
    lid velocity U -> steady u_x(z) = U (z + 1/2) / N.  Catches the literal BB sign
    reading (which drives the fluid backwards, R3) and a wrong wall position."""
    N = 8
    fl, wu, per = inputs.couette_flags(N)
    f = np.zeros((N, 1, 1, 19))
    out = oracle.run(f, fl, wu, 1.0 / 0.8, 4000, periodic=per)
    _, u = oracle.macroscopic(out, fl)
    ux = u[:, 0, 0, 0]
    expect = inputs.LDC_U * (np.arange(N) + 0.5) / N
    np.testing.assert_allclose(ux, expect, rtol=1e-6)
    np.testing.assert_allclose(u[:, 0, 0, 1:], 0.0, atol=1e-15)


def test_shear_wave_decay_matches_viscosity():
    """nu = (tau - 1/2) c_s^2 with omega = 1/tau, c_s^2 = 1/3:
    u_x = A sin(2 pi z / N) decays as exp(-nu k^2 t) (textbook).  Catches using tau
    for omega, a wrong c_s^2 or a wrong collision sign."""
    N, omega, T = 32, 1.2, 400
    A = 1e-3
    z = np.arange(N)
    f = np.zeros((N, 1, 1, 19))
    for k in range(N):
        f[k, 0, 0] = oracle.equilibrium(0.0, [A * np.sin(2 * np.pi * k / N), 0, 0])
    fl = np.zeros((N + 2, 3, 3), np.uint8)
    out = oracle.run(f, fl, np.zeros((0, 3)), omega, T, periodic=(1, 1, 1))
    _, u = oracle.macroscopic(out, fl)
    amp = 2.0 / N * np.sum(u[:, 0, 0, 0] * np.sin(2 * np.pi * z / N))
    nu = (1.0 / omega - 0.5) / 3.0
    expect = A * np.exp(-nu * (2 * np.pi / N) ** 2 * T)
    assert amp == pytest.approx(expect, rel=0.015)
    # and the decay is clearly not the one of a different viscosity reading
    nu_wrong = (omega - 0.5) / 3.0
    assert abs(amp - A * np.exp(-nu_wrong * (2 * np.pi / N) ** 2 * T)) > 0.05 * expect


# --------------------------------------------------------------------------- impulses (hand-derivable)
@pytest.mark.parametrize("i", range(19))
def test_impulse_streaming_and_bounce_back(i, golden_table):
    """omega = 0 isolates pull streaming + BB: a single f~_i(x0) = a moves to
    x0 + e_i in direction i, or -- if x0 + e_i is a no-slip wall -- stays at x0 in
    direction opp(i).  Positions: centre and a corner of a closed 5^3 box."""
    e, _, opp = golden_table
    n = (5, 5, 5)
    fl = inputs.shell_flags(n)
    a = 1e-3
    for x0 in [(2, 2, 2), (0, 0, 0), (4, 0, 4)]:
        f = np.zeros((5, 5, 5, 19))
        f[x0[2], x0[1], x0[0], i] = a
        out = oracle.run(f, fl, np.zeros((0, 3)), 0.0, 1)
        y = tuple(x0[k] + e[i, k] for k in range(3))
        if all(0 <= y[k] < 5 for k in range(3)):
            where, j = y, i
        else:
            where, j = x0, opp[i]
        expect = np.zeros((5, 5, 5, 19))
        expect[where[2], where[1], where[0], j] = a
        np.testing.assert_array_equal(out, expect)


@pytest.mark.parametrize("i", range(19))
def test_impulse_full_update(i, golden_table):
    """Same impulse with collision (omega = 1.5): only the receiving cell changes and
    dst_m = p_m - omega (p_m - w_m[a + 3a e_m.e_j + 4.5 a^2 (e_m.e_j)^2 - 1.5 a^2 |e_j|^2])
    with p = a delta_j (hand derivation from eq:lbm / eq:feq, rho0 = 1)."""
    e, w, opp = golden_table
    n = (4, 4, 4)
    fl = inputs.shell_flags(n)
    a, omega = 1e-3, 1.5
    x0 = (3, 1, 2)
    f = np.zeros((4, 4, 4, 19))
    f[x0[2], x0[1], x0[0], i] = a
    out = oracle.run(f, fl, np.zeros((0, 3)), omega, 1)
    y = tuple(x0[k] + e[i, k] for k in range(3))
    if all(0 <= y[k] < 4 for k in range(3)):
        where, j = y, i
    else:
        where, j = x0, opp[i]
    p = np.zeros(19)
    p[j] = a
    ej = e[j]
    cell = np.array([p[m] - omega * (p[m] - float(w[m]) * (a + 3 * a * (e[m] @ ej)
                                                            + 4.5 * a * a * (e[m] @ ej) ** 2
                                                            - 1.5 * a * a * (ej @ ej)))
                     for m in range(19)])
    expect = np.zeros((4, 4, 4, 19))
    expect[where[2], where[1], where[0]] = cell
    np.testing.assert_allclose(out, expect, rtol=0, atol=1e-18)


def test_lid_correction_golden(golden_table):
    """All-zero state under a moving lid, omega = 0: the cell under the lid receives
    exactly 6 w_i rho0 e_i.u_w in each direction pulled from the lid (R3);
    golden values +-1/120 (tests/golden/bb_lid_correction.txt)."""
    e, _, _ = golden_table
    n = (3, 3, 3)
    fl, wu = inputs.ldc_flags(n)
    f = np.zeros((3, 3, 3, 19))
    out = oracle.run(f, fl, wu, 0.0, 1)
    top = out[2, 1, 1]  # interior cell (1,1,2) just below the lid plane z = 3
    gold = {int(i): int(a) / int(b) for i, a, b in read_golden("bb_lid_correction.txt")}
    for i in range(19):
        if e[i, 2] == -1:
            assert top[i] == pytest.approx(gold[i], abs=1e-18), i
        else:
            assert top[i] == 0.0
    # a cell not under the lid receives nothing
    assert np.all(out[0] == 0.0)


# --------------------------------------------------------------------------- cavity properties
def test_ldc_lid_drives_positive_flow_and_mirror_symmetry(golden_table):
    """Lid moving in +x drags the fluid below it in +x (sign invariant), and the
    cavity is symmetric under y -> N-1-y with directions mirrored (S:95 variant)."""
    e, _, _ = golden_table
    n = (10, 10, 10)
    fl, wu = inputs.ldc_flags(n)
    f = np.zeros((10, 10, 10, 19))
    out = oracle.run(f, fl, wu, inputs.LDC_OMEGA, 100)
    _, u = oracle.macroscopic(out, fl)
    assert u[-1, :, :, 0].mean() > 0.01
    mirror = [int(np.where((e == e[i] * np.array([1, -1, 1])).all(1))[0][0]) for i in range(19)]
    np.testing.assert_allclose(out[:, ::-1, :, :][..., mirror], out, atol=1e-17)


# --------------------------------------------------------------------------- brute force exact
def _to_dict(f, fl, n):
    nx, ny, nz = n
    fd, fld = {}, {}
    for z in range(-1, nz + 1):
        for y in range(-1, ny + 1):
            for x in range(-1, nx + 1):
                fld[(x, y, z)] = int(fl[z + 1, y + 1, x + 1])
                if 0 <= x < nx and 0 <= y < ny and 0 <= z < nz:
                    fd[(x, y, z)] = [Fr(v) for v in f[z, y, x]]
    return fd, fld


@pytest.mark.parametrize("periodic", [(0, 0, 0), (1, 0, 0)])
def test_exact_rational_brute_force(periodic):
    """Exact-rational brute force (fractions) on a 4^3 box with shell, lid and an
    interior obstacle, dyadic init, 2 steps: fp64 oracle within rounding."""
    n = (4, 4, 4)
    fl, _ = inputs.ldc_flags(n, periodic)
    fl[2, 2, 3] = inputs.NOSLIP  # obstacle at (x=2, y=1, z=1)
    fl[3, 1, 1] = inputs.VELOCITY0 + 1  # second moving wall at (0,0,2)
    wu = np.array([[0.05, 0.0, 0.0], [0.0, -0.03125, 0.015625]])
    f0 = inputs.noise_pdfs(n, seed=7)
    omega = 1.5
    ref = oracle.run(f0, fl, wu, omega, 2, periodic=periodic)
    fd, fld = _to_dict(f0, fl, n)
    wu_fr = [tuple(Fr(v) for v in row) for row in wu]
    for _ in range(2):
        fd = exact.step(fd, fld, wu_fr, Fr(3, 2), periodic)
    ex = np.zeros_like(ref)
    for (x, y, z), v in fd.items():
        ex[z, y, x] = [float(t) for t in v]
    np.testing.assert_allclose(ref, ex, rtol=0, atol=1e-17)


def test_flag_validation():
    n = (3, 3, 3)
    fl = inputs.shell_flags(n)
    assert oracle.check_flags(n, (0, 0, 0), fl, 0) == 0
    bad = fl.copy()
    bad[0, 1, 1] = 0  # fluid shell cell on a non-periodic axis
    assert oracle.check_flags(n, (0, 0, 0), bad, 0) != 0
    assert oracle.check_flags(n, (0, 0, 1), bad, 0) == 0  # fine when z is periodic
    v = fl.copy()
    v[-1] = 3  # velocity wall k = 1
    assert oracle.check_flags(n, (0, 0, 0), v, 1) != 0
    assert oracle.check_flags(n, (0, 0, 0), v, 2) == 0


# --------------------------------------------------------------------------- macroscopic export
def test_macroscopic_rest_and_impulses(golden_table):
    """Macroscopic export (sec. 2.1): with centred PDFs rho = rho0 + sum f~
    and u = sum e_i f~_i / rho0, rho0 = 1 (R4, R7).  Pinned by hand-derivable states:
    the rest state f~ = 0 exports rho = 1 exactly (not 0: catches a dropped rho0),
    and a single impulse f~_i = a exports rho = 1 + a, u = a e_i with e_i from the
    golden table (catches a wrong sign / index in j).  Non-fluid cells export
    rho = u = 0 bitwise (R13)."""
    e, _, _ = golden_table
    n = (5, 4, 3)
    fl, _ = inputs.ldc_flags(n)
    fl[2, 2, 3] = inputs.NOSLIP  # interior obstacle at (x=2, y=1, z=1)
    solid = fl[1:-1, 1:-1, 1:-1] != 0
    rho, u = oracle.macroscopic(np.zeros(n[::-1] + (19,)), fl)
    assert np.all(rho[~solid] == 1.0) and np.all(rho[solid] == 0.0)
    assert np.all(u == 0.0)
    a = 0.0078125  # dyadic: 1 + a and a * e_i are exact
    for i in range(19):
        f = np.zeros(n[::-1] + (19,))
        f[..., i] = a
        rho, u = oracle.macroscopic(f, fl)
        assert np.all(rho[~solid] == 1.0 + a), i
        assert np.all(rho[solid] == 0.0)
        np.testing.assert_array_equal(u[~solid], np.broadcast_to(a * e[i].astype(float), u[~solid].shape))
        assert np.all(u[solid] == 0.0)


def test_macroscopic_of_equilibrium_closed_form():
    """A uniform state f~ = f~^eq(drho, u) must export rho = 1 + drho and u
    (P:443-450 applied to eq:feq; exact in rationals, so fp64 agrees to rounding)."""
    n = (3, 3, 3)
    fl = np.zeros((n[2] + 2, n[1] + 2, n[0] + 2), np.uint8)
    drho, uu = 0.01171875, [0.03125, -0.015625, 0.0078125]
    f = np.broadcast_to(oracle.equilibrium(drho, uu), n[::-1] + (19,)).copy()
    rho, u = oracle.macroscopic(f, fl)
    np.testing.assert_allclose(rho, 1.0 + drho, rtol=0, atol=1e-16)
    np.testing.assert_allclose(u, np.broadcast_to(uu, u.shape), rtol=0, atol=1e-16)
