"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Tolerances (BASELINE.json north_star): max |f~_GPU - f~_oracle| <= 1e-12 (fp64)
and <= 1e-5 (fp32, fp32 storage and arithmetic vs the fp64 oracle, R15) over
fluid cells; flags, fluid-cell counts and non-fluid rho/u bit-exact;
multi-patch / forced-buffer / graph variants bitwise equal to single patch.
"""
import numpy as np
import pytest

import oracle
from paper_1007_1388_b200 import inputs

pytestmark = pytest.mark.gpu

TOL = {8: 1e-12, 4: 1e-5}


def lbm():
    from paper_1007_1388_b200 import lbm as m
    return m


def fluid_mask(flags):
    return flags[1:-1, 1:-1, 1:-1] == 0


def max_fluid_diff(a, b, flags):
    m = fluid_mask(flags)
    return float(np.abs(a[m] - b[m]).max()) if m.any() else 0.0


def run_gpu(domain, flags, wall_u, f0, steps, prec=8, patch=None, omega=inputs.LDC_OMEGA, **kw):
    L = lbm().Lattice(domain, patch or domain, omega, prec, **kw)
    try:
        L.set_flags(flags, wall_u)
        L.set_pdfs(f0)
        L.step(steps)
        return L.get_pdfs()
    finally:
        L.close()


@pytest.mark.parametrize("prec", [8, 4])
def test_ldc_32_100_steps_vs_oracle(prec):
    """BASELINE configs[0]: LDC 32^3, single patch, 100 steps, dyadic noise init."""
    n = (32, 32, 32)
    fl, wu = inputs.ldc_flags(n)
    f0 = inputs.noise_pdfs(n)
    ref = oracle.run(f0, fl, wu, inputs.LDC_OMEGA, 100, nthreads=oracle.max_threads())
    got = run_gpu(n, fl, wu, f0, 100, prec)
    d = max_fluid_diff(got, ref, fl)
    assert d <= TOL[prec], d
    # non-fluid cells read back as 0 (R13)
    assert np.all(got[~fluid_mask(fl)] == 0.0)


@pytest.mark.parametrize("prec", [8, 4])
def test_ragged_obstacles_two_lids_periodic_x(prec):
    """Ragged sizes (not multiples of the 64 x 4 tile), interior obstacles, two moving
    walls, periodic x: 30 steps."""
    n = (37, 29, 23)
    fl, wu = inputs.ldc_flags(n, periodic=(1, 0, 0))
    fl = inputs.add_obstacles(fl, 0.08, seed=5, kinds=(inputs.NOSLIP, inputs.VELOCITY0 + 1))
    wu = np.vstack([wu, [[0.0, -0.02, 0.01]]])
    f0 = inputs.noise_pdfs(n, seed=11)
    ref = oracle.run(f0, fl, wu, 1.3, 30, periodic=(1, 0, 0), nthreads=oracle.max_threads())
    got = run_gpu(n, fl, wu, f0, 30, prec, omega=1.3, periodic=(1, 0, 0))
    assert max_fluid_diff(got, ref, fl) <= TOL[prec]


def test_fully_periodic_single_patch_self_exchange():
    """A periodic single patch is its own neighbour in all 18 directions."""
    n = (16, 12, 8)
    fl = np.zeros((n[2] + 2, n[1] + 2, n[0] + 2), np.uint8)
    f0 = inputs.noise_pdfs(n, seed=3)
    ref = oracle.run(f0, fl, np.zeros((0, 3)), 1.7, 40, periodic=(1, 1, 1))
    got = run_gpu(n, fl, None, f0, 40, 8, omega=1.7, periodic=(1, 1, 1))
    assert max_fluid_diff(got, ref, fl) <= 1e-12


@pytest.mark.parametrize("prec", [8, 4])
def test_multi_patch_bitwise_equal_single_patch(prec):
    """Decomposition invariance: 3x3x3 ragged patches with
    periodic y, obstacles; bitwise equal to one patch, within tolerance of the oracle."""
    n = (36, 30, 24)
    fl, wu = inputs.ldc_flags(n, periodic=(0, 1, 0))
    fl = inputs.add_obstacles(fl, 0.05, seed=9)
    f0 = inputs.noise_pdfs(n, seed=21)
    one = run_gpu(n, fl, wu, f0, 25, prec, periodic=(0, 1, 0))
    many = run_gpu(n, fl, wu, f0, 25, prec, patch=(12, 10, 8), periodic=(0, 1, 0))
    forced = run_gpu(n, fl, wu, f0, 25, prec, patch=(12, 10, 8), periodic=(0, 1, 0),
                     exchange_mode=lbm().LBM_EXCHANGE_FORCE_BUFFERS)
    np.testing.assert_array_equal(many, one)
    np.testing.assert_array_equal(forced, one)
    ref = oracle.run(f0, fl, wu, inputs.LDC_OMEGA, 25, periodic=(0, 1, 0), nthreads=oracle.max_threads())
    assert max_fluid_diff(one, ref, fl) <= TOL[prec]


def test_graphs_and_odd_steps_bitwise():
    n = (20, 18, 16)
    fl, wu = inputs.ldc_flags(n)
    f0 = inputs.noise_pdfs(n, seed=2)
    a = run_gpu(n, fl, wu, f0, 7, 8, patch=(10, 9, 8), use_graphs=1)
    b = run_gpu(n, fl, wu, f0, 7, 8, patch=(10, 9, 8), use_graphs=0)
    np.testing.assert_array_equal(a, b)
    # 7 = 3 + 4 via separate calls
    L = lbm().Lattice(n, (10, 9, 8))
    L.set_flags(fl, wu)
    L.set_pdfs(f0)
    L.step(3)
    L.step(4)
    np.testing.assert_array_equal(L.get_pdfs(), a)
    L.close()


@pytest.mark.parametrize("i", range(19))
def test_impulse_each_direction(i):
    """Hand-derivable single-PDF impulses (U = 0): one step moves f~_i(x0) to x0 + e_i
    or bounces it back at a wall; compared with the oracle at every cell."""
    n = (5, 5, 5)
    fl = inputs.shell_flags(n)
    for x0 in [(2, 2, 2), (0, 0, 0), (4, 0, 4), (0, 4, 2)]:
        f0 = np.zeros((5, 5, 5, 19))
        f0[x0[2], x0[1], x0[0], i] = 1e-3
        ref = oracle.run(f0, fl, np.zeros((0, 3)), 1.5, 1)
        got = run_gpu(n, fl, None, f0, 1, 8, omega=1.5)
        assert max_fluid_diff(got, ref, fl) <= 1e-18


def test_device_noise_init_matches_generator():
    """lbm_init_noise draws the same dyadic values as inputs.noise_pdfs (bitwise, both precisions)."""
    n = (20, 12, 9)
    expect = inputs.noise_pdfs(n, seed=1388)
    for prec in (8, 4):
        L = lbm().Lattice(n, (10, 6, 9), 1.0, prec, periodic=(1, 1, 1))
        L.set_flags(np.zeros((11, 14, 22), np.uint8))
        L.init_noise(1388)
        np.testing.assert_array_equal(L.get_pdfs(), expect)
        L.close()


def test_flags_readback_and_fluid_count_bit_exact():
    n = (24, 16, 12)
    fl, wu = inputs.ldc_flags(n)
    fl = inputs.add_obstacles(fl, 0.1, seed=4)
    L = lbm().Lattice(n, (12, 8, 6))
    L.set_flags(fl, wu)
    np.testing.assert_array_equal(L.get_flags(), fl)
    info = L.info()
    assert info["fluid_cells_global"] == int(fluid_mask(fl).sum()) == info["fluid_cells_local"]
    assert info["bytes_per_step_algorithmic"] == 2 * 19 * 8 * info["fluid_cells_local"]
    L.close()


def test_macroscopic_vs_oracle():
    n = (16, 16, 16)
    fl, wu = inputs.ldc_flags(n)
    fl = inputs.add_obstacles(fl, 0.05, seed=8)
    f0 = inputs.noise_pdfs(n)
    L = lbm().Lattice(n, (8, 8, 8))
    L.set_flags(fl, wu)
    L.set_pdfs(f0)
    L.step(50)
    rho, u = L.get_macroscopic()
    f = L.get_pdfs()
    L.close()
    ref = oracle.run(f0, fl, wu, inputs.LDC_OMEGA, 50)
    rr, ur = oracle.macroscopic(ref, fl)
    m = fluid_mask(fl)
    assert np.abs(rho[m] - rr[m]).max() <= 1e-12
    assert np.abs(u[m] - ur[m]).max() <= 1e-12
    assert np.all(rho[~m] == 0.0) and np.all(u[~m] == 0.0)
    # and the exported moments are those of the exported PDFs
    r2, u2 = oracle.macroscopic(f, fl)
    assert np.abs(rho - r2).max() <= 1e-15


def test_default_state_closed_box_at_rest():
    """After create: closed no-slip box at rest; stepping keeps it exactly zero."""
    L = lbm().Lattice((9, 7, 5), minimal=True)
    L.step(5)
    assert np.all(L.get_pdfs() == 0.0)
    assert L.info()["fluid_cells_global"] == 9 * 7 * 5
    L.close()


def test_edge_cases():
    m = lbm()
    # 1x1x1 fluid cell in a closed box; only rest + bounce-back
    n = (1, 1, 1)
    fl = inputs.shell_flags(n)
    f0 = inputs.noise_pdfs(n)
    ref = oracle.run(f0, fl, np.zeros((0, 3)), 1.2, 5)
    got = run_gpu(n, fl, None, f0, 5, 8, omega=1.2)
    assert max_fluid_diff(got, ref, fl) <= 1e-15
    # no fluid at all: step is a no-op, output zeros
    n = (6, 5, 4)
    fl = np.ones((6, 7, 8), np.uint8)
    L = m.Lattice(n)
    L.set_flags(fl)
    L.set_pdfs(inputs.noise_pdfs(n))
    L.step(3)
    assert np.all(L.get_pdfs() == 0.0) and L.info()["fluid_cells_global"] == 0
    # invalid flags leave the state unchanged
    fl_ok, wu = inputs.ldc_flags(n)
    L.set_flags(fl_ok, wu)
    bad = fl_ok.copy()
    bad[0, 2, 2] = 0  # fluid shell cell on non-periodic z
    with pytest.raises(m.LbmError) as ei:
        L.set_flags(bad, wu)
    assert ei.value.status == 1
    with pytest.raises(m.LbmError):
        L.set_flags(fl_ok, None)  # velocity wall without a velocity table
    np.testing.assert_array_equal(L.get_flags(), fl_ok)
    with pytest.raises(m.LbmError):
        L.step(-1)
    L.step(0)
    L.close()
    # nx = 1 rows, thin patches
    n = (1, 7, 9)
    fl, wu = inputs.ldc_flags(n, periodic=(1, 0, 0))
    f0 = inputs.noise_pdfs(n)
    ref = oracle.run(f0, fl, wu, 1.1, 12, periodic=(1, 0, 0))
    got = run_gpu(n, fl, wu, f0, 12, 8, omega=1.1, patch=(1, 7, 3), periodic=(1, 0, 0))
    assert max_fluid_diff(got, ref, fl) <= 1e-13


def test_sampled_cells_api():
    n = (16, 8, 8)
    L = lbm().Lattice(n, (8, 8, 8), 1.0, 8, periodic=(1, 1, 1))
    L.set_flags(np.zeros((10, 10, 18), np.uint8))
    L.init_noise(5)
    cells = [(0, 0, 0), (15, 7, 7), (8, 3, 4)]
    np.testing.assert_array_equal(L.get_pdfs_at(cells), inputs.noise_at(n, cells, seed=5))
    with pytest.raises(lbm().LbmError):
        L.get_pdfs_at([(16, 0, 0)])
    L.close()


@pytest.mark.parametrize("prec", [8, 4])
def test_sweep_occupancy_variants_bitwise_equal(prec, monkeypatch):
    """The x2 sweep's variants (LBM_SWEEP_VARIANT 0 / 1: occupancy targets, 2: the
    cp.async pull into shared memory) share one collide and one store-side
    bounce-back, so they agree bitwise; ragged patches, obstacles and a second
    moving wall, multi-patch exchange."""
    n = (80, 36, 20)
    fl, wu = inputs.ldc_flags(n, periodic=(0, 1, 0))
    fl = inputs.add_obstacles(fl, 0.04, seed=17, kinds=(inputs.NOSLIP, inputs.VELOCITY0 + 1))
    wu = np.vstack([wu, [[0.01, 0.0, -0.02]]])
    f0 = inputs.noise_pdfs(n, seed=19)
    out = {}
    for v in ("0", "1", "2"):
        monkeypatch.setenv("LBM_SWEEP_VARIANT", v)
        out[v] = run_gpu(n, fl, wu, f0, 13, prec, patch=(40, 18, 10), periodic=(0, 1, 0))
    np.testing.assert_array_equal(out["1"], out["0"])
    np.testing.assert_array_equal(out["2"], out["0"])
    ref = oracle.run(f0, fl, wu, inputs.LDC_OMEGA, 13, periodic=(0, 1, 0), nthreads=oracle.max_threads())
    assert max_fluid_diff(out["0"], ref, fl) <= TOL[prec]


# ---------------------------------------------------------------- the exchange paths on one GPU
# The multi-GPU exchange paths (NCCL send/recv with the shell / interior overlap,
# P:287-313 and the overlap the paper did not have; the fused NVLink
# exchange with its epoch handshake) run on one GPU through
# exchange_mode FORCE_BUFFERS (a one-rank NCCL communicator carries the
# self-peer messages) and SELF_PEER (this rank is its own fused-exchange peer).

EXCH_CASES = [((36, 30, 24), (12, 10, 8), (0, 1, 0)),   # 3x3x3 ragged patches, periodic y
              ((64, 16, 12), (64, 16, 12), (1, 1, 1)),  # one fully periodic patch: its own neighbour
              ((40, 12, 18), (20, 6, 9), (1, 0, 1))]    # 2x2x2 patches, periodic x and z


@pytest.mark.parametrize("prec", [8, 4])
@pytest.mark.parametrize("n,patch,periodic", EXCH_CASES)
@pytest.mark.parametrize("overlap", [1, 0])
def test_nccl_exchange_one_gpu_vs_oracle(prec, n, patch, periodic, overlap):
    """FORCE_BUFFERS on one GPU: pack -> grouped ncclSend/ncclRecv through a one-rank
    communicator -> unpack, with overlap = 1 the shells-first schedule (comm-stream
    transport and unpack while the interiors are swept).  Element-wise within
    tolerance of the oracle and bitwise equal to the default exchange."""
    m = lbm()
    fl, wu = inputs.ldc_flags(n, periodic=periodic)
    fl = inputs.add_obstacles(fl, 0.05, seed=51, kinds=(inputs.NOSLIP, inputs.VELOCITY0 + 1))
    wu = np.vstack([wu, [[0.0, 0.01, -0.01]]])
    f0 = inputs.noise_pdfs(n, seed=53)
    L = m.Lattice(n, patch, inputs.LDC_OMEGA, prec, periodic=periodic, overlap=overlap,
                  exchange_mode=m.LBM_EXCHANGE_FORCE_BUFFERS)
    try:
        info = L.info()
        assert info["nccl_ranks"] == 1 and info["exchange_fused"] == 0
        assert info["overlap_active"] == overlap
        L.set_flags(fl, wu)
        L.set_pdfs(f0)
        L.set_timing(True)  # one step timed: the overlap branch records its phases
        L.step(1)
        ph = L.phase_ms()
        L.set_timing(False)
        if overlap:
            assert ph["sweep_shell"][1] == 1 and ph["sweep_interior"][1] == 1 and ph["nccl"][1] == 1
        L.step(16)
        got = L.get_pdfs()
    finally:
        L.close()
    ref = oracle.run(f0, fl, wu, inputs.LDC_OMEGA, 17, periodic=periodic, nthreads=oracle.max_threads())
    assert max_fluid_diff(got, ref, fl) <= TOL[prec]
    np.testing.assert_array_equal(got, run_gpu(n, fl, wu, f0, 17, prec, patch=patch, periodic=periodic))


@pytest.mark.parametrize("prec", [8, 4])
@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("n,patch,periodic", EXCH_CASES)
def test_fused_exchange_self_peer_vs_oracle(prec, layout, n, patch, periodic):
    """SELF_PEER on one GPU: the fused multi-GPU exchange -- shells facing the
    (self-)peer swept on the comm stream with direct stores through the peer
    table, interiors concurrently on the compute stream, one epoch handshake
    (wait_peers / signal_peers) per step -- both layouts, odd and even step
    counts.  Element-wise within tolerance of the oracle, bitwise equal to the
    default exchange."""
    m = lbm()
    fl, wu = inputs.ldc_flags(n, periodic=periodic)
    fl = inputs.add_obstacles(fl, 0.05, seed=57, kinds=(inputs.NOSLIP, inputs.VELOCITY0 + 1))
    wu = np.vstack([wu, [[0.02, 0.0, 0.01]]])
    f0 = inputs.noise_pdfs(n, seed=59)
    L = m.Lattice(n, patch, inputs.LDC_OMEGA, prec, periodic=periodic, layout=layout,
                  exchange_mode=m.LBM_EXCHANGE_SELF_PEER)
    try:
        info = L.info()
        assert info["exchange_fused"] == 1 and info["fused_peers"] == 1 and info["nccl_ranks"] == 0
        L.set_flags(fl, wu)
        L.set_pdfs(f0)
        L.step(9)
        odd = L.get_pdfs()
        L.step(9)
        got = L.get_pdfs()
    finally:
        L.close()
    ref9 = oracle.run(f0, fl, wu, inputs.LDC_OMEGA, 9, periodic=periodic, nthreads=oracle.max_threads())
    ref = oracle.run(ref9, fl, wu, inputs.LDC_OMEGA, 9, periodic=periodic, nthreads=oracle.max_threads())
    assert max_fluid_diff(odd, ref9, fl) <= TOL[prec]
    assert max_fluid_diff(got, ref, fl) <= TOL[prec]
    np.testing.assert_array_equal(got, run_gpu(n, fl, wu, f0, 18, prec, patch=patch, periodic=periodic))


def test_self_peer_quiesce_then_set_pdfs_and_close():
    """with the fused exchange, state replacement and teardown wait for
    the peers' last stores.  AA layout, odd step count, then set_pdfs, step and
    close with no collective in between; the restarted run equals a fresh one."""
    m = lbm()
    n, patch = (32, 16, 16), (16, 8, 8)
    fl, wu = inputs.ldc_flags(n, periodic=(1, 0, 0))
    f0 = inputs.noise_pdfs(n, seed=61)
    f1 = inputs.noise_pdfs(n, seed=62)
    L = m.Lattice(n, patch, inputs.LDC_OMEGA, 8, periodic=(1, 0, 0), layout=1,
                  exchange_mode=m.LBM_EXCHANGE_SELF_PEER)
    L.set_flags(fl, wu)
    L.set_pdfs(f0)
    L.step_async(5)
    L.set_pdfs(f1)  # must drain the 5 queued steps and the handshake first
    L.step(4)
    got = L.get_pdfs()
    L.step_async(3)
    L.close()
    np.testing.assert_array_equal(got, run_gpu(n, fl, wu, f1, 4, 8, patch=patch, periodic=(1, 0, 0)))


@pytest.mark.parametrize("prec", [8, 4])
@pytest.mark.parametrize("n,patch,periodic", [((64, 30, 24), (16, 10, 12), (1, 0, 1)),
                                              ((60, 30, 24), (15, 30, 8), (1, 1, 0)),
                                              ((6, 4, 6), (1, 1, 2), (1, 1, 1)),
                                              ((8, 6, 4), (2, 3, 1), (1, 0, 1))])
def test_local_direct_equals_ghost_copies(prec, n, patch, periodic, monkeypatch):
    """The x2 sweep storing face / edge PDFs straight into same-GPU neighbour
    ghosts (the default) gives bitwise the ghost-copy result and the one-patch
    result: obstacles on patch boundaries, two moving walls, odd patch widths,
    a periodic self-neighbour (one patch along periodic y)."""
    fl, wu = inputs.ldc_flags(n, periodic=periodic)
    fl = inputs.add_obstacles(fl, 0.06, seed=31, kinds=(inputs.NOSLIP, inputs.VELOCITY0 + 1))
    wu = np.vstack([wu, [[0.0, 0.01, 0.02]]])
    f0 = inputs.noise_pdfs(n, seed=37)
    out = {}
    for ld in ("1", "0"):
        monkeypatch.setenv("LBM_LOCAL_DIRECT", ld)
        L = lbm().Lattice(n, patch, inputs.LDC_OMEGA, prec, periodic=periodic)
        assert L.info()["local_direct"] == int(ld)
        L.set_flags(fl, wu)
        L.set_pdfs(f0)
        L.step(11)
        out[ld] = L.get_pdfs()
        L.close()
    np.testing.assert_array_equal(out["1"], out["0"])
    one = run_gpu(n, fl, wu, f0, 11, prec, periodic=periodic)
    np.testing.assert_array_equal(out["1"], one)
    ref = oracle.run(f0, fl, wu, inputs.LDC_OMEGA, 11, periodic=periodic, nthreads=oracle.max_threads())
    assert max_fluid_diff(out["1"], ref, fl) <= TOL[prec]


@pytest.mark.parametrize("prec", [4, 8])
def test_patch_heavy_128_in_8_patches(prec):
    """SURVEY 8(d) config 5 parity: LDC 128^3 in 8 patches of 64^3 on one GPU
    (direct ghost stores between them) after 100 steps -- against the oracle
    and bitwise against one 128^3 patch."""
    n = (128, 128, 128)
    fl, wu = inputs.ldc_flags(n)
    f0 = inputs.noise_pdfs(n)
    patched = run_gpu(n, fl, wu, f0, 100, prec, patch=(64, 64, 64))
    single = run_gpu(n, fl, wu, f0, 100, prec)
    np.testing.assert_array_equal(patched, single)
    ref = oracle.run(f0, fl, wu, inputs.LDC_OMEGA, 100, nthreads=oracle.max_threads())
    assert max_fluid_diff(patched, ref, fl) <= TOL[prec]


def test_flags_upload_complete_at_size():
    """Regression: the flag upload is ordered with the
    library's stream -- a plain cudaMemcpy from pageable memory returned before
    its DMA landed and the lid plane was sometimes read as fluid.  Repeated
    set_flags / get_flags at 160^3 must read back exactly (the 128^3 parity
    test above checks the resulting dynamics)."""
    m = lbm()
    n = (160, 160, 160)
    fl, wu = inputs.ldc_flags(n)
    for prec in (4, 8):
        for _ in range(4):
            with m.Lattice(n, n, inputs.LDC_OMEGA, prec) as L:
                L.set_flags(fl, wu)
                np.testing.assert_array_equal(L.get_flags(), fl)


# ---------------------------------------------------------------- walls outside the sweep
# The sweeps carry no wall logic: the bounce-back list kernel (store side after a
# two-grid sweep / AA LOCAL, fix-up after AA PULL) handles every wall link, each
# entry carrying its wall mask and the shared velocity of its moving walls; tiles
# holding a non-fluid cell read the cells' kinds (per-tile descriptor bit).

def _mixed_wall_geometry(n):
    """A cavity whose fluid cells touch walls of three velocities at once: the lid
    (velocity 0), a moving-wall slab of velocity 1 just under it along y = 0, and a
    no-slip post, so some cells' moving walls disagree (the list entry's mixed case
    reads each wall's flag) while others share one velocity."""
    fl, wu = inputs.ldc_flags(n)
    nx, ny, nz = n
    fl[nz, 1, 1:nx + 1] = inputs.VELOCITY0 + 1       # z = nz - 1, y = 0: a second moving wall under the lid
    fl[1:nz + 1, ny // 2, nx // 2] = inputs.NOSLIP    # a no-slip post through the cavity
    fl[nz - 2, 3:6, 5:9] = inputs.VELOCITY0 + 2       # a moving block near the lid (velocity 2)
    wu = np.vstack([wu, [[0.0, 0.03, -0.01]], [[-0.02, 0.0, 0.015]]])
    return fl, wu


@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("prec", [8, 4])
def test_mixed_moving_walls_vs_oracle(prec, layout):
    n = (70, 23, 17)  # two x tiles (the second ragged), ragged y
    fl, wu = _mixed_wall_geometry(n)
    f0 = inputs.noise_pdfs(n, seed=29)
    ref = oracle.run(f0, fl, wu, 1.1, 25, nthreads=oracle.max_threads())
    got = run_gpu(n, fl, wu, f0, 25, prec, omega=1.1, patch=(70, 23, 17) if layout == 0 else (35, 23, 17),
                  layout=layout)
    assert max_fluid_diff(got, ref, fl) <= TOL[prec]


@pytest.mark.parametrize("layout", [0, 1])
def test_set_flags_again_rebuilds_wall_lists(layout):
    """set_flags after steps replaces the bounce-back list and the tiles' non-fluid
    bits: a run that starts from obstacles A, steps, switches to obstacles B and
    steps on matches the oracle run that does the same from B's switch point."""
    n = (48, 20, 14)
    fa, wu = inputs.ldc_flags(n)
    fa = inputs.add_obstacles(fa, 0.06, seed=41, kinds=(inputs.NOSLIP,))
    fb, _ = inputs.ldc_flags(n)
    fb = inputs.add_obstacles(fb, 0.05, seed=43, kinds=(inputs.NOSLIP, inputs.VELOCITY0 + 1))
    wub = np.vstack([wu, [[0.01, 0.0, 0.02]]])
    f0 = inputs.noise_pdfs(n, seed=47)
    L = lbm().Lattice(n, (24, 20, 14), 1.4, 8, layout=layout)
    try:
        L.set_flags(fa, wu)
        L.set_pdfs(f0)
        L.step(8)  # even: the AA layout accepts set_flags only in its swapped phase
        mid = L.get_pdfs()
        L.set_flags(fb, wub)
        L.set_pdfs(mid)  # cells fluid in B but solid in A start from zero
        L.step(9)
        got = L.get_pdfs()
    finally:
        L.close()
    ref = oracle.run(mid, fb, wub, 1.4, 9, nthreads=oracle.max_threads())
    assert max_fluid_diff(got, ref, fb) <= TOL[8]


@pytest.mark.parametrize("patch", [(70, 19, 13), (35, 19, 13)])
@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("prec", [8, 4])
def test_six_moving_walls_vs_oracle(prec, layout, patch):
    """Every side of the box a moving wall with its own velocity: all six sides are
    uniform walls, so the sweeps' face cells store the bounce-back through them
    (with the moving-wall term of their side), while the list handles the rims,
    edges and corners, where walls of two or three velocities meet; with two
    patches the sides between them are no walls (direct ghost stores)."""
    n = (70, 19, 13)
    fl = np.zeros((n[2] + 2, n[1] + 2, n[0] + 2), np.uint8)
    # later assignments win on the shared edges / corners
    fl[:, :, 0] = inputs.VELOCITY0 + 0
    fl[:, :, -1] = inputs.VELOCITY0 + 1
    fl[:, 0, :] = inputs.VELOCITY0 + 2
    fl[:, -1, :] = inputs.VELOCITY0 + 3
    fl[0, :, :] = inputs.VELOCITY0 + 4
    fl[-1, :, :] = inputs.VELOCITY0 + 5
    wu = np.array([[0.0, 0.02, -0.01], [0.0, -0.015, 0.02], [0.03, 0.0, 0.01],
                   [-0.02, 0.0, -0.025], [0.01, -0.02, 0.0], [0.05, 0.0, 0.0]])
    f0 = inputs.noise_pdfs(n, seed=53)
    ref = oracle.run(f0, fl, wu, 1.2, 21, nthreads=oracle.max_threads())
    got = run_gpu(n, fl, wu, f0, 21, prec, omega=1.2, layout=layout, patch=patch)
    assert max_fluid_diff(got, ref, fl) <= TOL[prec]


@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("n", [(40, 2, 5), (40, 5, 2), (1, 8, 9), (2, 3, 3), (66, 3, 4), (30, 6, 1), (24, 1, 7)])
def test_thin_boxes_vs_oracle(n, layout):
    """Boxes one to three cells thin along an axis: sides whose faces have no inner
    cells (uniform-wall detection needs at least 3 cells across the face) leave every
    link to the bounce-back list; with 3 cells the face has a single inner row; one
    cell thick, a face cell lies on both sides at once (found by the fuzz cases)."""
    fl, wu = inputs.ldc_flags(n)
    f0 = inputs.noise_pdfs(n, seed=61)
    ref = oracle.run(f0, fl, wu, 1.6, 17)
    for prec in (8, 4):
        got = run_gpu(n, fl, wu, f0, 17, prec, omega=1.6, layout=layout)
        assert max_fluid_diff(got, ref, fl) <= TOL[prec], (n, prec)
