"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This module holds NO arithmetic of the method (no equilibrium, moments,
streaming or bounce-back): only geometry (cell flags), wall-velocity tables
and the seeded initial PDF noise.  It imports nothing from ``oracle/`` nor
from the CUDA binding, and both sides receive its arrays as inputs.

Workload recipe:
  * lid-driven cavity ("Lid Driven Cavity scenarios in 3D"): a
    one-cell no-slip shell around an all-fluid box, the top plane z = nz is a
    moving lid with u_w = (U, 0, 0), U = 0.05, tau = 0.65 (omega = 1/0.65);
    the lid flag is written after the no-slip shell, so it wins on the top
    plane's edges and corners.
  * initial state: rest (all-zero centred PDFs) or dyadic noise
    f~ = k / 2**20, k uniform in [-1024, 1024], drawn by a counter-based
    generator (splitmix64 of the global (cell, q) index) so that the device
    initialiser ``lbm_init_noise`` draws the identical value at any size.
  * flag values: 0 fluid, 1 no-slip wall, 2+k wall moving with wall_u[k].
"""
from __future__ import annotations

import numpy as np

FLUID, NOSLIP, VELOCITY0 = 0, 1, 2
Q = 19
LDC_U = 0.05
LDC_TAU = 0.65
LDC_OMEGA = 1.0 / LDC_TAU
NOISE_SEED = 1388

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def shell_flags(n, periodic=(0, 0, 0)) -> np.ndarray:
    """uint8 [nz+2, ny+2, nx+2]: interior fluid, one-cell NOSLIP shell on every
    non-periodic axis (periodic axes: shell cells mirror nothing and are fluid)."""
    nx, ny, nz = n
    fl = np.zeros((nz + 2, ny + 2, nx + 2), np.uint8)
    if not periodic[0]:
        fl[:, :, 0] = NOSLIP
        fl[:, :, -1] = NOSLIP
    if not periodic[1]:
        fl[:, 0, :] = NOSLIP
        fl[:, -1, :] = NOSLIP
    if not periodic[2]:
        fl[0, :, :] = NOSLIP
        fl[-1, :, :] = NOSLIP
    return fl


def ldc_flags(n, periodic=(0, 0, 0)):
    """Lid-driven cavity: returns (flags, wall_u[1,3]); lid = plane z = nz."""
    fl = shell_flags(n, periodic)
    fl[-1, :, :] = VELOCITY0
    return fl, np.array([[LDC_U, 0.0, 0.0]], np.float64)


def couette_flags(nz, U=LDC_U):
    """Plane Couette channel: 1 x 1 x nz, periodic x and y, no-slip plane z = -1,
    lid z = nz moving with (U, 0, 0).  Returns (flags, wall_u, periodic)."""
    fl = np.zeros((nz + 2, 3, 3), np.uint8)
    fl[0] = NOSLIP
    fl[-1] = VELOCITY0
    return fl, np.array([[U, 0.0, 0.0]], np.float64), (1, 1, 0)


def add_obstacles(flags, fraction, seed, kinds=(NOSLIP,)) -> np.ndarray:
    """Randomly turn `fraction` of the interior cells into walls of the given kinds."""
    fl = flags.copy()
    rng = np.random.default_rng(seed)
    inner = fl[1:-1, 1:-1, 1:-1]
    mask = rng.random(inner.shape) < fraction
    kind = rng.choice(np.asarray(kinds, np.uint8), size=inner.shape)
    inner[mask] = kind[mask]
    return fl


def _splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = (x + np.uint64(0x9E3779B97F4A7C15)) & _M64
        z = x
        z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & _M64
        z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & _M64
        return z ^ (z >> np.uint64(31))


def noise_k(global_index: np.ndarray, q: np.ndarray, seed: int = NOISE_SEED) -> np.ndarray:
    """Counter-based integer k in [-1024, 1024] for (global cell index, q).
    key = (index*19 + q) + seed * 0x9E3779B97F4A7C15 (mod 2**64)."""
    gi = np.asarray(global_index, np.uint64)
    qq = np.asarray(q, np.uint64)
    with np.errstate(over="ignore"):
        key = (gi * np.uint64(Q) + qq + np.uint64(seed) * np.uint64(0x9E3779B97F4A7C15)) & _M64
    h = _splitmix64(key)
    return (h % np.uint64(2049)).astype(np.int64) - 1024


def noise_pdfs(domain, lo=(0, 0, 0), hi=None, seed: int = NOISE_SEED) -> np.ndarray:
    """Dyadic noise f~ = k / 2**20 over the box [lo, hi) of a global domain
    (nx, ny, nz); float64 [hz-lz, hy-ly, hx-lx, 19].  Exact in fp32 and fp64."""
    nx, ny, nz = domain
    if hi is None:
        hi = (nx, ny, nz)
    xs = np.arange(lo[0], hi[0], dtype=np.uint64)
    ys = np.arange(lo[1], hi[1], dtype=np.uint64)
    zs = np.arange(lo[2], hi[2], dtype=np.uint64)
    out = np.empty((len(zs), len(ys), len(xs), Q), np.float64)
    qq = np.arange(Q, dtype=np.uint64)
    for iz, z in enumerate(zs):
        gi = ((z * np.uint64(ny) + ys[:, None]) * np.uint64(nx) + xs[None, :])
        k = noise_k(gi[:, :, None], qq[None, None, :], seed)
        out[iz] = k.astype(np.float64) * (2.0 ** -20)
    return out


def noise_at(domain, cells, seed: int = NOISE_SEED) -> np.ndarray:
    """Noise PDFs at an explicit list of global cells [(x, y, z), ...] -> [n, 19]."""
    nx, ny, nz = domain
    c = np.asarray(cells, np.uint64).reshape(-1, 3)
    gi = (c[:, 2] * np.uint64(ny) + c[:, 1]) * np.uint64(nx) + c[:, 0]
    k = noise_k(gi[:, None], np.arange(Q, dtype=np.uint64)[None, :], seed)
    return k.astype(np.float64) * (2.0 ** -20)
