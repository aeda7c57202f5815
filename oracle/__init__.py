"""CPU oracle of the D3Q19 LBGK pull stream-collide update (arXiv:1007.1388 §2.1).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It shares no code with ``paper_1007_1388_b200`` (the CUDA path) and
neither imports the other; inputs come from ``paper_1007_1388_b200.inputs``,
which holds no arithmetic of the method.

``liblbm_oracle.so`` is the plain C oracle (``lbm_oracle.c``, fp64,
``-O2 -ffp-contract=off``); ``exact`` is an exact-rational (``fractions``)
re-statement of the same update for boxes of a few cells.  Every function
cites the PAPER.md passage it follows (see ``lbm_oracle.c`` header).

Parity pins live in ``tests/test_oracle_*.py``; every oracle function is
pinned (no "parity unpinned" entries).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

Q = 19
_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liblbm_oracle.so")
_lib = None


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"oracle library missing: {_LIB_PATH} (run `make oracle`)")
    lib = ctypes.CDLL(_LIB_PATH)
    dp = ctypes.POINTER(ctypes.c_double)
    ip = ctypes.POINTER(ctypes.c_int)
    u8p = ctypes.POINTER(ctypes.c_uint8)
    lib.lbm_oracle_table.argtypes = [ip, dp, ip]
    lib.lbm_oracle_equilibrium.argtypes = [ctypes.c_double, dp, dp]
    lib.lbm_oracle_cell_moments.argtypes = [dp, dp, dp]
    lib.lbm_oracle_collide.argtypes = [dp, ctypes.c_double, dp]
    lib.lbm_oracle_check_flags.argtypes = [ctypes.c_int] * 3 + [ip, u8p, ctypes.c_int]
    lib.lbm_oracle_check_flags.restype = ctypes.c_int
    lib.lbm_oracle_step.argtypes = ([ctypes.c_int] * 3 + [ip, u8p, dp, ctypes.c_int, ctypes.c_double,
                                                           dp, dp, ctypes.c_int, ctypes.c_int, ctypes.c_int])
    lib.lbm_oracle_run.argtypes = ([ctypes.c_int] * 3 + [ip, u8p, dp, ctypes.c_int, ctypes.c_double,
                                                          ctypes.c_int, dp, ctypes.c_int])
    lib.lbm_oracle_run.restype = ctypes.c_int
    lib.lbm_oracle_macroscopic.argtypes = [ctypes.c_int] * 3 + [u8p, dp, dp, dp]
    lib.lbm_oracle_max_threads.restype = ctypes.c_int
    _lib = lib
    return lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _u8p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))


def _ip(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int))


def table():
    """Return (e[19,3] int, w[19] float64, opp[19] int) of the oracle's own frozen table."""
    lib = _load()
    e = np.zeros((Q, 3), np.int32)
    w = np.zeros(Q, np.float64)
    opp = np.zeros(Q, np.int32)
    lib.lbm_oracle_table(_ip(e), _dp(w), _ip(opp))
    return e, w, opp


def equilibrium(drho: float, u) -> np.ndarray:
    """Centred eq:feq."""
    lib = _load()
    uu = np.ascontiguousarray(u, np.float64)
    out = np.zeros(Q, np.float64)
    lib.lbm_oracle_equilibrium(float(drho), _dp(uu), _dp(out))
    return out


def cell_moments(f):
    """(drho, u) of one cell's 19 centred PDFs (u divides by rho0)."""
    lib = _load()
    ff = np.ascontiguousarray(f, np.float64)
    d = np.zeros(1, np.float64)
    u = np.zeros(3, np.float64)
    lib.lbm_oracle_cell_moments(_dp(ff), _dp(d), _dp(u))
    return float(d[0]), u


def collide(p, omega: float) -> np.ndarray:
    """BGK collision of pulled values p (eq:lbm)."""
    lib = _load()
    pp = np.ascontiguousarray(p, np.float64)
    out = np.zeros(Q, np.float64)
    lib.lbm_oracle_collide(_dp(pp), float(omega), _dp(out))
    return out


def _periodic(periodic):
    return np.ascontiguousarray([int(bool(v)) for v in periodic], np.int32)


def check_flags(shape, periodic, flags, nvel) -> int:
    nx, ny, nz = shape
    lib = _load()
    fl = np.ascontiguousarray(flags, np.uint8)
    return lib.lbm_oracle_check_flags(nx, ny, nz, _ip(_periodic(periodic)), _u8p(fl), int(nvel))


def run(f, flags, wall_u, omega, nsteps, periodic=(0, 0, 0), nthreads=1) -> np.ndarray:
    """Run nsteps oracle time steps.

    f: float64 [nz, ny, nx, 19] centred PDFs (copied; the result is returned).
    flags: uint8 [nz+2, ny+2, nx+2]; wall_u: float64 [nvel, 3].
    """
    lib = _load()
    f = np.array(f, dtype=np.float64, order="C", copy=True)
    nz, ny, nx, q = f.shape
    assert q == Q
    fl = np.ascontiguousarray(flags, np.uint8)
    assert fl.shape == (nz + 2, ny + 2, nx + 2)
    wu = np.ascontiguousarray(np.asarray(wall_u, np.float64).reshape(-1, 3))
    if wu.size == 0:
        wu = np.zeros((1, 3), np.float64)
        nvel = 0
    else:
        nvel = wu.shape[0]
    rc = lib.lbm_oracle_run(nx, ny, nz, _ip(_periodic(periodic)), _u8p(fl), _dp(wu), nvel,
                            float(omega), int(nsteps), _dp(f), int(nthreads))
    if rc != 0:
        raise ValueError(f"oracle rejected the input (code {rc})")
    return f


def step_slab(src, dst, flags, wall_u, omega, z0, z1, periodic=(0, 0, 0), nthreads=1):
    """One oracle time step over interior planes [z0, z1), src -> dst (in place in dst)."""
    lib = _load()
    nz, ny, nx, _ = src.shape
    wu = np.ascontiguousarray(np.asarray(wall_u, np.float64).reshape(-1, 3))
    nvel = wu.shape[0]
    if nvel == 0:
        wu = np.zeros((1, 3))
    lib.lbm_oracle_step(nx, ny, nz, _ip(_periodic(periodic)), _u8p(flags), _dp(wu), nvel,
                        float(omega), _dp(src), _dp(dst), int(z0), int(z1), int(nthreads))


def macroscopic(f, flags):
    """(rho[nz,ny,nx], u[nz,ny,nx,3]); rho = rho0 + sum f~ at fluid cells, 0 elsewhere."""
    lib = _load()
    f = np.ascontiguousarray(f, np.float64)
    nz, ny, nx, _ = f.shape
    fl = np.ascontiguousarray(flags, np.uint8)
    rho = np.zeros((nz, ny, nx), np.float64)
    u = np.zeros((nz, ny, nx, 3), np.float64)
    lib.lbm_oracle_macroscopic(nx, ny, nz, _u8p(fl), _dp(f), _dp(rho), _dp(u))
    return rho, u


def max_threads() -> int:
    return int(_load().lbm_oracle_max_threads())
