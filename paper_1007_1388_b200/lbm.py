"""ctypes binding of ``liblbm_b200.so`` (C ABI in ``include/lbm.h``).

Argument marshalling only: every step of the update runs in the library's
sm_100a kernels.  Importing this module loads the CUDA library and raises
ImportError if it is missing (there is no CPU fallback).
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

Q = 19
LBM_FP32, LBM_FP64 = 4, 8
LBM_FLUID, LBM_NOSLIP, LBM_VELOCITY0 = 0, 1, 2
LBM_EXCHANGE_AUTO, LBM_EXCHANGE_FORCE_BUFFERS, LBM_EXCHANGE_SELF_PEER = 0, 1, 2
LBM_LAYOUT_AB, LBM_LAYOUT_AA = 0, 1
NCCL_ID_BYTES = 128
NPHASES = 8
PHASES = ("sweep", "sweep_shell", "sweep_interior", "pack", "nccl", "unpack", "step", "reserved")
STATUS = {0: "LBM_OK", 1: "LBM_ERR_ARG", 2: "LBM_ERR_STATE", 3: "LBM_ERR_OOM", 4: "LBM_ERR_CUDA",
          5: "LBM_ERR_NCCL", 6: "LBM_ERR_INTERNAL"}

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "liblbm_b200.so")
# LBM_LIBRARY selects another build of the same ABI -- the checked build
# (liblbm_b200_checked.so, tools/sanitize_cases.py); there is no fallback.
LIB_PATH = os.environ.get("LBM_LIBRARY") or LIB_PATH

# Every symbol include/lbm.h declares (checked by tests/test_abi.py).
EXPORTED = ("lbm_abi_version", "lbm_config_default", "lbm_create", "lbm_create_ex", "lbm_destroy",
            "lbm_set_flags", "lbm_get_flags", "lbm_set_pdfs", "lbm_init_noise", "lbm_step",
            "lbm_step_async", "lbm_synchronize", "lbm_get_pdfs", "lbm_get_pdfs_at",
            "lbm_get_macroscopic", "lbm_total_mass", "lbm_get_info", "lbm_set_timing", "lbm_get_stream",
            "lbm_last_error", "lbm_nccl_unique_id", "lbm_plan")


class LbmConfig(ctypes.Structure):
    _fields_ = [("domain", ctypes.c_int64 * 3), ("patch", ctypes.c_int32 * 3), ("omega", ctypes.c_double),
                ("precision", ctypes.c_int32), ("periodic", ctypes.c_int32 * 3), ("device", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("nranks", ctypes.c_int32), ("proc_grid", ctypes.c_int32 * 3),
                ("nccl_unique_id", ctypes.c_void_p), ("exchange_mode", ctypes.c_int32),
                ("overlap", ctypes.c_int32), ("use_graphs", ctypes.c_int32), ("stream", ctypes.c_void_p),
                ("layout", ctypes.c_int32)]


class LbmInfo(ctypes.Structure):
    _fields_ = [("domain", ctypes.c_int64 * 3), ("patch", ctypes.c_int32 * 3), ("precision", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("nranks", ctypes.c_int32), ("proc_grid", ctypes.c_int32 * 3),
                ("proc_coord", ctypes.c_int32 * 3), ("owned_lo", ctypes.c_int64 * 3),
                ("owned_hi", ctypes.c_int64 * 3), ("patches_local", ctypes.c_int32),
                ("patches_global", ctypes.c_int32), ("peers", ctypes.c_int32),
                ("messages_remote", ctypes.c_int32), ("fluid_cells_local", ctypes.c_int64),
                ("fluid_cells_global", ctypes.c_int64), ("steps_done", ctypes.c_int64),
                ("bytes_per_step_algorithmic", ctypes.c_double), ("halo_bytes_remote_per_step", ctypes.c_int64),
                ("halo_bytes_local_per_step", ctypes.c_int64), ("kernel_launches", ctypes.c_int64),
                ("device_bytes", ctypes.c_int64), ("phase_ms", ctypes.c_double * NPHASES),
                ("phase_count", ctypes.c_int64 * NPHASES), ("row_pitch_elems", ctypes.c_int64),
                ("align_bytes", ctypes.c_int32), ("graphs_active", ctypes.c_int32), ("layout", ctypes.c_int32),
                ("aa_phase", ctypes.c_int32), ("exchange_fused", ctypes.c_int32),
                ("local_pull", ctypes.c_int32), ("local_direct", ctypes.c_int32),
                ("overlap_active", ctypes.c_int32), ("nccl_ranks", ctypes.c_int32),
                ("fused_peers", ctypes.c_int32), ("reserved0", ctypes.c_int32)]

    def to_dict(self) -> dict:
        out = {}
        for name, _ in self._fields_:
            v = getattr(self, name)
            out[name] = list(v) if hasattr(v, "__len__") else v
        return out


class LbmMsg(ctypes.Structure):
    _fields_ = [("peer", ctypes.c_int32), ("send", ctypes.c_int32), ("patch_local", ctypes.c_int32),
                ("patch_remote", ctypes.c_int32), ("dir", ctypes.c_int32 * 3), ("nq", ctypes.c_int32),
                ("cells", ctypes.c_int64), ("offset", ctypes.c_int64)]


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"CUDA library missing: {LIB_PATH} -- build it with `make lib` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.POINTER
    c = ctypes
    sig = {
        "lbm_abi_version": (c.c_int32, []),
        "lbm_config_default": (None, [P(LbmConfig)]),
        "lbm_create": (c.c_int, [P(c.c_int64), P(c.c_int32), c.c_double, c.c_int32, P(c.c_void_p)]),
        "lbm_create_ex": (c.c_int, [P(LbmConfig), P(c.c_void_p)]),
        "lbm_destroy": (c.c_int, [c.c_void_p]),
        "lbm_set_flags": (c.c_int, [c.c_void_p, c.c_void_p, c.c_void_p, c.c_int32]),
        "lbm_get_flags": (c.c_int, [c.c_void_p, c.c_void_p]),
        "lbm_set_pdfs": (c.c_int, [c.c_void_p, c.c_void_p]),
        "lbm_init_noise": (c.c_int, [c.c_void_p, c.c_uint64]),
        "lbm_step": (c.c_int, [c.c_void_p, c.c_int64]),
        "lbm_step_async": (c.c_int, [c.c_void_p, c.c_int64]),
        "lbm_synchronize": (c.c_int, [c.c_void_p]),
        "lbm_get_pdfs": (c.c_int, [c.c_void_p, c.c_void_p]),
        "lbm_get_pdfs_at": (c.c_int, [c.c_void_p, c.c_void_p, c.c_int64, c.c_void_p]),
        "lbm_get_macroscopic": (c.c_int, [c.c_void_p, c.c_void_p, c.c_void_p]),
        "lbm_total_mass": (c.c_int, [c.c_void_p, P(c.c_double)]),
        "lbm_get_info": (c.c_int, [c.c_void_p, P(LbmInfo)]),
        "lbm_set_timing": (c.c_int, [c.c_void_p, c.c_int32]),
        "lbm_get_stream": (c.c_int, [c.c_void_p, P(c.c_void_p)]),
        "lbm_last_error": (c.c_char_p, [c.c_void_p]),
        "lbm_nccl_unique_id": (c.c_int, [c.c_void_p, c.c_int64]),
        "lbm_plan": (c.c_int, [P(LbmConfig), P(LbmInfo), P(LbmMsg), c.c_int32, P(c.c_int32)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.lbm_abi_version() != 1:
        raise ImportError("liblbm_b200.so ABI version mismatch")
    return lib


_lib = _load()


class LbmError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def _ptr(a: np.ndarray) -> ctypes.c_void_p:
    return ctypes.c_void_p(a.ctypes.data)


def default_config(domain, patch=None, omega=1.0 / 0.65, precision=LBM_FP64, periodic=(0, 0, 0), device=-1,
                   rank=0, nranks=1, proc_grid=(0, 0, 0), exchange_mode=LBM_EXCHANGE_AUTO, overlap=1,
                   use_graphs=1, stream=None, layout=LBM_LAYOUT_AB) -> LbmConfig:
    cfg = LbmConfig()
    _lib.lbm_config_default(ctypes.byref(cfg))
    patch = domain if patch is None else patch
    for a in range(3):
        cfg.domain[a] = int(domain[a])
        cfg.patch[a] = int(patch[a])
        cfg.periodic[a] = int(bool(periodic[a]))
        cfg.proc_grid[a] = int(proc_grid[a])
    cfg.omega = float(omega)
    cfg.precision = int(precision)
    cfg.device = int(device)
    cfg.rank = int(rank)
    cfg.nranks = int(nranks)
    cfg.exchange_mode = int(exchange_mode)
    cfg.overlap = int(overlap)
    cfg.use_graphs = int(use_graphs)
    cfg.stream = stream
    cfg.layout = int(layout)
    return cfg


def plan(cfg: LbmConfig):
    """Host-only decomposition + remote message plan (no GPU needed)."""
    info = LbmInfo()
    n = ctypes.c_int32(0)
    st = _lib.lbm_plan(ctypes.byref(cfg), ctypes.byref(info), None, 0, ctypes.byref(n))
    if st != 0:
        raise LbmError(st, _lib.lbm_last_error(None).decode())
    msgs = (LbmMsg * max(n.value, 1))()
    st = _lib.lbm_plan(ctypes.byref(cfg), ctypes.byref(info), msgs, n.value, ctypes.byref(n))
    if st != 0:
        raise LbmError(st, _lib.lbm_last_error(None).decode())
    out = [dict(peer=m.peer, send=m.send, patch_local=m.patch_local, patch_remote=m.patch_remote,
                dir=tuple(m.dir), nq=m.nq, cells=m.cells, offset=m.offset) for m in msgs[:n.value]]
    return info.to_dict(), out


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(NCCL_ID_BYTES)
    st = _lib.lbm_nccl_unique_id(buf, NCCL_ID_BYTES)
    if st != 0:
        raise LbmError(st, _lib.lbm_last_error(None).decode())
    return buf.raw


def _check_out(a, shape, name):
    """The library writes the whole owned box into caller buffers: refuse anything
    that is not a C-contiguous float64 array of exactly that shape."""
    if not isinstance(a, np.ndarray) or a.dtype != np.float64 or not a.flags.c_contiguous \
            or tuple(a.shape) != tuple(shape) or not a.flags.writeable:
        raise ValueError(f"{name} must be a writeable C-contiguous float64 array of shape {tuple(shape)}")


class Lattice:
    """One rank's view of the patch-decomposed lattice (owns an lbm_ctx)."""

    def __init__(self, domain: Sequence[int], patch: Optional[Sequence[int]] = None, omega: float = 1.0 / 0.65,
                 precision: int = LBM_FP64, *, minimal: bool = False, nccl_id: Optional[bytes] = None, **kw):
        self._ctx = ctypes.c_void_p()
        self._id_buf = None
        if minimal:
            dom = (ctypes.c_int64 * 3)(*[int(v) for v in domain])
            pat = (ctypes.c_int32 * 3)(*[int(v) for v in (patch or domain)])
            st = _lib.lbm_create(dom, pat, float(omega), int(precision), ctypes.byref(self._ctx))
        else:
            cfg = default_config(domain, patch, omega, precision, **kw)
            if nccl_id is not None:
                self._id_buf = ctypes.create_string_buffer(bytes(nccl_id), NCCL_ID_BYTES)
                cfg.nccl_unique_id = ctypes.cast(self._id_buf, ctypes.c_void_p)
            st = _lib.lbm_create_ex(ctypes.byref(cfg), ctypes.byref(self._ctx))
        if st != 0:
            raise LbmError(st, _lib.lbm_last_error(None).decode())
        self.domain = tuple(int(v) for v in domain)
        self.precision = int(precision)
        info = self.info()
        self.owned_lo = tuple(info["owned_lo"])
        self.owned_hi = tuple(info["owned_hi"])
        self.owned_shape = tuple(self.owned_hi[a] - self.owned_lo[a] for a in range(3))

    # -- plumbing
    def _check(self, st: int):
        if st != 0:
            raise LbmError(st, _lib.lbm_last_error(self._ctx).decode())

    def close(self):
        if self._ctx:
            _lib.lbm_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- API
    def set_flags(self, flags: np.ndarray, wall_u=None):
        fl = np.ascontiguousarray(flags, np.uint8)
        nx, ny, nz = self.domain
        if fl.shape != (nz + 2, ny + 2, nx + 2):
            raise ValueError(f"flags must have shape {(nz + 2, ny + 2, nx + 2)}")
        if wall_u is None or len(wall_u) == 0:
            wu = None
            nvel = 0
        else:
            wu = np.ascontiguousarray(np.asarray(wall_u, np.float64).reshape(-1, 3))
            nvel = wu.shape[0]
        self._check(_lib.lbm_set_flags(self._ctx, _ptr(fl), _ptr(wu) if wu is not None else None, nvel))

    def get_flags(self) -> np.ndarray:
        sx, sy, sz = self.owned_shape
        out = np.empty((sz + 2, sy + 2, sx + 2), np.uint8)
        self._check(_lib.lbm_get_flags(self._ctx, _ptr(out)))
        return out

    def set_pdfs(self, f: np.ndarray):
        sx, sy, sz = self.owned_shape
        a = np.ascontiguousarray(f, np.float64)
        if a.shape != (sz, sy, sx, Q):
            raise ValueError(f"pdfs must have shape {(sz, sy, sx, Q)}")
        self._check(_lib.lbm_set_pdfs(self._ctx, _ptr(a)))

    def init_noise(self, seed: int):
        self._check(_lib.lbm_init_noise(self._ctx, ctypes.c_uint64(int(seed))))

    def step(self, n: int = 1):
        self._check(_lib.lbm_step(self._ctx, int(n)))

    def step_async(self, n: int = 1):
        self._check(_lib.lbm_step_async(self._ctx, int(n)))

    def synchronize(self):
        self._check(_lib.lbm_synchronize(self._ctx))

    def get_pdfs(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        sx, sy, sz = self.owned_shape
        if out is None:
            out = np.empty((sz, sy, sx, Q), np.float64)
        _check_out(out, (sz, sy, sx, Q), "out")
        self._check(_lib.lbm_get_pdfs(self._ctx, _ptr(out)))
        return out

    def get_pdfs_at(self, cells) -> np.ndarray:
        c = np.ascontiguousarray(np.asarray(cells, np.int64).reshape(-1, 3))
        out = np.empty((c.shape[0], Q), np.float64)
        self._check(_lib.lbm_get_pdfs_at(self._ctx, _ptr(c), c.shape[0], _ptr(out)))
        return out

    def get_macroscopic(self, rho_out: Optional[np.ndarray] = None, u_out: Optional[np.ndarray] = None):
        sx, sy, sz = self.owned_shape
        rho = np.empty((sz, sy, sx), np.float64) if rho_out is None else rho_out
        u = np.empty((sz, sy, sx, 3), np.float64) if u_out is None else u_out
        _check_out(rho, (sz, sy, sx), "rho_out")
        _check_out(u, (sz, sy, sx, 3), "u_out")
        self._check(_lib.lbm_get_macroscopic(self._ctx, _ptr(rho), _ptr(u)))
        return rho, u

    def total_mass(self) -> float:
        """Sum of rho over all fluid cells of the whole lattice (a collective across ranks)."""
        m = ctypes.c_double()
        self._check(_lib.lbm_total_mass(self._ctx, ctypes.byref(m)))
        return m.value

    def info(self) -> dict:
        info = LbmInfo()
        self._check(_lib.lbm_get_info(self._ctx, ctypes.byref(info)))
        return info.to_dict()

    def set_timing(self, enable: bool):
        self._check(_lib.lbm_set_timing(self._ctx, int(bool(enable))))

    def stream(self) -> int:
        s = ctypes.c_void_p()
        self._check(_lib.lbm_get_stream(self._ctx, ctypes.byref(s)))
        return s.value or 0

    def phase_ms(self) -> dict:
        inf = self.info()
        return {PHASES[i]: (inf["phase_ms"][i], inf["phase_count"][i]) for i in range(NPHASES)}
