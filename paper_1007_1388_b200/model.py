"""Performance model of the paper (host-side arithmetic, no GPU).

* bytes per lattice-cell update, n_bytes = n_stencil (n_loads + n_stores) s_PDF
  (P:1075-1082): 152 / 304 B on a GPU (no write-allocate), 228 / 456 B on a CPU
  (read-for-ownership adds one load per store).
* kernel and transfer times of Table 1 (tab:HybridComputingEstimate):
      t_k = n^3 / P,     t_t = 2 n^2 n_PDF n_plane s_PDF / B
  for a cubic domain of n^3 cells whose 6 boundary planes exchange 5 PDFs per
  cell.
* the same model re-parameterised for a B200 brick: sweep time from the HBM
  roofline, halo time from the NVLink bandwidth, with the exact halo volume of
  the D3Q19 exchange (5 PDFs per face cell, 1 per edge cell; no corners).
"""
from __future__ import annotations

Q = 19


def bytes_per_update(s_pdf: int, gpu: bool = True, n_stencil: int = Q) -> int:
    """n_bytes = n_stencil * (n_loads + n_stores) * s_PDF; CPUs pay one extra load
    per store for read-for-ownership."""
    loads, stores = 1, 1
    if not gpu:
        loads += stores
    return n_stencil * (loads + stores) * s_pdf


def roofline_mflups(bandwidth_gbs: float, s_pdf: int, gpu: bool = True) -> float:
    """Upper-bound MFLUPS = bandwidth / bytes per update."""
    return bandwidth_gbs * 1e9 / bytes_per_update(s_pdf, gpu) / 1e6


def t_kernel(n: int, mflups: float) -> float:
    """t_k = n^3 / P in seconds."""
    return n ** 3 / (mflups * 1e6)


def t_transfer(n: int, bandwidth_gbs: float, s_pdf: int, n_pdf: int = 5, n_plane: int = 6) -> float:
    """t_t = 2 n^2 n_PDF n_plane s_PDF / B in seconds (both directions)."""
    return 2 * n * n * n_pdf * n_plane * s_pdf / (bandwidth_gbs * 1e9)


def table1(n: int = 100, kernel_ms: float = 3.3, pcie_gbs: float = 5.0, ib_gbs: float = 3.0, s_pdf: int = 4):
    """Reproduce Table 1: returns dict of times (ms) and MFLUPS estimates."""
    tk = kernel_ms * 1e-3
    tp = t_transfer(n, pcie_gbs, s_pdf)
    ti = t_transfer(n, ib_gbs, s_pdf)
    return {"compute_ms": tk * 1e3, "pcie_ms": tp * 1e3, "ib_ms": ti * 1e3,
            "total_I_ms": (tk + tp) * 1e3, "mflups_I": n ** 3 / (tk + tp) / 1e6,
            "total_I_II_ms": (tk + tp + ti) * 1e3, "mflups_I_II": n ** 3 / (tk + tp + ti) / 1e6}


def halo_bytes(brick, proc_coord, proc_grid, s_pdf: int, periodic=(0, 0, 0)) -> int:
    """Bytes a rank sends per step for a brick of cells (nx, ny, nz): 5 PDFs per
    cell of every face with a neighbouring rank, 1 per cell of every such edge."""
    total = 0
    dirs = [(dx, dy, dz) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)
            if 1 <= abs(dx) + abs(dy) + abs(dz) <= 2]
    for d in dirs:
        ok = True
        for a in range(3):
            c = proc_coord[a] + d[a]
            if (c < 0 or c >= proc_grid[a]) and not (periodic[a] and proc_grid[a] > 1):
                ok = False
            if d[a] != 0 and proc_grid[a] == 1:
                ok = False  # wraps onto itself: local, not sent
        if not ok:
            continue
        cells = 1
        for a in range(3):
            if d[a] == 0:
                cells *= brick[a]
        nz = sum(1 for v in d if v != 0)
        total += cells * (5 if nz == 1 else 1) * s_pdf
    return total


def b200_step_estimate(brick, proc_coord, proc_grid, s_pdf: int, hbm_gbs: float, nvlink_gbs: float = 770.0,
                       overlap: bool = True) -> dict:
    """Per-step time estimate of one rank on B200: sweep at the HBM roofline plus
    the halo at the NVLink per-direction bandwidth (hidden when overlapped)."""
    cells = brick[0] * brick[1] * brick[2]
    t_sweep = cells * bytes_per_update(s_pdf) / (hbm_gbs * 1e9)
    hb = halo_bytes(brick, proc_coord, proc_grid, s_pdf)
    t_halo = hb / (nvlink_gbs * 1e9)
    t = max(t_sweep, t_halo) if overlap else t_sweep + t_halo
    return {"sweep_ms": t_sweep * 1e3, "halo_bytes": hb, "halo_ms": t_halo * 1e3, "step_ms": t * 1e3,
            "mflups": cells / t / 1e6}


def hetero_balance(gpu_mflups: float, cpu_mflups: float, n_gpu: int, n_cpu: int, block_cells: int,
                   gpu_blocks: int | None = None) -> dict:
    """Static block-count balancing of a heterogeneous GPU + CPU node (P:989-1000,
    sec:hetero_perf): every CPU process owns one Block, every GPU process b Blocks,
    and one step takes as long as the slowest process,
        t = max(b * cells / r_gpu, cells / r_cpu),
    so the balanced count is b = round(r_gpu / r_cpu) (r_gpu: a GPU process's rate
    with many Blocks, r_cpu: a CPU process's rate).  Returns b, the step time and
    the node rate (n_gpu b + n_cpu) cells / t; the exchange overhead the paper
    names is not modelled.  gpu_blocks overrides b."""
    b = max(1, round(gpu_mflups / cpu_mflups)) if gpu_blocks is None else gpu_blocks
    t_gpu = b * block_cells / (gpu_mflups * 1e6)
    t_cpu = block_cells / (cpu_mflups * 1e6)
    t = max(t_gpu, t_cpu) if n_cpu else t_gpu
    cells = (n_gpu * b + n_cpu) * block_cells
    gpu_only = n_gpu * gpu_mflups
    return {"gpu_blocks": b, "step_s": t, "node_mflups": cells / t / 1e6, "gpu_only_mflups": gpu_only,
            "gain": cells / t / 1e6 / gpu_only - 1.0}
