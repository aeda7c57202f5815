"""Worker for tests/test_multi_gpu.py::test_full_size_bitwise_vs_one_gpu
(torchrun, one rank per GPU).

SURVEY 8(d) row 3: "1 vs N GPUs bitwise at full size for 10 steps".  The
BASELINE weak-scaling configuration -- 384^3 fp64 per GPU, process grid
1x1x2 / 1x2x2 / 2x2x2, lid-driven cavity, dyadic noise start -- runs 10 steps
decomposed over the ranks with the default exchange (fused NVLink stores);
also "strong" (768^3 in 384^3 patches), "patchy" (384^3 fp32 per GPU in 64^3
patches) and "aa" (256^3 fp64 per GPU, AA layout).
Every rank samples the PDFs of its brick at: every cell of the planes on both
sides of each process cut (which contain the edge lines where three bricks
meet), and seeded random cells.  Rank 0 then runs the whole domain on one GPU
(same patches, precision and layout) and compares the samples bitwise.  Exit
code 0 = pass.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

GRIDS = {2: (1, 1, 2), 4: (1, 2, 2), 8: (2, 2, 2)}
STEPS = 10
N = 384


def samples(domain, pgrid, rng):
    """Global cells: planes straddling each process cut (every cell) + random cells."""
    cells = []
    for a in range(3):
        for k in range(1, pgrid[a]):
            cut = k * domain[a] // pgrid[a]
            for c in (cut - 1, cut):
                # full plane would be 384*384 or more cells: take every cell of
                # every 7th line plus all lines within 1 of the other cuts
                other = [b for b in range(3) if b != a]
                u = np.arange(domain[other[0]])
                v = np.arange(domain[other[1]])
                keep_v = np.zeros(domain[other[1]], bool)
                keep_v[::7] = True
                for kk in range(1, pgrid[other[1]]):
                    cc = kk * domain[other[1]] // pgrid[other[1]]
                    keep_v[max(cc - 1, 0):cc + 1] = True
                keep_v[[0, -1]] = True
                vv = v[keep_v]
                g = np.stack(np.meshgrid(u, vv, indexing="ij"), -1).reshape(-1, 2)
                xyz = np.empty((g.shape[0], 3), np.int64)
                xyz[:, a] = c
                xyz[:, other[0]] = g[:, 0]
                xyz[:, other[1]] = g[:, 1]
                cells.append(xyz)
    cells.append(np.stack([rng.integers(0, domain[a], 20000) for a in range(3)], -1))
    return np.unique(np.concatenate(cells), axis=0)


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    config = sys.argv[1] if len(sys.argv) > 1 else "weak"
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    from paper_1007_1388_b200 import inputs, lbm
    pgrid = GRIDS[world]
    prec, layout = lbm.LBM_FP64, lbm.LBM_LAYOUT_AB
    if config == "weak":
        domain, patch = tuple(N * p for p in pgrid), (N, N, N)
    elif config == "strong":  # 768^3 in 8 patches of 384^3, 8 / world patches per GPU
        domain, patch = (2 * N, 2 * N, 2 * N), (N, N, N)
    elif config == "patchy":  # 384^3 fp32 per GPU in 216 patches of 64^3 (BASELINE config 5)
        domain, patch, prec = tuple(N * p for p in pgrid), (64, 64, 64), lbm.LBM_FP32
    else:  # aa: 256^3 fp64 per GPU, AA layout
        domain, patch, layout = tuple(256 * p for p in pgrid), (256, 256, 256), lbm.LBM_LAYOUT_AA
    fl, wu = inputs.ldc_flags(domain)
    cells = samples(domain, pgrid, np.random.default_rng(1007))
    obj = [lbm.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    L = lbm.Lattice(domain, patch, inputs.LDC_OMEGA, prec, device=local, rank=rank, nranks=world,
                    nccl_id=obj[0], proc_grid=pgrid, layout=layout)
    L.set_flags(fl, wu)
    L.init_noise(inputs.NOISE_SEED)
    L.step(STEPS)
    lo, hi = np.array(L.owned_lo), np.array(L.owned_hi)
    mine = np.all((cells >= lo) & (cells < hi), axis=1)
    part = (cells[mine], L.get_pdfs_at(cells[mine]))
    fused = L.info()["exchange_fused"]
    L.close()
    parts = [None] * world
    dist.all_gather_object(parts, part)
    ok = True
    if rank == 0:
        got_cells = np.concatenate([p[0] for p in parts])
        got = np.concatenate([p[1] for p in parts])
        assert got_cells.shape[0] == cells.shape[0], "every sample is owned by exactly one rank"
        with lbm.Lattice(domain, patch, inputs.LDC_OMEGA, prec, device=local, layout=layout) as L1:
            L1.set_flags(fl, wu)
            L1.init_noise(inputs.NOISE_SEED)
            L1.step(STEPS)
            ref = L1.get_pdfs_at(got_cells)
        same = np.array_equal(got, ref)
        moved = float(np.abs(got).max())
        print(f"config={config} world={world} grid={pgrid} domain={domain} patch={patch} fused={fused} "
              f"samples={got_cells.shape[0]} bitwise_vs_1gpu={same} max|f|={moved:.3e}", flush=True)
        ok = same and moved > 0
    flag = torch.tensor([1 if ok else 0])
    dist.broadcast(flag, 0)
    dist.destroy_process_group()
    sys.exit(0 if flag.item() == 1 else 1)


if __name__ == "__main__":
    main()
