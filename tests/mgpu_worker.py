"""Worker for tests/test_multi_gpu.py (launched by torchrun, one rank per GPU).

Runs the lid-driven cavity decomposed over the ranks (NCCL ghost exchange,
overlap on and off), gathers the owned bricks on rank 0 and checks them
bitwise against a single-GPU run of the same lattice and against the oracle.
Exit code 0 = pass.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    from paper_1007_1388_b200 import inputs, lbm
    domain, patch, periodic = (48, 40, 64), (24, 20, 16), (1, 0, 0)
    steps = 60
    fl, wu = inputs.ldc_flags(domain, periodic)
    fl = inputs.add_obstacles(fl, 0.03, seed=13)
    ok = True
    results = {}
    masses = {}
    # (prec, overlap, layout, exchange): AB uses the fused sweep + NVLink peer stores
    # by default; "nccl" forces pack -> NCCL -> unpack (LBM_EXCHANGE=nccl)
    # plus process grids that split x (the driver's 8-GPU run is 2x2x2)
    grids = {2: [(0, 0, 0), (2, 1, 1)], 4: [(0, 0, 0), (2, 2, 1), (2, 1, 2)]}.get(world, [(0, 0, 0)])
    # "fused_copies": fused exchange with same-GPU ghost copies instead of the
    # sweep's direct ghost stores (LBM_LOCAL_DIRECT=0)
    combos = [(8, 1, 0, "fused", grids[0]), (4, 1, 0, "fused", grids[0]), (8, 1, 0, "fused_copies", grids[0]),
              (4, 1, 1, "fused_copies", grids[0]),
              (8, 1, 0, "nccl", grids[0]), (8, 1, 1, "fused", grids[0]), (4, 1, 1, "fused", grids[0]),
              (8, 0, 0, "nccl", grids[0]), (4, 1, 0, "nccl", grids[0]), (8, 1, 1, "nccl", grids[0]),
              (4, 0, 1, "nccl", grids[0])]
    for pg in grids[1:]:
        combos += [(8, 1, 0, "fused", pg), (4, 1, 0, "fused", pg), (8, 1, 0, "nccl", pg), (8, 1, 1, "nccl", pg),
                   (8, 1, 1, "fused", pg)]
    for prec, overlap, layout, exch, pgrid in combos:
        if exch == "nccl":
            os.environ["LBM_EXCHANGE"] = "nccl"
        else:
            os.environ.pop("LBM_EXCHANGE", None)
        if exch == "fused_copies":
            os.environ["LBM_LOCAL_DIRECT"] = "0"
        else:
            os.environ.pop("LBM_LOCAL_DIRECT", None)
        if True:
            obj = [lbm.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            L = lbm.Lattice(domain, patch, inputs.LDC_OMEGA, prec, device=local, rank=rank, nranks=world,
                            nccl_id=obj[0], periodic=periodic, overlap=overlap, layout=layout, proc_grid=pgrid)
            L.set_flags(fl, wu)
            f0 = inputs.noise_pdfs(domain, L.owned_lo, L.owned_hi)
            L.set_pdfs(f0)
            L.step(steps)
            mine = (L.owned_lo, L.owned_hi, L.get_pdfs())
            mass = L.total_mass()  # collective: every rank calls it
            info = L.info()
            L.close()
            parts = [None] * world
            dist.all_gather_object(parts, mine)
            if rank == 0:
                full = np.zeros((domain[2], domain[1], domain[0], 19))
                for lo, hi, a in parts:
                    full[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]] = a
                results[(prec, overlap, layout, exch, tuple(pgrid))] = full
                masses[(prec, overlap, layout, exch, tuple(pgrid))] = mass
                assert info["exchange_fused"] == (1 if exch.startswith("fused") else 0), info["exchange_fused"]
                # 8+ patches per rank: same-GPU neighbours take the direct ghost stores
                assert info["local_direct"] == (0 if exch == "fused_copies" else 1), info
                print(f"prec={prec} overlap={overlap} layout={layout} exchange={exch} peers={info['peers']} "
                      f"halo={info['halo_bytes_remote_per_step']} local_direct={info['local_direct']}", flush=True)
    if rank == 0:
        import oracle
        ref = oracle.run(inputs.noise_pdfs(domain), fl, wu, inputs.LDC_OMEGA, steps, periodic=periodic,
                         nthreads=oracle.max_threads())
        mask = fl[1:-1, 1:-1, 1:-1] == 0
        for prec in (8, 4):
            with lbm.Lattice(domain, patch, inputs.LDC_OMEGA, prec, device=local, periodic=periodic) as L:
                L.set_flags(fl, wu)
                L.set_pdfs(inputs.noise_pdfs(domain))
                L.step(steps)
                single = L.get_pdfs()
                single_mass = L.total_mass()
            for (p2, overlap, layout, exch, pgrid), res in results.items():
                if p2 != prec:
                    continue
                same = np.array_equal(res, single)
                dm = abs(masses[(p2, overlap, layout, exch, pgrid)] - single_mass)
                err = float(np.abs(res[mask] - ref[mask]).max())
                tol = 1e-12 if prec == 8 else 1e-5
                print(f"prec={prec} overlap={overlap} layout={layout} exchange={exch} grid={pgrid} bitwise_vs_1gpu={same} "
                      f"max|oracle diff|={err:.3e} |total mass - 1 GPU|={dm:.1e}", flush=True)
                ok = ok and same and err <= tol and dm <= 1e-9
    flag = torch.tensor([1 if ok else 0])
    dist.broadcast(flag, 0)
    dist.destroy_process_group()
    sys.exit(0 if flag.item() == 1 else 1)


if __name__ == "__main__":
    main()
