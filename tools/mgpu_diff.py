"""Where does an N-rank run differ from one GPU?  Debug aid (torchrun, one rank
per GPU): runs the multi-GPU test's cavity for STEPS (env, comma list) and
prints, per axis and direction, how many PDF values differ from the one-GPU run.
Env GRAPHS=0 disables CUDA graphs, ONE_BY_ONE=1 steps one at a time."""
import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch, torch.distributed as dist
rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"]); local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local); dist.init_process_group("gloo")
from paper_1007_1388_b200 import inputs, lbm
domain, patch, periodic = (48, 40, 64), (24, 20, 16), (1, 0, 0)
fl, wu = inputs.ldc_flags(domain, periodic); fl = inputs.add_obstacles(fl, 0.03, seed=13)
for steps in [int(v) for v in os.environ.get("STEPS", "1,2,3,5,20").split(",")]:
    obj = [lbm.nccl_unique_id() if rank == 0 else None]; dist.broadcast_object_list(obj, src=0)
    L = lbm.Lattice(domain, patch, inputs.LDC_OMEGA, 8, device=local, rank=rank, nranks=world, nccl_id=obj[0], periodic=periodic,
                    use_graphs=int(os.environ.get("GRAPHS", "1")))
    L.set_flags(fl, wu); f0 = inputs.noise_pdfs(domain, L.owned_lo, L.owned_hi); L.set_pdfs(f0)
    for _ in range(steps if os.environ.get("ONE_BY_ONE") else 1): L.step(1 if os.environ.get("ONE_BY_ONE") else steps)
    mine = (L.owned_lo, L.owned_hi, L.get_pdfs()); L.close()
    parts = [None] * world; dist.all_gather_object(parts, mine)
    if rank == 0:
        full = np.zeros((domain[2], domain[1], domain[0], 19))
        for lo, hi, a in parts: full[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]] = a
        with lbm.Lattice(domain, patch, inputs.LDC_OMEGA, 8, device=local, periodic=periodic) as L1:
            L1.set_flags(fl, wu); L1.set_pdfs(inputs.noise_pdfs(domain)); L1.step(steps); single = L1.get_pdfs()
        d = np.abs(full - single)
        bad = np.argwhere(d > 0)
        print("steps", steps, "ndiff", len(bad), "max", d.max(), flush=True)
        if len(bad):
            zs, ys, xs, qs = bad.T
            for name, v, n in (("x", xs, domain[0]), ("y", ys, domain[1]), ("z", zs, domain[2]), ("q", qs, 19)):
                print(f"  bad per {name}:", np.bincount(v, minlength=n).tolist(), flush=True)
dist.destroy_process_group()
