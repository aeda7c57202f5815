"""Worker for tests/test_multi_gpu.py::test_peer_timeout_reports_error (torchrun,
2 ranks).  Rank 1 sets up its lattice and then never steps; rank 0's fused
exchange must give up after LBM_PEER_TIMEOUT_S and report LBM_ERR_INTERNAL
through lbm_step instead of hanging the GPU.  Exit code 0 = pass."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    os.environ["LBM_PEER_TIMEOUT_S"] = "2"
    from paper_1007_1388_b200 import inputs, lbm
    domain, patch = (32, 32, 32 * world), (32, 32, 32)
    fl, wu = inputs.ldc_flags(domain)
    obj = [lbm.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    L = lbm.Lattice(domain, patch, inputs.LDC_OMEGA, lbm.LBM_FP64, device=local, rank=rank, nranks=world,
                    nccl_id=obj[0])
    L.set_flags(fl, wu)
    L.init_noise(inputs.NOISE_SEED)
    ok = L.info()["exchange_fused"] == 1
    dist.barrier()
    if rank == 0:
        t0 = time.time()
        try:
            L.step(3)
            ok = False
            print("rank 0: step returned without error", flush=True)
        except lbm.LbmError as e:
            dt = time.time() - t0
            print(f"rank 0: {e} after {dt:.1f} s", flush=True)
            ok = ok and e.status == 6 and "peer" in str(e) and 1.5 < dt < 60  # LBM_ERR_INTERNAL
    else:
        time.sleep(8)  # never steps
    dist.barrier()
    L.close()
    flag = torch.tensor([1 if ok else 0])
    dist.broadcast(flag, 0)
    dist.destroy_process_group()
    sys.exit(0 if flag.item() == 1 else 1)


if __name__ == "__main__":
    main()
