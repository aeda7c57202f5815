"""Small cases covering every sweep family and exchange path once, in both
precisions -- two grids and AA, both occupancy variants, multi-patch direct
ghost stores, the NCCL exchange with the shell / interior overlap
(FORCE_BUFFERS, one-rank communicator) and the fused exchange with its epoch
handshake (SELF_PEER), with periodic wrap, obstacles on patch faces and two
moving walls.

compute-sanitizer is closed on the GPU pool (its runs left GPUs needing a
reset), so the cases run against the checked build instead (make checked;
kernels.cuh Checker: bounds, single writer per step, read/write races within
a launch), which fails the step with LBM_ERR_INTERNAL on any finding:

    LBM_LIBRARY=paper_1007_1388_b200/liblbm_b200_checked.so python tools/sanitize_cases.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1007_1388_b200 import inputs  # noqa: E402


def run(layout=0, prec=8, env=None, exchange_mode=0, n=(36, 21, 13), patches=((36, 21, 13), (36, 7, 13), (18, 7, 13))):
    for k, v in (env or {}).items():
        os.environ[k] = v
    from paper_1007_1388_b200 import lbm
    fl, wu = inputs.ldc_flags(n, periodic=(0, 1, 0))
    fl = inputs.add_obstacles(fl, 0.05, seed=3, kinds=(inputs.NOSLIP, inputs.VELOCITY0 + 1))
    wu = np.vstack([wu, [[0.0, 0.01, 0.0]]])
    for patch in patches:
        L = lbm.Lattice(n, patch, 1.3, prec, periodic=(0, 1, 0), layout=layout, exchange_mode=exchange_mode)
        L.set_flags(fl, wu)
        L.init_noise(1)
        L.step(3)
        L.get_pdfs()
        L.get_macroscopic()
        L.total_mass()
        L.close()
    for k in (env or {}):
        os.environ.pop(k)


if __name__ == "__main__":
    if "--first" in sys.argv:  # one case (the checked build's negative control)
        run(0, 8, patches=((36, 21, 13),))
        print("first case done")
        sys.exit(0)
    for prec in (8, 4):
        for layout in (0, 1):
            run(layout, prec)                                         # one patch, several, direct stores
            run(layout, prec, n=(37, 21, 13), patches=((37, 21, 13),))  # odd row length
            run(layout, prec, exchange_mode=1, patches=((18, 7, 13),))  # NCCL exchange, overlap
            run(layout, prec, exchange_mode=2, patches=((18, 7, 13),))  # fused exchange, handshake
        run(0, prec, {"LBM_SWEEP_VARIANT": "1"})
        run(0, prec, {"LBM_LOCAL_DIRECT": "0"}, patches=((18, 7, 13),))
    print("sanitize cases done")
