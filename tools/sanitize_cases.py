"""Small cases for compute-sanitizer: every sweep variant family once (two-grid
one/two cells, AA, TMA, local pull), multi-patch with periodic wrap and obstacles."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1007_1388_b200 import inputs  # noqa: E402


def run(layout=0, prec=8, env=None):
    for k, v in (env or {}).items():
        os.environ[k] = v
    from paper_1007_1388_b200 import lbm
    n = (37, 21, 13)
    fl, wu = inputs.ldc_flags(n, periodic=(0, 1, 0))
    fl = inputs.add_obstacles(fl, 0.05, seed=3, kinds=(inputs.NOSLIP, inputs.VELOCITY0 + 1))
    wu = np.vstack([wu, [[0.0, 0.01, 0.0]]])
    for patch in ((37, 21, 13), (37, 7, 13)):
        L = lbm.Lattice(n, patch, 1.3, prec, periodic=(0, 1, 0), layout=layout)
        L.set_flags(fl, wu)
        L.init_noise(1)
        L.step(3)
        L.get_pdfs()
        L.get_macroscopic()
        L.close()
    for k in (env or {}):
        os.environ.pop(k)


if __name__ == "__main__":
    for prec in (8, 4):
        run(0, prec)
        run(1, prec)
        run(0, prec, {"LBM_SWEEP_VARIANT": "5"})
        run(0, prec, {"LBM_SWEEP_IMPL": "tma"})
        run(0, prec, {"LBM_SWEEP_VARIANT": "5" if prec == 8 else "6", "LBM_LOCAL_PULL": "1"})
    print("sanitize cases done")
