import sys, os
sys.path.insert(0, '/root/repo')
from paper_1007_1388_b200 import lbm, inputs
n=(32,32,32)
fl,wu=inputs.ldc_flags(n)
L=lbm.Lattice(n,n,1.5,int(sys.argv[1]),device=0)
L.set_flags(fl,wu); L.init_noise(1)
L.step(1)
print("ok", os.environ.get("LBM_TMA_DEBUG"), sys.argv[1])
