# bounce-back list kernel at 4 blocks of 256 threads per SM (64 registers)
PATCHES = [("aux_kernels.cu", "__global__ void __launch_bounds__(256, 3) bb_list_kernel", "__global__ void __launch_bounds__(256, 4) bb_list_kernel")]
